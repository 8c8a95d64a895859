// kernels.cu — sm_100a kernels of the flow-analysis hot path.
//
//   K1  k_sample, k_hot_select, k_table_slots
//                         hot-site plan for skewed batches (see plan_hot)
//   K2  k2_soa / k2_gen   classify -> attribute -> rate -> per-site aggregate
//                         (reduce_slice, rate_engine.cpp:197-240 + add :9-23)
//   K3a k3a_median_sb     per-site count and median super-bucket (round 1)
//   K2b k2b_fine          the median super-bucket's fine counts from the log
//   K3b k3b_finalize      per-site median / clamp / avg / flag
//                         (finalize + stats_from + median_bps,
//                          rate_engine.cpp:42-58, 242-292; monitor.cpp:22)
//       k_hist_from_log   dense histograms on request
//       k_classify        per-record class/site (classify/attribute :71-86, 127-146)
//
// Paths are relative to /root/reference/proj/core/src.
//
// The path is HBM-bound integer work: 32 algorithmic bytes per
// record, no tensor cores. K2 streams the six SoA columns with vector
// non-allocating loads, probes a shared-memory-resident radix table
// (registry.hpp), and reduces into order-independent integer/min/max
// accumulators, so the result is bit-identical to the reference for any
// grid, partitioning or GPU count.
//
// K2 is two stages per warp. Stage A (every lane, every record): the class
// filter and the /16 directory bits of both endpoints. Candidates (~40% of
// records at D3) are compacted into a per-warp shared-memory queue, and
// stage B drains it 32 at a time with full warps: the /24 lookup tail, the
// rate, the exact micro-bps, the bucket and the reductions, plus one log
// entry per flow (site, bucket) for the second round of the median.
//
// Contention: with Zipf-distributed sites the hottest site receives ~10% of
// all Forward flows; same-address L2 atomics serialise and returning
// shared-memory atomics expose their latency to the warp. The sums of the hot
// sites (up to 2047, chosen by K1 from a 1/64 sample) therefore accumulate in
// block-private shared memory through NON-returning 32-bit adds of 16-bit
// limbs; a persistent CTA normalises the limbs at a barrier every
// kEpochRounds rounds (fewer than 2^16 adds per limb in between), and the
// top 32 hot sites also keep their coarse counts in shared memory. Cold sites
// go straight to L2 with RED; the median needs only 157 coarse counts per
// site (round 1) and, at finalize, the fine counts of one super-bucket.
#include <cuda_runtime.h>

#include <algorithm>

#include "kernels.cuh"
#include "rate.cuh"

namespace gnm {
namespace {

constexpr uint32_t kNone = 0xFFFFFFFFu;
constexpr uint32_t kDirWordsDev = 4096u; // registry.hpp kDirWords
#ifndef GNM_K2_BLOCK
#define GNM_K2_BLOCK 768
#endif
constexpr int kK2Block = GNM_K2_BLOCK; // 24 warps: up to 80 registers per thread
constexpr uint32_t kWarps = kK2Block / 32;
// Records one non-persistent K2 CTA (k2_gen) may process: every 16-bit limb
// of a hot slot then sums fewer than 2^16 values below 2^16 and cannot wrap
// its u32. The persistent k2_soa bounds them per epoch instead.
constexpr uint64_t kCtaRecords = 65536 - 64;
// k2_soa epochs: kEpochRounds rounds of kWarps 64-record tiles, plus the
// queue residue (< 32 per warp) and the < 64-record tail, stay below 2^16
// adds per limb; between epochs any limb that could wrap in the next one
// (>= kLimbFlush) is flushed to L2.
#ifndef GNM_EPOCH_ROUNDS
#define GNM_EPOCH_ROUNDS 29
#endif
constexpr uint32_t kEpochRounds = GNM_EPOCH_ROUNDS; // measurement builds may override (unsafe above 29)
constexpr uint32_t kLimbFlush = 1u << 28;
constexpr uint32_t kQueue = 96; // per-warp queue capacity: < 32 left + 2 x 32 pushed
// The top kCoarseSlots hot slots also keep their coarse counts in shared memory.
constexpr uint32_t kCoarseSlots = 32;
// Hot slots 1..kTopReplicas all belong to the most sampled site (a power of 2).
#ifndef GNM_TOP_REPLICAS
#define GNM_TOP_REPLICAS 4
#endif
constexpr uint32_t kTopReplicas = GNM_TOP_REPLICAS;
// K2b's shared-memory fine rows for the heaviest sites.
constexpr uint32_t kHeavy = 64;
constexpr uint32_t kHeavyNone = 0xFFFFFFu;
constexpr uint64_t kHeavyMin = 1u << 16;
constexpr uint32_t kLogChunk = 2048; // K2b work-item size
constexpr size_t kHotBytes = kHotStride * (5 * 4 + 2 * 8) + kCoarseSlots * kCoarse * 4;
constexpr size_t kSmemMax = 227 * 1024;
constexpr size_t kQueueBytes = kWarps * kQueue * 16;
constexpr size_t kSmemTableMax = kSmemMax - kHotBytes - kQueueBytes - 1024;

extern __shared__ __align__(16) uint32_t g_smem[];

// ---- streaming loads (read once: do not pollute L1) ----------------------
// The input is read once: stream it through L2 with an evict-first policy so
// it does not push out the histogram and accumulator lines the reductions
// hit (profiles/round1: RED throughput collapses once they miss L2).
__device__ __forceinline__ uint64_t evict_first_policy() {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ uint2 ld_stream_u2(const void* p, uint64_t pol) {
    uint2 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.L2::256B.v2.u32 {%0,%1}, [%2], %3;"
                 : "=r"(r.x), "=r"(r.y)
                 : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ ulonglong2 ld_stream_u64x2(const void* p, uint64_t pol) {
    ulonglong2 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.L2::256B.v2.u64 {%0,%1}, [%2], %3;"
                 : "=l"(r.x), "=l"(r.y)
                 : "l"(p), "l"(pol));
    return r;
}

// ---- fire-and-forget reductions (RED, never a returning ATOM) --------------
__device__ __forceinline__ void red_add(unsigned long long* p, unsigned long long v) {
    asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v));
}
__device__ __forceinline__ void red_add(unsigned int* p, unsigned int v) {
    asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v));
}
__device__ __forceinline__ void red_min(unsigned long long* p, unsigned long long v) {
    asm volatile("red.relaxed.gpu.global.min.u64 [%0], %1;" ::"l"(p), "l"(v));
}
__device__ __forceinline__ void red_max(unsigned long long* p, unsigned long long v) {
    asm volatile("red.relaxed.gpu.global.max.u64 [%0], %1;" ::"l"(p), "l"(v));
}
__device__ __forceinline__ void red_add_shared(uint32_t* p, uint32_t v) {
    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(p))),
                 "r"(v)
                 : "memory");
}

// ---- registry table (layout in registry.hpp, DeviceTable) -----------------
template <bool kSmem>
__device__ __forceinline__ uint32_t table_word(const uint32_t* __restrict__ gt, uint32_t i) {
    if constexpr (kSmem) return g_smem[i];
    else return __ldg(gt + i);
}
template <bool kSmem>
__device__ __forceinline__ uint2 table_pair(const uint32_t* __restrict__ gt, uint32_t pair) {
    if constexpr (kSmem) return reinterpret_cast<const uint2*>(g_smem)[pair];
    else return __ldg(reinterpret_cast<const uint2*>(gt) + pair);
}

// SiteCatalog::lookup (site_catalog.hpp:99-112) over the radix table:
// one LDS.64 for a miss, three dependent LDS for a /24 hit. Returns the
// packed (slot << 20 | site) value, or kNone.
template <bool kSmem>
__device__ __forceinline__ uint32_t lookup(const uint32_t* __restrict__ gt, uint32_t ip) {
    const uint32_t d = ip >> 16;
    const uint2 w = table_pair<kSmem>(gt, d >> 5);
    const uint32_t bit = d & 31u;
    if (!((w.x >> bit) & 1u)) return kNone;
    const uint32_t node = table_word<kSmem>(gt, kDirWordsDev + w.y + __popc(w.x & ((1u << bit) - 1u)));
    if (node & 0x80000000u) return node & 0x7FFFFFFFu;
    return table_word<kSmem>(gt, node + ((ip >> 8) & 0xFFu));
}

// attribute (rate_engine.cpp:127-146) with full src-then-dst probes.
template <bool kSmem>
__device__ __forceinline__ uint32_t site_of_full(const uint32_t* __restrict__ gt, uint32_t src,
                                                 uint32_t dst) {
    const uint32_t v = lookup<kSmem>(gt, src);
    return v != kNone ? v : lookup<kSmem>(gt, dst);
}

template <bool kSmem>
__device__ __forceinline__ void load_table(const uint32_t* __restrict__ gt, uint32_t words) {
    if constexpr (kSmem) {
        const uint4* g4 = reinterpret_cast<const uint4*>(gt);
        uint4* s4 = reinterpret_cast<uint4*>(g_smem);
        for (uint32_t i = threadIdx.x; i < words / 4; i += blockDim.x) s4[i] = __ldg(g4 + i);
    }
}

// A table word with this call's hot slot (k_table_slots' rewrite, done here
// on the shared-memory copy): uniform nodes and leaf entries carry
// slot << 20 | site.
__device__ __forceinline__ uint32_t with_slot(uint32_t w, uint32_t j, const DevHot& hot) {
    if (j < hot.node_begin) return w;
    if (j < hot.leaf_begin) {
        if (!(w & 0x80000000u)) return w;
        const uint32_t site = w & 0xFFFFFu;
        return 0x80000000u | __ldg(hot.site_slot + site) << 20 | site;
    }
    if (w == 0xFFFFFFFFu) return w;
    const uint32_t site = w & 0xFFFFFu;
    return __ldg(hot.site_slot + site) << 20 | site;
}

template <bool kSmem, bool kHot>
__device__ __forceinline__ void load_table_slots(const uint32_t* __restrict__ gt, uint32_t words, const DevHot& hot) {
    if constexpr (kSmem && kHot) {
        if (hot.site_slot) {
            const uint4* g4 = reinterpret_cast<const uint4*>(gt);
            uint4* s4 = reinterpret_cast<uint4*>(g_smem);
            for (uint32_t i = threadIdx.x; i < words / 4; i += blockDim.x) {
                uint4 v = __ldg(g4 + i);
                v.x = with_slot(v.x, 4 * i, hot);
                v.y = with_slot(v.y, 4 * i + 1, hot);
                v.z = with_slot(v.z, 4 * i + 2, hot);
                v.w = with_slot(v.w, 4 * i + 3, hot);
                s4[i] = v;
            }
            return;
        }
    }
    load_table<kSmem>(gt, words);
}

// ---- block-private hot-site accumulators ---------------------------------
// Per slot: octets as two 16-bit limbs, micro-bps (< 2^48) as three 16-bit
// limbs, each summed into its own u32 by non-returning shared adds; min/max
// as f64 bit patterns.
struct HotSmem {
    uint32_t* limb; // [5][kHotStride]: oct lo16, oct hi16, ubps bits 0-15, 16-31, 32-47
    unsigned long long* mn;
    unsigned long long* mx;
    uint32_t* coarse; // [kCoarseSlots][kCoarse], slot 1 first
};

__device__ __forceinline__ HotSmem hot_smem(uint32_t table_words_in_smem) {
    uint32_t* base = g_smem + table_words_in_smem;
    HotSmem h;
    h.limb = base;
    h.mn = reinterpret_cast<unsigned long long*>(base + 5 * kHotStride);
    h.mx = h.mn + kHotStride;
    h.coarse = reinterpret_cast<uint32_t*>(h.mx + kHotStride);
    return h;
}

// The min/max caches start from the hot sites' global bounds, which K1
// already pulled in from the sample's flows (k_sample): every value there is
// a rate whose reduction was issued, so the cache invariant below holds, and
// the CTA's first flows of a hot site no longer all win against +inf / 0.
__device__ __forceinline__ void hot_init(const HotSmem& h, const DevHot& hot, const DevPartials& P) {
    for (uint32_t i = threadIdx.x; i < kHotStride; i += blockDim.x) {
#pragma unroll
        for (int k = 0; k < 5; ++k) h.limb[k * kHotStride + i] = 0;
        unsigned long long mn = kMinInitBits, mx = kMaxInitBits;
        if (i >= 1 && i <= hot.n_slots) {
            const uint32_t site = __ldg(hot.hot_site + i); // unassigned slots: stale, unused
            if (site < P.n_sites) {
                mn = __ldcg(P.mn + site);
                mx = __ldcg(P.mx + site);
            }
        }
        h.mn[i] = mn;
        h.mx[i] = mx;
    }
    for (uint32_t i = threadIdx.x; i < kCoarseSlots * kCoarse; i += blockDim.x) h.coarse[i] = 0;
}

// ---- per-flow arithmetic -----------------------------------------------------
// flow_rate_dev / ubps_of / ubps_slow: rate.cuh (shared with hosts.cu).

// bucket_index (rate_engine.cpp:119-125) from the exact quotient:
// floor(RN(RN(8000*oct/dur)/1e4)) == floor(4*oct/(5*dur)) for every u32 oct
// (the two roundings move the value by < v*2^-52, while a non-integer
// 4*oct/(5*dur) is at least 1/(5*dur) away from the next integer, and
// 4*oct < 2^52), and floor(4*oct/(5*dur)) == floor(ubps / 1e10).
// Checked against the reference's double arithmetic on adversarial inputs
// (tests/test_oracle_golden.py::test_integer_bucket_identity).
__device__ __forceinline__ uint32_t bucket_of_ubps(uint64_t lo, uint64_t hi) {
    const uint64_t b = lo / 10000000000ull;
    return (hi || b >= 10000u) ? 10000u : static_cast<uint32_t>(b);
}


// ---- per-record classification (stage A, every lane) -----------------------
// FlowStore::snapshot's predicate (flow_store.cpp:75): end_ms in [lo, hi).
// The window-fused K2 applies it before classification, exactly as the
// reference analyzes only the snapshot's copy of the window.
template <bool kWin>
__device__ __forceinline__ bool window_in(uint64_t end, const DevParams& p) {
    if constexpr (kWin) return end >= p.win_lo && end < p.win_hi;
    else return true;
}

// Per-lane tallies (ClassTallies, rate_engine.hpp:101-110).
struct Ctr {
    uint32_t fwd = 0, ack = 0, adm = 0, unm = 0;
};

// A queued flow's site code: either RESOLVED | site value, or the node index
// (< 2^16) of the /16 block that holds the winning endpoint << 8 | the
// endpoint's third octet, resolved to a site in stage B.
constexpr uint32_t kResolved = 0x80000000u;
constexpr uint32_t kSkip = 0xFFFFFFFFu;

// `in`: the record lies in the analysis window (window-fused variant, see
// window_in); records outside it are not counted at all.
// reduce_slice's per-record filter (rate_engine.cpp:199-215) and the first
// half of attribute (:127-146), branch-free, in the reference's order:
//   ack = octets < (ack_max+1) * pkts          (false when pkts == 0)
//   rej = pkts < max(min_packets,1) || dur < max(min_duration,1)
// (pkts == 0 and dur == 0 fold into rej), then both endpoints' /16
// directory bits (one LDS.64 each). A candidate whose endpoints both miss
// is Unmatched here; otherwise the src-first winner's node index is queued.
// When both /16s hold sites (src may still miss at /24) the full lookup runs
// now, on those lanes only.
template <bool kSmem>
__device__ __forceinline__ uint32_t stage_a(uint32_t src, uint32_t dst, uint32_t pkts, uint32_t oct,
                                            uint64_t dur, const DevParams& p,
                                            const uint32_t* __restrict__ gt, Ctr& c, uint32_t& host,
                                            bool in = true) {
    const bool ack = static_cast<uint64_t>(oct) < p.ack_plus1 * pkts;
    const bool rej = pkts < p.min_packets1 || dur < static_cast<uint64_t>(p.min_duration1);
    const uint32_t ds = src >> 16, dd = dst >> 16;
    const uint2 ws = table_pair<kSmem>(gt, ds >> 5);
    const uint2 wd = table_pair<kSmem>(gt, dd >> 5);
    const bool hs = (ws.x >> (ds & 31u)) & 1u;
    const bool hd = (wd.x >> (dd & 31u)) & 1u;
    if (in && ack) ++c.ack;
    if (in && !ack && rej) ++c.adm;
    const bool cand = in && !ack && !rej;
    if (cand && !(hs | hd)) ++c.unm;
    const uint32_t bits = hs ? ws.x : wd.x;
    const uint32_t rank0 = hs ? ws.y : wd.y;
    const uint32_t d = hs ? ds : dd;
    const uint32_t ip = hs ? src : dst;
    const uint32_t rank = rank0 + __popc(bits & ~(0xFFFFFFFFu << (d & 31u)));
    uint32_t code = (cand && (hs | hd)) ? (rank << 8 | ((ip >> 8) & 0xFFu)) : kSkip;
    host = ip; // the matched endpoint (rate_engine.cpp:218-223): src unless only dst's /16 holds sites
#ifdef GNM_K2_ABLATION
    if (p.ablation == 1) {
        if (cand) c.fwd += rank;
        code = kSkip;
    }
#endif
    if (cand && hs && hd) {
        const uint32_t vs = lookup<kSmem>(gt, src);
        const uint32_t v = vs != kNone ? vs : lookup<kSmem>(gt, dst);
        host = vs != kNone ? src : dst;
        if (v == kNone) ++c.unm;
        code = v == kNone ? kSkip : (kResolved | v);
    }
    return code;
}

// Stage B: the site value of a queued code (kNone: Unmatched at /24).
template <bool kSmem>
__device__ __forceinline__ uint32_t resolve(const uint32_t* __restrict__ gt, uint32_t code) {
    const bool res = code & kResolved;
    const uint32_t node = table_word<kSmem>(gt, res ? 0u : kDirWordsDev + (code >> 8));
    const bool uni = node >> 31;
    const uint32_t leaf = table_word<kSmem>(gt, (res || uni) ? 0u : node + (code & 0xFFu));
    return res ? (code & 0x7FFFFFFFu) : (uni ? (node & 0x7FFFFFFFu) : leaf);
}

// RateHistogram::add (rate_engine.cpp:9-23) for one Forward flow, as
// order-independent reductions:
//   coarse[site][bucket >> 6] += 1   (+ a log entry: the exact bucket for round 2)
//   octets and micro-bps sums        exact integers
//   min/max of the f64 rate via u64 min/max on the bit pattern (rates > 0,
//   SURVEY.md §8a' #8)
// Hot sites: non-returning shared adds of 16-bit limbs (micro-bps >= 2^48 go
// to L2 instead), coarse counts of the top kCoarseSlots slots in shared
// memory too; min/max go to L2 only when the slot's cached bounds say they
// can win. Cold sites: straight to L2 (RED).
// Returns the site (kNone: Unmatched at /24) and the bucket.
// K2 compile-time modes (kMode bits).
constexpr int kModeWindow = 1; // FlowStore::snapshot window fused (DevParams::windowed)
constexpr int kModeHosts = 2;  // hosts mode: log host, octets, duration per Forward flow

struct FlowOut {
    uint32_t bucket = 0;
    unsigned long long rate_bits = 0;
    uint64_t lo = 0, hi = 0;
    uint32_t oct = 0; // hosts mode: what H1 recomputes the rate and micro-bps from
    uint64_t dur = 0;
};

template <bool kSmem, bool kHot>
__device__ __forceinline__ uint32_t accumulate(uint32_t code, uint32_t oct, uint64_t dur,
                                               const uint32_t* __restrict__ gt, const DevParams& p,
                                               const DevPartials& P, const HotSmem& h, Ctr& c,
                                               FlowOut& fo) {
    uint32_t& bucket = fo.bucket;
    bucket = 0;
    fo.oct = oct;
    fo.dur = dur;
    // flow_rate (rate_engine.cpp:88-94): exact product, one IEEE division.
    // Issued before the lookup: it needs only the record, so its dependent
    // DFMA chain overlaps the table loads (an Unmatched item wastes it).
#ifdef GNM_K2_ABLATION
    // 5: a single-MUFU approximate rate instead of the IEEE division (wrong
    // results; measures what the exact division costs)
    const double rate = p.ablation == 5
        ? static_cast<double>(__fdividef(8000.0f * static_cast<float>(oct), static_cast<float>(dur)))
        : flow_rate_dev(oct, dur);
#else
    const double rate = flow_rate_dev(oct, dur);
#endif
    const uint32_t v = resolve<kSmem>(gt, code);
    if (v == kNone) {
        ++c.unm;
        return kNone;
    }
    ++c.fwd;
    const uint32_t site = v & p.site_mask;
#ifdef GNM_K2_ABLATION
    if (p.ablation == 2) {
        c.unm ^= v ^ oct ^ static_cast<uint32_t>(dur);
        return site;
    }
#endif
    uint32_t slot = kHot ? (v >> 20) & 0x7FFu : 0u;
    if (kHot && slot == 1u) slot += threadIdx.x & (kTopReplicas - 1); // the top site's replicas (k_hot_select)
    unsigned long long cmn = 0, cmx = ~0ull;
    if (kHot && slot) { // issued early: the latency hides behind the division
        cmn = h.mn[slot];
        cmx = h.mx[slot];
    }
    uint64_t lo, hi;
    ubps_of(oct, dur, rate, lo, hi);
    const unsigned long long rb = static_cast<unsigned long long>(__double_as_longlong(rate));
    bucket = bucket_of_ubps(lo, hi);
    fo.rate_bits = rb;
    fo.lo = lo;
    fo.hi = hi;
    const uint32_t sb = bucket >> 6;
#ifdef GNM_K2_ABLATION
    // Measurement builds only (tools/ablation.sh): 3 = no reductions at all,
    // 4 = coarse counts (and the log) only. Results are wrong in these modes.
    if (p.ablation == 3 || p.ablation == 4) {
        if (p.ablation == 4) {
            if (kHot && slot && slot <= kCoarseSlots)
                red_add_shared(h.coarse + (slot - 1) * kCoarse + sb, 1u);
            else red_add(P.coarse + static_cast<size_t>(sb) * P.n_sites + site, 1u);
        }
        c.unm ^= static_cast<uint32_t>(lo ^ hi ^ rb) ^ static_cast<uint32_t>(cmn ^ cmx);
        return p.ablation == 3 ? kNone : site;
    }
#endif
    unsigned long long* s = P.sums + static_cast<size_t>(site) * 4;
#ifdef GNM_K2_ABLATION
    // 6: everything but min/max; 7: everything but the octet / micro-bps sums
    const bool abl_nominmax = p.ablation == 6, abl_nosums = p.ablation == 7;
#else
    constexpr bool abl_nominmax = false, abl_nosums = false;
#endif
    if (kHot && slot) {
        uint32_t* l = h.limb + slot;
        if (!abl_nosums) {
        red_add_shared(l, oct & 0xFFFFu);
        red_add_shared(l + kHotStride, oct >> 16);
        if (hi == 0 && lo < (1ull << 48)) {
            red_add_shared(l + 2 * kHotStride, static_cast<uint32_t>(lo) & 0xFFFFu);
            red_add_shared(l + 3 * kHotStride, static_cast<uint32_t>(lo) >> 16);
            red_add_shared(l + 4 * kHotStride, static_cast<uint32_t>(lo >> 32));
        } else {
            red_add(s + 1, lo & 0xFFFFFFFFull);
            red_add(s + 2, lo >> 32);
            if (hi) red_add(s + 3, hi);
        }
        }
        if (slot <= kCoarseSlots)
            red_add_shared(h.coarse + (slot - 1) * kCoarse + sb, 1u);
        else
            red_add(P.coarse + static_cast<size_t>(sb) * P.n_sites + site, 1u);
        // min/max: the slot's cached bounds filter the global reductions. The
        // cache moves (shared atomics; rare after the first flows) only AFTER
        // the RED, so it only ever holds rates whose RED was issued: a stale
        // read costs an extra RED but never hides a winning update.
        if (rb < cmn && !abl_nominmax) {
            red_min(P.mn + site, rb);
            atomicMin(h.mn + slot, rb);
        }
        if (rb > cmx && !abl_nominmax) {
            red_max(P.mx + site, rb);
            atomicMax(h.mx + slot, rb);
        }
    } else {
        red_add(P.coarse + static_cast<size_t>(sb) * P.n_sites + site, 1u);
        if (!abl_nosums) {
            red_add(s + 0, static_cast<unsigned long long>(oct));
            red_add(s + 1, lo & 0xFFFFFFFFull);
            if (lo >> 32) red_add(s + 2, lo >> 32);
            if (hi) red_add(s + 3, hi);
        }
        if (!abl_nominmax) {
            red_min(P.mn + site, rb);
            red_max(P.mx + site, rb);
        }
    }
    return site;
}

// Warp-level stream compaction of candidates: lanes append {code, octets,
// duration} to the warp's shared queue (ballot + popc, one STS.128), and
// every time 32 are queued the whole warp drains one per lane (stage B), so
// the lookup tail and the per-flow arithmetic never run with the ~50% lane
// occupancy the class mix would otherwise leave them. Each drained item
// leaves one log entry (a 128-byte coalesced streaming store per drain) in
// the warp's region of the launch's log.
struct WarpQueue {
    uint4* q;
    uint32_t* qh;       // hosts mode: the matched host IP per queued item
    uint32_t n;         // warp-uniform fill
    uint32_t pos;       // warp-uniform log entries written
    unsigned int* log;  // this warp's log region
    unsigned int* logb; // wide registries: bucket column of the region
    size_t region_off;  // hosts mode: the region's offset into the host columns
};

template <bool kHosts>
__device__ __forceinline__ void push(uint32_t code, uint32_t oct, uint64_t dur, WarpQueue& wq,
                                     uint32_t lane, uint32_t host) {
    const bool f = code != kSkip;
    const unsigned m = __ballot_sync(0xFFFFFFFFu, f);
    if (f) {
        const uint32_t i = wq.n + __popc(m & ((1u << lane) - 1u));
        wq.q[i] = make_uint4(code, oct, static_cast<uint32_t>(dur), static_cast<uint32_t>(dur >> 32));
        if constexpr (kHosts) wq.qh[i] = host;
    }
    wq.n += __popc(m);
}

// The drained Forward flows' entries, compacted (Unmatched lanes write none);
// every lane of the warp calls this.
template <bool kHosts>
__device__ __forceinline__ void log_entry(WarpQueue& wq, uint32_t lane, uint32_t site, const FlowOut& fo,
                                          uint32_t host, const DevLog& L) {
    const bool v = site != kNone;
    const unsigned m = __ballot_sync(0xFFFFFFFFu, v);
    if (v) {
        const uint32_t i = wq.pos + __popc(m & ((1u << lane) - 1u));
        if (wq.logb) {
            __stcs(wq.log + i, site);
            __stcs(wq.logb + i, fo.bucket);
        } else {
            __stcs(wq.log + i, site << kLogSiteShift | fo.bucket);
        }
        if constexpr (kHosts) { // the flow's host, octets and duration (H1 recomputes rate and micro-bps)
            const size_t j = wq.region_off + i;
            __stcs(L.hosts + j, host);
            __stcs(L.octs + j, fo.oct);
            __stcs(L.durs + j, static_cast<unsigned long long>(fo.dur));
        }
    }
    wq.pos += __popc(m);
}

template <bool kSmem, bool kHot, bool kHosts>
__device__ __forceinline__ void drain_full(WarpQueue& wq, uint32_t lane,
                                           const uint32_t* __restrict__ gt, const DevParams& p,
                                           const DevPartials& P, const HotSmem& h, Ctr& c,
                                           const DevLog& L) {
    while (wq.n >= 32) {
        __syncwarp();
        const uint32_t k = wq.n - 32 + lane;
        const uint4 x = wq.q[k];
        uint32_t host = 0;
        if constexpr (kHosts) host = wq.qh[k];
        wq.n -= 32;
        __syncwarp();
        FlowOut fo;
        const uint32_t site =
            accumulate<kSmem, kHot>(x.x, x.y, static_cast<uint64_t>(x.w) << 32 | x.z, gt, p, P, h, c, fo);
        log_entry<kHosts>(wq, lane, site, fo, host, L);
    }
}

template <bool kSmem, bool kHot, bool kHosts>
__device__ __forceinline__ void drain_rest(WarpQueue& wq, uint32_t lane,
                                           const uint32_t* __restrict__ gt, const DevParams& p,
                                           const DevPartials& P, const HotSmem& h, Ctr& c,
                                           const DevLog& L) {
    __syncwarp();
    uint32_t site = kNone, host = 0;
    FlowOut fo;
    if (lane < wq.n) {
        const uint4 x = wq.q[lane];
        if constexpr (kHosts) host = wq.qh[lane];
        site = accumulate<kSmem, kHot>(x.x, x.y, static_cast<uint64_t>(x.w) << 32 | x.z, gt, p, P, h, c, fo);
    }
    log_entry<kHosts>(wq, lane, site, fo, host, L);
    wq.n = 0;
}

__device__ __forceinline__ void flush_tallies(const Ctr& t, unsigned long long* out) {
    const uint32_t f = __reduce_add_sync(0xFFFFFFFFu, t.fwd);
    const uint32_t a = __reduce_add_sync(0xFFFFFFFFu, t.ack);
    const uint32_t d = __reduce_add_sync(0xFFFFFFFFu, t.adm);
    const uint32_t u = __reduce_add_sync(0xFFFFFFFFu, t.unm);
    if ((threadIdx.x & 31u) == 0) {
        if (f) red_add(out + 0, static_cast<unsigned long long>(f));
        if (a) red_add(out + 1, static_cast<unsigned long long>(a));
        if (d) red_add(out + 2, static_cast<unsigned long long>(d));
        if (u) red_add(out + 3, static_cast<unsigned long long>(u));
    }
}

// One flush per CTA. The limb sums are exact (< 2^32 each, see kCtaRecords)
// and land in the global limbs K3b reassembles: sums[1] takes the low 32
// bits of every flow's micro-bps (so it stays below count * 2^32), sums[2]
// the bits above. Coarse counts of the top slots: each u16 half to its
// super-bucket. (min/max went to L2 during the run.)
__device__ __forceinline__ void hot_flush(const HotSmem& h, const DevHot& hot, const DevPartials& P) {
    for (uint32_t slot = 1 + threadIdx.x; slot <= hot.n_slots; slot += blockDim.x) {
        const uint32_t* l = h.limb + slot;
        const uint64_t oct = static_cast<uint64_t>(l[0]) + (static_cast<uint64_t>(l[kHotStride]) << 16);
        const uint64_t u01 = static_cast<uint64_t>(l[2 * kHotStride]) +
                             (static_cast<uint64_t>(l[3 * kHotStride]) << 16);
        const uint32_t u2 = l[4 * kHotStride];
        if (oct == 0) continue; // untouched: every Forward flow has >= 1 octet
        const uint32_t site = __ldg(hot.hot_site + slot);
        unsigned long long* s = P.sums + static_cast<size_t>(site) * 4;
        red_add(s + 0, oct);
        if (u01) red_add(s + 1, u01);
        if (u2) red_add(s + 2, static_cast<unsigned long long>(u2));
    }
    const uint32_t words = min(hot.n_slots, kCoarseSlots) * kCoarse;
    for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) {
        const uint32_t w = h.coarse[i];
        if (!w) continue;
        const uint32_t site = __ldg(hot.hot_site + 1 + i / kCoarse);
        red_add(P.coarse + static_cast<size_t>(i % kCoarse) * P.n_sites + site, w);
    }
}

// Between k2_soa epochs (CTA-wide, after a barrier): flush and clear every
// limb that might wrap during the next epoch; everything else stays.
__device__ __forceinline__ void hot_normalize(const HotSmem& h, const DevHot& hot, const DevPartials& P) {
    for (uint32_t slot = 1 + threadIdx.x; slot <= hot.n_slots; slot += blockDim.x) {
        uint32_t* l = h.limb + slot;
        const uint32_t m = max(max(max(l[0], l[kHotStride]), max(l[2 * kHotStride], l[3 * kHotStride])),
                               l[4 * kHotStride]);
        if (m < kLimbFlush) continue;
        const uint32_t site = __ldg(hot.hot_site + slot);
        unsigned long long* s = P.sums + static_cast<size_t>(site) * 4;
        red_add(s + 0, static_cast<uint64_t>(l[0]) + (static_cast<uint64_t>(l[kHotStride]) << 16));
        red_add(s + 1, static_cast<uint64_t>(l[2 * kHotStride]) + (static_cast<uint64_t>(l[3 * kHotStride]) << 16));
        red_add(s + 2, static_cast<unsigned long long>(l[4 * kHotStride]));
#pragma unroll
        for (int k = 0; k < 5; ++k) l[k * kHotStride] = 0;
    }
    const uint32_t words = min(hot.n_slots, kCoarseSlots) * kCoarse;
    for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) {
        const uint32_t w = h.coarse[i];
        if (w < kLimbFlush) continue;
        red_add(P.coarse + static_cast<size_t>(i % kCoarse) * P.n_sites + __ldg(hot.hot_site + 1 + i / kCoarse), w);
        h.coarse[i] = 0;
    }
}

// One record by index (scalar loads; tails and the non-vector layouts).
// kLayout 1: SoA; 2/3: 64-byte flowmon::FlowRecord rows (netflow.hpp:59-67).
template <int kLayout>
__device__ __forceinline__ void load_record(const DevBatch& b, uint64_t i, uint32_t& src, uint32_t& dst,
                                            uint32_t& pkts, uint32_t& oct, uint64_t& dur, uint64_t& end) {
    if constexpr (kLayout == 1) {
        const DevSoA& c = b.soa;
        src = c.src[i], dst = c.dst[i], pkts = c.pkts[i], oct = c.octets[i];
        end = c.end[i];
        dur = end - c.start[i];
    } else if constexpr (kLayout == 5) { // compacted: only the duration (never windowed)
        const DevSoA& c = b.soa;
        src = c.src[i], dst = c.dst[i], pkts = c.pkts[i], oct = c.octets[i];
        dur = c.dur32[i];
        end = dur;
    } else if constexpr (kLayout == 2) {
        const unsigned char* r = static_cast<const unsigned char*>(b.rec) + i * 64;
        const uint2 a = __ldg(reinterpret_cast<const uint2*>(r));                 // src dst
        const uint2 cc = __ldg(reinterpret_cast<const uint2*>(r + 16));           // pkts octets
        const ulonglong2 e = __ldg(reinterpret_cast<const ulonglong2*>(r + 48));  // start end
        src = a.x, dst = a.y, pkts = cc.x, oct = cc.y, dur = e.y - e.x, end = e.y;
    } else if constexpr (kLayout == 3) {
        const unsigned char* r = static_cast<const unsigned char*>(b.rec) + i * 64;
        const uint32_t* w = reinterpret_cast<const uint32_t*>(r);
        const uint64_t* qq = reinterpret_cast<const uint64_t*>(r + 48);
        src = w[0], dst = w[1], pkts = w[4], oct = w[5], dur = qq[1] - qq[0], end = qq[1];
    } else {
        // FLOWARC1 entry in place (flow_store.cpp:158-162): be64 start, be64
        // end, then the 48-byte big-endian raw record (netflow.cpp:52-75).
        // Entries sit at 20 + 64*i: 4-byte aligned words, byte-swapped.
        const uint32_t* w = reinterpret_cast<const uint32_t*>(static_cast<const unsigned char*>(b.rec) + i * 64);
        const uint64_t start = static_cast<uint64_t>(__byte_perm(__ldg(w + 0), 0, 0x0123)) << 32 |
                               __byte_perm(__ldg(w + 1), 0, 0x0123);
        end = static_cast<uint64_t>(__byte_perm(__ldg(w + 2), 0, 0x0123)) << 32 | __byte_perm(__ldg(w + 3), 0, 0x0123);
        src = __byte_perm(__ldg(w + 4), 0, 0x0123);
        dst = __byte_perm(__ldg(w + 5), 0, 0x0123);
        pkts = __byte_perm(__ldg(w + 8), 0, 0x0123);
        oct = __byte_perm(__ldg(w + 9), 0, 0x0123);
        dur = end - start;
    }
}

// Records [first, last) in warp-strided 32-record rounds, scalar loads.
template <int kLayout, bool kSmem, bool kHot, int kMode>
__device__ __forceinline__ void run_scalar(const DevBatch& b, uint64_t first, uint64_t last,
                                           uint64_t stride, uint32_t lane,
                                           const uint32_t* __restrict__ gt, const DevParams& p,
                                           const DevPartials& P, const HotSmem& h, Ctr& t,
                                           WarpQueue& wq, const DevLog& L) {
    constexpr bool kWin = kMode & kModeWindow, kHosts = kMode & kModeHosts;
    // One round ahead: the next record's loads are in flight while this one
    // is classified.
    uint32_t nsrc = 0, ndst = 0, npkts = 0, noct = 0;
    uint64_t ndur = 0, nend = 0;
    if (first + lane < last) load_record<kLayout>(b, first + lane, nsrc, ndst, npkts, noct, ndur, nend);
    for (uint64_t base = first; base < last; base += stride) {
        const uint64_t i = base + lane;
        const uint32_t src = nsrc, dst = ndst, pkts = npkts, oct = noct;
        const uint64_t dur = ndur, end = nend;
        const bool ok = i < last;
        if (i + stride < last) load_record<kLayout>(b, i + stride, nsrc, ndst, npkts, noct, ndur, nend);
        Ctr one;
        uint32_t host;
        const uint32_t code = stage_a<kSmem>(src, dst, pkts, oct, dur, p, gt, one, host, window_in<kWin>(end, p));
        if (ok) {
            t.ack += one.ack;
            t.adm += one.adm;
            t.unm += one.unm;
        }
        push<kHosts>(ok ? code : kSkip, oct, dur, wq, lane, host);
        drain_full<kSmem, kHot, kHosts>(wq, lane, gt, p, P, h, t, L);
    }
}

// ---- K2 ----------------------------------------------------------------------
// Block prologue: registry table and hot slots into shared memory, the
// warp's queue after them, the warp's log region.
template <bool kSmem, bool kHot, bool kHosts>
__device__ __forceinline__ void k2_prologue(const uint32_t* __restrict__ gt, uint32_t table_words,
                                            const DevLog& L, const DevHot& hot, const DevPartials& P,
                                            HotSmem& h, WarpQueue& wq) {
    load_table_slots<kSmem, kHot>(gt, table_words, hot);
    const uint32_t smem_words = kSmem ? table_words : 0u;
    if constexpr (kHot) {
        h = hot_smem(smem_words);
        hot_init(h, hot, P);
    }
    const uint32_t warp = threadIdx.x >> 5;
    uint4* queues = reinterpret_cast<uint4*>(g_smem + smem_words + (kHot ? kHotBytes / 4 : 0u));
    wq.q = queues + warp * kQueue;
    wq.qh = kHosts ? reinterpret_cast<uint32_t*>(queues + (blockDim.x >> 5) * kQueue) + warp * kQueue : nullptr;
    wq.n = 0;
    wq.pos = 0;
    const size_t region = static_cast<size_t>(blockIdx.x) * (blockDim.x >> 5) + warp;
    wq.log = L.entries + region * L.warp_cap;
    wq.logb = L.buckets ? L.buckets + region * L.warp_cap : nullptr;
    wq.region_off = region * L.warp_cap;
    __syncthreads();
}

template <bool kSmem, bool kHot, bool kHosts>
__device__ __forceinline__ void k2_epilogue(Ctr& t, WarpQueue& wq, uint32_t lane,
                                            const uint32_t* __restrict__ gt, const DevParams& p,
                                            const DevPartials& P, const HotSmem& h,
                                            const DevHot& hot, const DevLog& L) {
    drain_full<kSmem, kHot, kHosts>(wq, lane, gt, p, P, h, t, L);
    drain_rest<kSmem, kHot, kHosts>(wq, lane, gt, p, P, h, t, L);
    if (lane == 0) L.counts[static_cast<size_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5)] = wq.pos;
    // Zero the region's entries up to the next multiple of 4: the log
    // readers load whole 16-byte vectors (and ignore entries past the count).
    const uint32_t i = wq.pos + lane;
    if (lane < ((4u - (wq.pos & 3u)) & 3u)) {
        wq.log[i] = 0;
        if (wq.logb) wq.logb[i] = 0;
        if constexpr (kHosts) {
            const size_t j = wq.region_off + i;
            L.hosts[j] = 0;
            L.octs[j] = 0;
            L.durs[j] = 1; // never read (past the count); a valid duration all the same
        }
    }
    flush_tallies(t, P.sums + static_cast<size_t>(P.n_sites) * 4);
    if constexpr (kHot) {
        __syncthreads();
        hot_flush(h, hot, P);
    }
}

// One 64-record tile in registers: two records per lane (x and y).
struct TileRegs {
    uint2 s, d, k, o;     // src, dst, d_pkts, d_octets of (x, y)
    ulonglong2 ts, te;    // start_ms, end_ms of (x, y)
};

// Streaming loads that may allocate in L1: the 64-byte FlowRecord rows are
// read with two loads into their first 32-byte sector (src/dst at 0,
// pkts/octets at 16) and one into the second (start/end at 48), so the
// second load of a sector must hit L1 rather than go back to L2.
__device__ __forceinline__ uint2 ld_rec_u2(const void* p, uint64_t pol) {
    uint2 r;
    asm volatile("ld.global.nc.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;" : "=r"(r.x), "=r"(r.y) : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ uint4 ld_rec_u4(const void* p, uint64_t pol) {
    uint4 r;
    asm volatile("ld.global.nc.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ ulonglong2 ld_rec_u64x2(const void* p, uint64_t pol) {
    ulonglong2 r;
    asm volatile("ld.global.nc.L2::cache_hint.v2.u64 {%0,%1}, [%2], %3;" : "=l"(r.x), "=l"(r.y) : "l"(p), "l"(pol));
    return r;
}

// FLOWARC1 entries (layout 4) are only 4-byte aligned and big-endian: the
// tile keeps the 8 raw words of each of its two records and swaps them only
// when the tile is processed, so the loads stay in flight a whole round.
struct TileRaw4 {
    uint32_t x[8], y[8]; // be64 start, be64 end, src, dst, pkts, octets
};
template <int kLayout>
struct TileOf {
    using type = TileRegs;
};
template <>
struct TileOf<4> {
    using type = TileRaw4;
};

__device__ __forceinline__ uint64_t be64(uint32_t hi_word, uint32_t lo_word) {
    return static_cast<uint64_t>(__byte_perm(hi_word, 0, 0x0123)) << 32 | __byte_perm(lo_word, 0, 0x0123);
}

template <int kLayout>
__device__ __forceinline__ TileRegs unpack_tile(const typename TileOf<kLayout>::type& t) {
    if constexpr (kLayout == 4) {
        TileRegs r;
        r.ts = make_ulonglong2(be64(t.x[0], t.x[1]), be64(t.y[0], t.y[1]));
        r.te = make_ulonglong2(be64(t.x[2], t.x[3]), be64(t.y[2], t.y[3]));
        r.s = make_uint2(__byte_perm(t.x[4], 0, 0x0123), __byte_perm(t.y[4], 0, 0x0123));
        r.d = make_uint2(__byte_perm(t.x[5], 0, 0x0123), __byte_perm(t.y[5], 0, 0x0123));
        r.k = make_uint2(__byte_perm(t.x[6], 0, 0x0123), __byte_perm(t.y[6], 0, 0x0123));
        r.o = make_uint2(__byte_perm(t.x[7], 0, 0x0123), __byte_perm(t.y[7], 0, 0x0123));
        return r;
    } else {
        return t;
    }
}

// Tile loads. kLayout 0 (aligned SoA): lane takes records 2*lane, 2*lane+1
// of the tile (one LDG.64 per u32 column, one LDG.128 per u64 column,
// non-allocating). kLayout 2 (16-byte aligned AoS, the reference's 64-byte
// FlowRecord rows): lane takes records lane and 32+lane, three vector loads
// each (src/dst, pkts/octets, start/end).
template <int kLayout>
__device__ __forceinline__ void load_tile(const DevBatch& b, uint32_t tile, uint32_t lane, uint64_t pol,
                                          typename TileOf<kLayout>::type& t) {
    if constexpr (kLayout == 4) {
        // entry words at 0,4 (start) 8,12 (end) 16 (src) 20 (dst) 32 (pkts)
        // 36 (octets) of the 64-byte entry (flow_store.cpp:158-162, netflow.cpp:52-75)
        if ((reinterpret_cast<uintptr_t>(b.rec) & 15u) == 4u) {
            // The usual case (a 16-byte-aligned archive: entries at 20 + 64*i):
            // the 16-byte vectors at entry - 4, + 12, + 28 hold entry words
            // (-1, 0, 1, 2), (3, 4, 5, 6), (7, 8, 9, 10) -- three LDG.128 per
            // record instead of eight LDG.32 (the -4 of entry 0 is the header).
            const uint4* vx = reinterpret_cast<const uint4*>(static_cast<const unsigned char*>(b.rec) - 4 +
                                                             (static_cast<size_t>(tile) * 64u + lane) * 64u);
            const uint4* vy = vx + 32u * 4u;
            const uint4 a0 = ld_rec_u4(vx, pol), a1 = ld_rec_u4(vx + 1, pol), a2 = ld_rec_u4(vx + 2, pol);
            const uint4 b0 = ld_rec_u4(vy, pol), b1 = ld_rec_u4(vy + 1, pol), b2 = ld_rec_u4(vy + 2, pol);
            t.x[0] = a0.y, t.x[1] = a0.z, t.x[2] = a0.w, t.x[3] = a1.x;
            t.x[4] = a1.y, t.x[5] = a1.z, t.x[6] = a2.y, t.x[7] = a2.z;
            t.y[0] = b0.y, t.y[1] = b0.z, t.y[2] = b0.w, t.y[3] = b1.x;
            t.y[4] = b1.y, t.y[5] = b1.z, t.y[6] = b2.y, t.y[7] = b2.z;
        } else {
            const uint32_t* wx = reinterpret_cast<const uint32_t*>(static_cast<const unsigned char*>(b.rec) +
                                                                    (static_cast<size_t>(tile) * 64u + lane) * 64u);
            const uint32_t* wy = wx + 32u * 16u;
            constexpr int kWord[8] = {0, 1, 2, 3, 4, 5, 8, 9};
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                t.x[q] = __ldg(wx + kWord[q]);
                t.y[q] = __ldg(wy + kWord[q]);
            }
        }
    } else if constexpr (kLayout == 5) {
        // compacted SoA: the duration column replaces start/end (ts = 0, te = dur)
        const DevSoA& c = b.soa;
        const uint32_t g = tile * 32u + lane;
        t.s = ld_stream_u2(reinterpret_cast<const uint2*>(c.src) + g, pol);
        t.d = ld_stream_u2(reinterpret_cast<const uint2*>(c.dst) + g, pol);
        t.k = ld_stream_u2(reinterpret_cast<const uint2*>(c.pkts) + g, pol);
        t.o = ld_stream_u2(reinterpret_cast<const uint2*>(c.octets) + g, pol);
        const uint2 du = ld_stream_u2(reinterpret_cast<const uint2*>(c.dur32) + g, pol);
        t.ts = make_ulonglong2(0ull, 0ull);
        t.te = make_ulonglong2(du.x, du.y);
    } else if constexpr (kLayout == 0) {
        const DevSoA& c = b.soa;
        const uint32_t g = tile * 32u + lane;
        t.s = ld_stream_u2(reinterpret_cast<const uint2*>(c.src) + g, pol);
        t.d = ld_stream_u2(reinterpret_cast<const uint2*>(c.dst) + g, pol);
        t.k = ld_stream_u2(reinterpret_cast<const uint2*>(c.pkts) + g, pol);
        t.o = ld_stream_u2(reinterpret_cast<const uint2*>(c.octets) + g, pol);
        t.ts = ld_stream_u64x2(reinterpret_cast<const ulonglong2*>(c.start) + g, pol);
        t.te = ld_stream_u64x2(reinterpret_cast<const ulonglong2*>(c.end) + g, pol);
    } else {
        const unsigned char* rx = static_cast<const unsigned char*>(b.rec) + (static_cast<size_t>(tile) * 64u + lane) * 64u;
        const unsigned char* ry = rx + 32u * 64u;
        const uint2 ax = ld_rec_u2(rx, pol), ay = ld_rec_u2(ry, pol);
        const uint2 cx = ld_rec_u2(rx + 16, pol), cy = ld_rec_u2(ry + 16, pol);
        const ulonglong2 ex = ld_rec_u64x2(rx + 48, pol), ey = ld_rec_u64x2(ry + 48, pol);
        t.s = make_uint2(ax.x, ay.x);
        t.d = make_uint2(ax.y, ay.y);
        t.k = make_uint2(cx.x, cy.x);
        t.o = make_uint2(cx.y, cy.y);
        t.ts = make_ulonglong2(ex.x, ey.x);
        t.te = make_ulonglong2(ex.y, ey.y);
    }
}

// Main variants: aligned SoA columns (k2_soa) or aligned AoS rows (k2_aos),
// n < 2^32. Persistent: one 768-thread CTA per SM owns the contiguous
// 64-record tiles [b*T/G, (b+1)*T/G) and walks them in rounds of kWarps
// tiles (warp w takes tile t0 + r*kWarps + w), two records per lane per tile
// (load_tile), software-pipelined: the next round's loads are in flight
// while this one is classified. Every kEpochRounds rounds the CTA meets at a
// barrier and normalizes the hot limbs (hot_normalize). The last CTA also
// takes the < 64-record remainder through the scalar path.
template <int kLayout, bool kSmem, bool kHot, int kMode>
__device__ __forceinline__ void k2_tiles(const DevBatch& b, const uint32_t* __restrict__ gt, uint32_t table_words,
                                         const DevParams& p, const DevPartials& P, const DevHot& hot,
                                         const DevLog& L) {
    constexpr bool kWin = kMode & kModeWindow, kHosts = kMode & kModeHosts;
    HotSmem h{};
    WarpQueue wq;
    k2_prologue<kSmem, kHot, kHosts>(gt, table_words, L, hot, P, h, wq);
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t warp = threadIdx.x >> 5;
    const uint64_t tiles = b.n >> 6;
    const uint32_t t0 = static_cast<uint32_t>(tiles * blockIdx.x / gridDim.x);
    const uint32_t t_end = static_cast<uint32_t>(tiles * (blockIdx.x + 1) / gridDim.x);
    const uint32_t rounds = (t_end - t0 + kWarps - 1) / kWarps; // CTA-uniform
    Ctr t;
    const uint64_t pol = evict_first_policy();
    uint32_t tile = t0 + warp;
    typename TileOf<kLayout>::type raw;
    if (tile < t_end) load_tile<kLayout>(b, tile, lane, pol, raw);
    for (uint32_t r = 0; r < rounds; ++r) {
        const uint32_t next = tile + kWarps;
        typename TileOf<kLayout>::type nx;
        if (next < t_end) load_tile<kLayout>(b, next, lane, pol, nx);
        if (tile < t_end) {
            const TileRegs cur = unpack_tile<kLayout>(raw);
            const uint64_t dx = cur.te.x - cur.ts.x, dy = cur.te.y - cur.ts.y;
            uint32_t hx, hy;
            const uint32_t cx = stage_a<kSmem>(cur.s.x, cur.d.x, cur.k.x, cur.o.x, dx, p, gt, t, hx,
                                               window_in<kWin>(cur.te.x, p));
            const uint32_t cy = stage_a<kSmem>(cur.s.y, cur.d.y, cur.k.y, cur.o.y, dy, p, gt, t, hy,
                                               window_in<kWin>(cur.te.y, p));
            push<kHosts>(cx, cur.o.x, dx, wq, lane, hx);
            push<kHosts>(cy, cur.o.y, dy, wq, lane, hy);
            drain_full<kSmem, kHot, kHosts>(wq, lane, gt, p, P, h, t, L);
        }
        raw = nx;
        tile = next;
        if constexpr (kHot) {
            if ((r + 1) % kEpochRounds == 0 && r + 1 < rounds) {
                __syncthreads();
                hot_normalize(h, hot, P);
                __syncthreads();
            }
        }
    }
    if (blockIdx.x == gridDim.x - 1 && warp == 0)
        run_scalar<kLayout == 0 ? 1 : kLayout, kSmem, kHot, kMode>(b, tiles << 6, b.n, 32, lane, gt, p, P, h, t, wq,
                                                                  L);
    k2_epilogue<kSmem, kHot, kHosts>(t, wq, lane, gt, p, P, h, hot, L);
}

template <bool kSmem, bool kHot, int kMode>
__global__ void __launch_bounds__(kK2Block, 1) k2_soa(DevBatch b, const uint32_t* __restrict__ gt,
                                                    uint32_t table_words, DevParams p,
                                                    DevPartials P, DevHot hot, DevLog L) {
    k2_tiles<0, kSmem, kHot, kMode>(b, gt, table_words, p, P, hot, L);
}

template <bool kSmem, bool kHot, int kMode>
__global__ void __launch_bounds__(kK2Block, 1) k2_aos(DevBatch b, const uint32_t* __restrict__ gt,
                                                    uint32_t table_words, DevParams p,
                                                    DevPartials P, DevHot hot, DevLog L) {
    k2_tiles<2, kSmem, kHot, kMode>(b, gt, table_words, p, P, hot, L);
}

// Loader-compacted SoA (u32 durations in place of start/end).
template <bool kSmem, bool kHot, int kMode>
__global__ void __launch_bounds__(kK2Block, 1) k2_dur(DevBatch b, const uint32_t* __restrict__ gt,
                                                    uint32_t table_words, DevParams p,
                                                    DevPartials P, DevHot hot, DevLog L) {
    k2_tiles<5, kSmem, kHot, kMode>(b, gt, table_words, p, P, hot, L);
}

// FLOWARC1 entries read in place (the archive's big-endian rows).
template <bool kSmem, bool kHot, int kMode>
__global__ void __launch_bounds__(kK2Block, 1) k2_arc(DevBatch b, const uint32_t* __restrict__ gt,
                                                    uint32_t table_words, DevParams p,
                                                    DevPartials P, DevHot hot, DevLog L) {
    k2_tiles<4, kSmem, kHot, kMode>(b, gt, table_words, p, P, hot, L);
}

// Other layouts: unaligned SoA (1), AoS 64-byte rows with vector (2) or
// scalar (3) loads, FLOWARC1 archive entries read in place (4). CTA b owns records [b*n/G, (b+1)*n/G) (at most
// kCtaRecords), one record per lane per round.
template <int kLayout, bool kSmem, bool kHot, int kMode>
__global__ void __launch_bounds__(kK2Block, 1) k2_gen(DevBatch b, const uint32_t* __restrict__ gt,
                                                    uint32_t table_words, DevParams p,
                                                    DevPartials P, DevHot hot, DevLog L) {
    constexpr bool kHosts = kMode & kModeHosts;
    HotSmem h{};
    WarpQueue wq;
    k2_prologue<kSmem, kHot, kHosts>(gt, table_words, L, hot, P, h, wq);
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t r0 = b.n * blockIdx.x / gridDim.x, r1 = b.n * (blockIdx.x + 1) / gridDim.x;
    Ctr t;
    run_scalar<kLayout, kSmem, kHot, kMode>(b, r0 + (threadIdx.x >> 5) * 32, r1, kK2Block, lane, gt, p, P,
                                            h, t, wq, L);
    k2_epilogue<kSmem, kHot, kHosts>(t, wq, lane, gt, p, P, h, hot, L);
}

// ---- K1: hot-site plan ------------------------------------------------------
// Each block classifies one contiguous chunk of the batch and counts Forward
// flows per site; their rates also seed the sites' min/max (see hot_init).
template <bool kSmem>
__global__ void __launch_bounds__(kK2Block) k_sample(DevBatch b, const uint32_t* __restrict__ gt,
                                                      uint32_t table_words, DevParams p,
                                                      uint64_t chunk_stride, uint32_t chunk_len,
                                                      uint32_t* __restrict__ cnt,
                                                      unsigned long long* __restrict__ mn,
                                                      unsigned long long* __restrict__ mx) {
    load_table<kSmem>(gt, table_words);
    if constexpr (kSmem) __syncthreads();
    // blockIdx.y picks the chunk; blockIdx.x * blockDim.x the first record
    // within it: one record per thread, so the whole sample is one wave of
    // independent lookup chains.
    const uint64_t base = static_cast<uint64_t>(blockIdx.y) * chunk_stride;
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < chunk_len; j += gridDim.x * blockDim.x) {
        const uint64_t i = base + j;
        uint32_t src, dst, pkts, oct;
        uint64_t dur, end;
        if (b.archive) load_record<4>(b, i, src, dst, pkts, oct, dur, end);
        else if (b.aos) load_record<3>(b, i, src, dst, pkts, oct, dur, end);
        else if (b.soa.dur32) load_record<5>(b, i, src, dst, pkts, oct, dur, end);
        else load_record<1>(b, i, src, dst, pkts, oct, dur, end);
        if (static_cast<uint64_t>(oct) < p.ack_plus1 * pkts || pkts < p.min_packets1 ||
            dur < static_cast<uint64_t>(p.min_duration1) || (p.windowed && !(end >= p.win_lo && end < p.win_hi)))
            continue;
        const uint32_t v = site_of_full<kSmem>(gt, src, dst);
        if (v == kNone) continue;
        const uint32_t site = v & p.site_mask;
        atomicAdd(cnt + site, 1u);
        // The sampled Forward flow's rate (flow_rate, rate_engine.cpp:88-94)
        // into its site's min/max now; K2 reduces the same flow again, which
        // min/max absorb. A read filters the reductions (a stale read only
        // costs an extra one).
        const unsigned long long rb = static_cast<unsigned long long>(
            __double_as_longlong(__ddiv_rn(8000.0 * static_cast<double>(oct), __ull2double_rn(dur))));
        if (rb < __ldcg(mn + site)) red_min(mn + site, rb);
        if (rb > __ldcg(mx + site)) red_max(mx + site, rb);
    }
}

// One block: the sites with the most sampled Forward flows (at least `thr`)
// get slots 1..kHotSlots. A 4096-bin histogram of the counts gives the
// smallest count threshold whose sites fit the slots; the numbering itself
// does not affect results. Resets the counts for the next call.
constexpr int kSelectBlock = 1024;
constexpr uint32_t kCountBins = 4096;
__global__ void __launch_bounds__(kSelectBlock) k_hot_select(uint32_t* __restrict__ cnt, uint32_t n_sites,
                                                             uint32_t thr, uint32_t* __restrict__ site_slot,
                                                             uint32_t* __restrict__ hot_site) {
    __shared__ uint32_t bins[kCountBins];
    __shared__ uint32_t part[kSelectBlock];
    __shared__ uint32_t cut, cut_a, next, next_a;
    __shared__ unsigned long long top; // count << 32 | site of the most sampled site
    for (uint32_t i = threadIdx.x; i < kCountBins; i += blockDim.x) bins[i] = 0;
    if (threadIdx.x == 0) {
        next = 0;
        top = 0;
    }
    __syncthreads();
    unsigned long long best = 0;
    for (uint32_t s4 = threadIdx.x * 4; s4 < n_sites; s4 += blockDim.x * 4) { // 16-byte loads
        const uint4 c4 = *reinterpret_cast<const uint4*>(cnt + s4);
        const uint32_t cs[4] = {c4.x, c4.y, c4.z, c4.w};
#pragma unroll
        for (uint32_t q = 0; q < 4; ++q)
            if (s4 + q < n_sites && cs[q] >= thr) {
                atomicAdd(&bins[min(cs[q], kCountBins - 1)], 1u);
                best = max(best, static_cast<unsigned long long>(cs[q]) << 32 | (s4 + q));
            }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(0xFFFFFFFFu, best, o));
    if ((threadIdx.x & 31u) == 0 && best) atomicMax(&top, best);
    __syncthreads();
    // Suffix sums over the bins: thread i owns bins [4i, 4i+4).
    const uint32_t i0 = threadIdx.x * (kCountBins / kSelectBlock);
    uint32_t own = 0;
    for (uint32_t k = 0; k < kCountBins / kSelectBlock; ++k) own += bins[i0 + k];
    // Inclusive suffix scan of `own` over the threads: within each warp by
    // shuffles, then over the 32 warp totals by warp 0.
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    uint32_t suf = own;
#pragma unroll
    for (uint32_t o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_down_sync(0xFFFFFFFFu, suf, o);
        if (lane + o < 32) suf += y;
    }
    __shared__ uint32_t wsum[kSelectBlock / 32];
    if (lane == 0) wsum[warp] = suf;
    __syncthreads();
    if (warp == 0) {
        uint32_t v = wsum[lane], t = v;
#pragma unroll
        for (uint32_t o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_down_sync(0xFFFFFFFFu, t, o);
            if (lane + o < 32) t += y;
        }
        wsum[lane] = t - v; // the warps after this one
    }
    __syncthreads();
    part[threadIdx.x] = suf + wsum[warp];
    if (threadIdx.x == 0) {
        cut = 0xFFFFFFFFu;
        cut_a = 0xFFFFFFFFu;
        next_a = 0;
    }
    __syncthreads();
    {
        // cut: the lowest bin b with suffix(b) <= kHotSlots; cut_a the same
        // for the kCoarseSlots slots that also keep coarse counts in smem.
        // Warp-reduced first: one shared atomic per warp, not per bin.
        uint32_t suffix = threadIdx.x + 1 < kSelectBlock ? part[threadIdx.x + 1] : 0u;
        uint32_t lc = 0xFFFFFFFFu, lca = 0xFFFFFFFFu;
        for (int k = kCountBins / kSelectBlock - 1; k >= 0; --k) {
            suffix += bins[i0 + k];
            if (suffix <= kHotSlots - (kTopReplicas - 1)) lc = i0 + k;
            if (suffix <= kCoarseSlots - (kTopReplicas - 1)) lca = i0 + k;
        }
        lc = __reduce_min_sync(0xFFFFFFFFu, lc);
        lca = __reduce_min_sync(0xFFFFFFFFu, lca);
        if (lane == 0) {
            if (lc != 0xFFFFFFFFu) atomicMin(&cut, lc);
            if (lca != 0xFFFFFFFFu) atomicMin(&cut_a, lca);
        }
    }
    __syncthreads();
    const uint32_t t = max(max(cut, thr), 1u);
    const uint32_t ta = max(cut_a, t);
    // Slots 1..kTopReplicas: the most sampled site (~10% of a Zipf batch's
    // Forward flows), one replica per lane & (kTopReplicas - 1) in K2, so its
    // flows in one drain do not all add to the same shared-memory words.
    // Reserved (unassigned) when no site is hot.
    const uint32_t top_cnt = static_cast<uint32_t>(top >> 32);
    const uint32_t top_site = top_cnt >= t ? static_cast<uint32_t>(top) : 0xFFFFFFFFu;
    // Slots 1..n_a: the top sites (count >= ta); the rest follow them.
    uint32_t n_a = 0;
    for (uint32_t b = threadIdx.x; b < kCountBins; b += blockDim.x)
        if (b >= ta) n_a += bins[b];
    n_a = __reduce_add_sync(0xFFFFFFFFu, n_a);
    if ((threadIdx.x & 31u) == 0 && n_a) atomicAdd(&next_a, n_a);
    __syncthreads();
    const uint32_t base_b = next_a - (top_site != 0xFFFFFFFFu && top_cnt >= ta ? 1u : 0u) + kTopReplicas;
    if (threadIdx.x < kTopReplicas && top_site != 0xFFFFFFFFu) hot_site[1 + threadIdx.x] = top_site;
    __syncthreads();
    if (threadIdx.x == 0) next_a = 0;
    __syncthreads();
    // Slot numbers by warp-aggregated allocation (ballot + one shared
    // atomic per warp and class), so the hot sites never serialise on the
    // two counters.
    const uint32_t lt = (1u << lane) - 1u;
    for (uint32_t s0 = warp * 128; s0 < n_sites; s0 += blockDim.x * 4) { // warp-uniform trip count
        const uint32_t s4 = s0 + lane * 4;
        uint4 c4 = make_uint4(0, 0, 0, 0);
        if (s4 < n_sites) c4 = *reinterpret_cast<const uint4*>(cnt + s4);
        const uint32_t cs[4] = {c4.x, c4.y, c4.z, c4.w};
#pragma unroll
        for (uint32_t q = 0; q < 4; ++q) {
            const uint32_t s = s4 + q;
            const bool in = s < n_sites;
            const bool is_top = s == top_site;
            const bool a = in && !is_top && cs[q] >= ta, bclass = in && !is_top && !a && cs[q] >= t;
            const unsigned ma = __ballot_sync(0xFFFFFFFFu, a), mb = __ballot_sync(0xFFFFFFFFu, bclass);
            uint32_t fa = 0, fb = 0;
            if (lane == 0) {
                if (ma) fa = atomicAdd(&next_a, __popc(ma));
                if (mb) fb = atomicAdd(&next, __popc(mb));
            }
            fa = __shfl_sync(0xFFFFFFFFu, fa, 0);
            fb = __shfl_sync(0xFFFFFFFFu, fb, 0);
            if (!in) continue;
            cnt[s] = 0;
            uint32_t slot = 0;
            if (a) slot = kTopReplicas + fa + __popc(ma & lt) + 1;
            else if (bclass) slot = base_b + fb + __popc(mb & lt) + 1;
            if (slot) hot_site[slot] = s;
            if (is_top) slot = 1;
            site_slot[s] = slot;
        }
    }
}

// Rewrites the slot bits of every site value in the table (nodes flagged
// uniform and leaf entries).
__global__ void k_table_slots(uint32_t* __restrict__ words, uint32_t node_begin,
                              uint32_t leaf_begin, uint32_t end,
                              const uint32_t* __restrict__ site_slot) {
    const uint32_t i0 = blockIdx.x * blockDim.x + threadIdx.x;
    for (uint32_t i = node_begin + i0; i < end; i += gridDim.x * blockDim.x) {
        const uint32_t w = words[i];
        if (i < leaf_begin) {
            if (w & 0x80000000u) {
                const uint32_t site = w & 0xFFFFFu;
                words[i] = 0x80000000u | site_slot[site] << 20 | site;
            }
        } else if (w != kNone) {
            const uint32_t site = w & 0xFFFFFu;
            words[i] = site_slot[site] << 20 | site;
        }
    }
}

// ---- per-record classification --------------------------------------------
template <bool kSmem>
__global__ void __launch_bounds__(kK2Block) k_classify(DevSoA b, const uint32_t* __restrict__ gt,
                                                        uint32_t table_words, DevParams p,
                                                        uint32_t* __restrict__ out) {
    load_table<kSmem>(gt, table_words);
    if constexpr (kSmem) __syncthreads();
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < b.n;
         i += stride) {
        const uint32_t pkts = b.pkts[i], oct = b.octets[i];
        const uint64_t dur = b.end[i] - b.start[i];
        uint32_t cls, site = 0x3FFFFFFFu;
        if (pkts == 0) cls = GNM_ADMINISTRATIVE;
        else if (static_cast<uint64_t>(oct) < p.ack_plus1 * pkts) cls = GNM_PURE_ACK;
        else if (pkts < p.min_packets || dur < p.min_duration_ms || dur == 0) cls = GNM_ADMINISTRATIVE;
        else {
            uint32_t v = lookup<kSmem>(gt, b.src[i]);
            if (v == kNone) v = lookup<kSmem>(gt, b.dst[i]);
            if (v == kNone) cls = GNM_UNMATCHED;
            else {
                cls = GNM_FORWARD;
                site = (v & p.site_mask) & 0x3FFFFFFFu;
            }
        }
        out[i] = cls << 30 | site;
    }
}

// ---- K3: per-site synthesis (two-round exact median) ---------------------------
// K3a, thread per site (coalesced over the sb-major coarse array): the flow
// count and the super-bucket holding the lower median, i.e. the first
// super-bucket whose cumulative count reaches ceil(count/2)
// (RateHistogram::median_bps, rate_engine.cpp:42-58), and the median's rank
// inside it. The 157 counts are loaded in unrolled batches (independent
// loads in flight) and kept in registers between the two passes.
__global__ void __launch_bounds__(128) k3a_median_sb(DevPartials P) {
    // Four lanes per site, each over ~40 of the 157 super-buckets (a site's
    // counts are n_sites apart; neighbouring sites' are adjacent, so each
    // load instruction stays coalesced across quads).
    constexpr uint32_t kPart = (kCoarse + 3) / 4; // 40
    const uint32_t n = P.n_sites;
    const uint32_t lane = threadIdx.x & 31u, part = lane & 3u;
    const uint32_t stride = (gridDim.x * blockDim.x) >> 2;
    for (uint32_t site0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 2;; site0 += stride) {
        const bool in = site0 < n;
        if (!__any_sync(0xFFFFFFFFu, in)) break; // warp-uniform: the quads shuffle below
        const uint32_t site = in ? site0 : 0u;
        const uint32_t sb0 = part * kPart;
        const unsigned int* col = P.coarse + site;
        uint32_t v[kPart];
        uint64_t c = 0;
#pragma unroll
        for (uint32_t i = 0; i < kPart; ++i) {
            v[i] = (in && sb0 + i < kCoarse) ? __ldcg(col + static_cast<size_t>(sb0 + i) * n) : 0u;
            c += v[i];
        }
        uint64_t pre = __shfl_up_sync(0xFFFFFFFFu, c, 1); // exclusive prefix within the quad
        pre = part >= 1 ? pre : 0;
        uint64_t p2 = __shfl_up_sync(0xFFFFFFFFu, pre + c, 2);
        pre += part >= 2 ? p2 : 0;
        const uint64_t tot = __shfl_sync(0xFFFFFFFFu, pre + c, (lane & ~3u) + 3u);
        const uint64_t target = (tot + 1) / 2;
        unsigned long long found = 0; // (msb + 1) << 32 | rank, from the part that holds the median
        if (tot && pre < target && pre + c >= target) {
            uint64_t cum = pre;
#pragma unroll
            for (uint32_t i = 0; i < kPart; ++i) {
                if (!found && cum + v[i] >= target) found = static_cast<unsigned long long>(sb0 + i + 1) << 32 | (target - cum);
                cum += v[i];
            }
        }
        found = max(found, __shfl_xor_sync(0xFFFFFFFFu, found, 1));
        found = max(found, __shfl_xor_sync(0xFFFFFFFFu, found, 2));
        if (in && part == 0) {
            const uint32_t msb = found ? static_cast<uint32_t>(found >> 32) - 1u : kLogSkip;
            const uint32_t rank = static_cast<uint32_t>(found);
            // Heavy sites (>= kHeavyMin flows) get one of kHeavy shared-memory
            // fine rows in K2b: their median super-bucket draws thousands of
            // same-address reductions otherwise.
            uint32_t hidx = kHeavyNone;
            if (tot >= kHeavyMin) {
                const uint32_t k = atomicAdd(P.heavy_next, 1u);
                if (k < kHeavy) {
                    hidx = k;
                    P.heavy_next[1 + k] = site; // heavy row -> site, for K2b's flush
                }
            }
            P.msb[site] = msb | hidx << 8;
            P.map16[site] = static_cast<unsigned short>((msb & 0xFFu) | (hidx == kHeavyNone ? 0xFF00u : hidx << 8));
            P.mrank[site] = rank;
            P.cnt[site] = tot;
        }
    }
}

// K2b: one launch's log, the entries that fall into their site's median
// super-bucket count into its 64 fine buckets -- in shared memory for the
// heavy sites (flushed once per CTA, persistent grid), with L2 reductions
// for the rest. Work item = (region, chunk of kLogChunk entries), many
// warps per region; each lane reads 4 entries per LDG.128 (region bases are
// multiples of 4 entries), 4 of those in flight. kMap: each site's
// (median super-bucket | heavy row << 8) in shared memory (small
// registries), else read from L2/L1.
constexpr uint32_t kMapSites = 12288; // 24 KB of static shared memory
// Three 512-thread CTAs per SM with four 16-byte log vectors in flight per
// lane (40 registers) measured ahead of two CTAs with eight (finalize 0.082
// -> 0.080 ms, profiles/round2/ab_k2b_occupancy.txt).
#ifndef GNM_K2B_CTAS
#define GNM_K2B_CTAS 3
#endif
#ifndef GNM_K2B_V
#define GNM_K2B_V 4
#endif
template <bool kMap, bool kWide>
__global__ void __launch_bounds__(512, GNM_K2B_CTAS) k2b_fine(DevPartials P, DevLog L) {
    __shared__ uint32_t hf[kHeavy * kFineW];
    __shared__ uint4 map4[kMap ? kMapSites / 8 : 1];
    const uint16_t* map = reinterpret_cast<const uint16_t*>(map4);
    for (uint32_t i = threadIdx.x; i < kHeavy * kFineW; i += blockDim.x) hf[i] = 0;
    if constexpr (kMap) // K3a's packed per-site map, 8 sites per 16-byte load
        for (uint32_t i = threadIdx.x; i < (P.n_sites + 7) / 8; i += blockDim.x)
            map4[i] = __ldg(reinterpret_cast<const uint4*>(P.map16) + i);
    __syncthreads();
    const uint32_t hf_base = static_cast<uint32_t>(__cvta_generic_to_shared(hf));
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    const uint32_t chunks = (L.warp_cap + kLogChunk - 1) / kLogChunk;
    const uint32_t items = L.regions * chunks;
    constexpr uint32_t kV = kWide ? 4 : GNM_K2B_V; // LDG.128 per lane in flight
    // One log entry: skip unless in its site's median super-bucket; heavy
    // sites count in shared memory, the rest in L2.
    auto one = [&](uint32_t site, uint32_t bk) {
        uint32_t msb, hh;
        if constexpr (kMap) {
            const uint32_t m = map[site];
            msb = m & 0xFFu;
            hh = m >> 8;
        } else {
            const uint32_t m = __ldg(P.msb + site);
            msb = m & 0xFFu;
            hh = (m >> 8) == kHeavyNone ? 0xFFu : m >> 8;
        }
        // branch-free: both addresses computed, the two reductions predicated
        const uint32_t hit = (bk >> 6) == msb;
        const uint32_t heavy = hit & (hh != 0xFFu), light = hit & (hh == 0xFFu);
        const uint32_t sa = hf_base + ((hh & 0xFFu) * kFineW + (bk & 63u)) * 4;
        unsigned int* ga = P.fine + static_cast<size_t>(site) * kFineW + (bk & 63u);
        asm volatile("{\n\t.reg .pred ph, pl;\n\tsetp.ne.u32 ph, %2, 0;\n\tsetp.ne.u32 pl, %3, 0;\n\t"
                     "@ph red.shared.add.u32 [%0], 1;\n\t@pl red.relaxed.gpu.global.add.u32 [%1], 1;\n\t}"
                     ::"r"(sa), "l"(ga), "r"(heavy), "r"(light) : "memory");
    };
    for (uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < items; w += nwarps) {
        const uint32_t r = w / chunks;
        const uint32_t c0 = (w % chunks) * kLogChunk;
        const uint32_t cnt = min(L.counts[r], c0 + kLogChunk);
        const unsigned int* e = L.entries + static_cast<size_t>(r) * L.warp_cap;
        const unsigned int* eb = kWide ? L.buckets + static_cast<size_t>(r) * L.warp_cap : nullptr;
        for (uint32_t base = c0; base < cnt; base += 32 * 4 * kV) {
            uint4 x[kV], bb[kWide ? kV : 1];
#pragma unroll
            for (uint32_t u = 0; u < kV; ++u) {
                const uint32_t i = base + (u * 32 + lane) * 4;
                x[u] = i < cnt ? __ldcs(reinterpret_cast<const uint4*>(e + i)) : make_uint4(0, 0, 0, 0);
                if constexpr (kWide)
                    bb[u] = i < cnt ? __ldcs(reinterpret_cast<const uint4*>(eb + i)) : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
            for (uint32_t u = 0; u < kV; ++u) {
                const uint32_t i = base + (u * 32 + lane) * 4;
                const uint32_t xs[4] = {x[u].x, x[u].y, x[u].z, x[u].w};
                uint32_t bs[4] = {0, 0, 0, 0};
                if constexpr (kWide) {
                    bs[0] = bb[u].x, bs[1] = bb[u].y, bs[2] = bb[u].z, bs[3] = bb[u].w;
                }
                if (i + 4 <= cnt) { // whole vector valid: no per-entry bounds checks
#pragma unroll
                    for (uint32_t q = 0; q < 4; ++q)
                        one(kWide ? xs[q] : xs[q] >> kLogSiteShift,
                            kWide ? bs[q] : xs[q] & ((1u << kLogSiteShift) - 1u));
                } else {
#pragma unroll
                    for (uint32_t q = 0; q < 4; ++q)
                        if (i + q < cnt)
                            one(kWide ? xs[q] : xs[q] >> kLogSiteShift,
                                kWide ? bs[q] : xs[q] & ((1u << kLogSiteShift) - 1u));
                }
            }
        }
    }
    __syncthreads();
    const uint32_t n_heavy = min(*P.heavy_next, kHeavy);
    for (uint32_t i = threadIdx.x; i < n_heavy * kFineW; i += blockDim.x)
        if (hf[i]) red_add(P.fine + static_cast<size_t>(P.heavy_next[1 + i / kFineW]) * kFineW + (i % kFineW), hf[i]);
}

// K3b, thread per site: count (coarse), the exact median bucket from the
// fine counts, stats_from (rate_engine.cpp:242-253: median clamped into
// [min, max]) and the flag (monitor.cpp:22); optionally resets the sums and
// min/max (the launcher clears coarse and fine).
__global__ void __launch_bounds__(128) k3b_finalize(DevPartials P, double threshold,
                                                    gnm_site_stats* __restrict__ out,
                                                    unsigned long long* __restrict__ tallies_out,
                                                    int write_out, int reset) {
    const uint32_t n = P.n_sites;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        unsigned long long* t = P.sums + static_cast<size_t>(n) * 4;
        if (write_out)
            for (int i = 0; i < 4; ++i) tallies_out[i] = t[i];
        if (reset)
            for (int i = 0; i < 4; ++i) t[i] = 0;
    }
    for (uint32_t site = blockIdx.x * blockDim.x + threadIdx.x; site < n; site += gridDim.x * blockDim.x) {
        const uint64_t cnt = P.cnt[site];
        uint4* fine = reinterpret_cast<uint4*>(P.fine + static_cast<size_t>(site) * kFineW);
        unsigned long long* s = P.sums + static_cast<size_t>(site) * 4;
        if (write_out) {
            gnm_site_stats o = {};
            if (cnt) {
                const uint32_t msb = P.msb[site] & 0xFFu, rank = P.mrank[site];
                uint4 f[kFineW / 4];
#pragma unroll
                for (uint32_t j = 0; j < kFineW / 4; ++j) f[j] = __ldcg(fine + j);
                uint32_t cum = 0, k = kBuckets - 1;
                bool found = false;
#pragma unroll
                for (uint32_t j = 0; j < kFineW / 4; ++j) {
                    const uint32_t v[4] = {f[j].x, f[j].y, f[j].z, f[j].w};
#pragma unroll
                    for (uint32_t q = 0; q < 4; ++q) {
                        cum += v[q];
                        const bool hit = !found && cum >= rank;
                        if (hit) k = msb * kFineW + 4 * j + q;
                        found |= hit;
                    }
                }
                const double mn = __longlong_as_double(static_cast<long long>(P.mn[site]));
                const double mx = __longlong_as_double(static_cast<long long>(P.mx[site]));
                // median_bps (rate_engine.cpp:42-58), clamped (stats_from :251).
                double med = median_of_bucket(k);
                med = med < mn ? mn : (mx < med ? mx : med);
                const unsigned __int128 u = static_cast<unsigned __int128>(s[1]) +
                                            (static_cast<unsigned __int128>(s[2]) << 32) +
                                            (static_cast<unsigned __int128>(s[3]) << 64);
                o.flow_count = cnt;
                o.octets = s[0];
                o.rate_ubps_lo = static_cast<uint64_t>(u);
                o.rate_ubps_hi = static_cast<uint64_t>(u >> 64);
                o.min_bps = mn;
                o.max_bps = mx;
                o.avg_bps = avg_of(static_cast<uint64_t>(u), static_cast<uint64_t>(u >> 64), cnt);
                o.median_bps = med;
                o.below_threshold = med < threshold ? 1u : 0u; // monitor.cpp:22
            }
            out[site] = o;
        }
        if (reset) { // coarse and fine: bulk memsets after this kernel
            s[0] = s[1] = s[2] = s[3] = 0;
            P.mn[site] = kMinInitBits;
            P.mx[site] = kMaxInitBits;
        }
    }
}

// Dense [site][10001] histograms (RateHistogram::buckets_) from one launch's log.
__global__ void __launch_bounds__(256) k_hist_from_log(DevLog L, uint32_t* __restrict__ dense) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < L.regions; r += nwarps) {
        const uint32_t cnt = L.counts[r];
        const unsigned int* e = L.entries + static_cast<size_t>(r) * L.warp_cap;
        const unsigned int* eb = L.buckets ? L.buckets + static_cast<size_t>(r) * L.warp_cap : nullptr;
        for (uint32_t i = lane; i < cnt; i += 32) {
            const uint32_t x = e[i];
            if (x == kLogSkip) continue;
            const uint32_t site = eb ? x : x >> kLogSiteShift;
            const uint32_t b = eb ? eb[i] : x & ((1u << kLogSiteShift) - 1u);
            red_add(dense + static_cast<size_t>(site) * kBuckets + b, 1u);
        }
    }
}

__global__ void k_fill_u64(unsigned long long* p, size_t n, unsigned long long v) {
    for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        p[i] = v;
}

int sm_count(int device) {
    static int cached[64] = {0};
    if (device >= 0 && device < 64 && cached[device]) return cached[device];
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device);
    if (n <= 0) n = 1;
    if (device >= 0 && device < 64) cached[device] = n;
    return n;
}

template <typename K>
int occupancy(K kernel, int block, size_t smem) {
    int blocks = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, kernel, block, smem);
    return blocks > 0 ? blocks : 1;
}

template <typename K>
cudaError_t allow_smem(K kernel) {
    return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(kSmemMax));
}

template <int L, bool kS, bool kH, int kW>
constexpr auto k2_kernel() {
    if constexpr (L == 0) return k2_soa<kS, kH, kW>;
    else if constexpr (L == 2) return k2_aos<kS, kH, kW>;
    else if constexpr (L == 4) return k2_arc<kS, kH, kW>;
    else if constexpr (L == 5) return k2_dur<kS, kH, kW>;
    else return k2_gen<L, kS, kH, kW>;
}

template <int L, int kW>
cudaError_t allow_layout_w() {
    cudaError_t e;
    if ((e = allow_smem(k2_kernel<L, true, true, kW>()))) return e;
    if ((e = allow_smem(k2_kernel<L, true, false, kW>()))) return e;
    if ((e = allow_smem(k2_kernel<L, false, true, kW>()))) return e;
    return allow_smem(k2_kernel<L, false, false, kW>());
}

template <int L>
cudaError_t allow_layout() {
    cudaError_t e;
    if ((e = allow_layout_w<L, 0>())) return e;
    if ((e = allow_layout_w<L, kModeWindow>())) return e;
    if ((e = allow_layout_w<L, kModeHosts>())) return e;
    return allow_layout_w<L, kModeWindow | kModeHosts>();
}

template <int L, bool kS, bool kH, int kW>
void launch_k2_t(const LaunchCfg& cfg, const DevBatch& b, const DevTable& t, const DevParams& p,
                 const DevPartials& P, const DevHot& hot, const DevLog& log, cudaStream_t s) {
    k2_kernel<L, kS, kH, kW>()<<<cfg.grid, cfg.block, cfg.smem, s>>>(b, t.words, t.n_words, p, P, hot, log);
}

template <int L, int kW>
void launch_k2_w(const LaunchCfg& cfg, const DevBatch& b, const DevTable& t, const DevParams& p,
                 const DevPartials& P, const DevHot& hot, const DevLog& log, cudaStream_t s) {
    const bool hh = hot.n_slots > 0;
    if (cfg.table_in_smem) {
        if (hh) launch_k2_t<L, true, true, kW>(cfg, b, t, p, P, hot, log, s);
        else launch_k2_t<L, true, false, kW>(cfg, b, t, p, P, hot, log, s);
    } else {
        if (hh) launch_k2_t<L, false, true, kW>(cfg, b, t, p, P, hot, log, s);
        else launch_k2_t<L, false, false, kW>(cfg, b, t, p, P, hot, log, s);
    }
}

template <int L>
void launch_k2_l(const LaunchCfg& cfg, const DevBatch& b, const DevTable& t, const DevParams& p,
                 const DevPartials& P, const DevHot& hot, const DevLog& log, cudaStream_t s) {
    // Fused snapshot window and hosts-mode logging are compile-time modes.
    switch ((p.windowed ? kModeWindow : 0) | (log.hosts ? kModeHosts : 0)) {
    case 0: launch_k2_w<L, 0>(cfg, b, t, p, P, hot, log, s); break;
    case kModeWindow: launch_k2_w<L, kModeWindow>(cfg, b, t, p, P, hot, log, s); break;
    case kModeHosts: launch_k2_w<L, kModeHosts>(cfg, b, t, p, P, hot, log, s); break;
    default: launch_k2_w<L, kModeWindow | kModeHosts>(cfg, b, t, p, P, hot, log, s); break;
    }
}

size_t table_smem_bytes(uint32_t table_words) { return static_cast<size_t>(table_words) * 4; }

int k2_layout(const DevBatch& b) {
    if (b.archive) return 4;
    if (b.aos) return (reinterpret_cast<uintptr_t>(b.rec) & 15u) == 0 ? 2 : 3;
    const DevSoA& c = b.soa;
    if (c.dur32) return 5; // the loader's staging: 16-byte aligned columns
    const bool vec = ((reinterpret_cast<uintptr_t>(c.src) | reinterpret_cast<uintptr_t>(c.dst) |
                       reinterpret_cast<uintptr_t>(c.pkts) | reinterpret_cast<uintptr_t>(c.octets) |
                       reinterpret_cast<uintptr_t>(c.start) | reinterpret_cast<uintptr_t>(c.end)) &
                      15u) == 0;
    return vec ? 0 : 1;
}

} // namespace

cudaError_t init_kernel_attributes() {
    cudaError_t e;
    if ((e = allow_layout<0>())) return e;
    if ((e = allow_layout<1>())) return e;
    if ((e = allow_layout<2>())) return e;
    if ((e = allow_layout<3>())) return e;
    if ((e = allow_layout<4>())) return e;
    if ((e = allow_layout<5>())) return e;
    if ((e = allow_smem(k_sample<true>))) return e;
    return allow_smem(k_classify<true>);
}

LaunchCfg k2_config(int device, const DevBatch& b, uint32_t table_words, bool hot, int* occ_cache,
                    bool hosts) {
    (void)occ_cache;
    LaunchCfg c;
    const size_t tbytes = table_smem_bytes(table_words);
    const size_t qbytes = kQueueBytes + (hosts ? kWarps * kQueue * 4 : 0);
    c.block = kK2Block;
    c.table_in_smem = tbytes + qbytes <= kSmemTableMax + kQueueBytes;
    c.smem = (c.table_in_smem ? tbytes : 0) + (hot ? kHotBytes : 0) + qbytes;
    const uint64_t sms = static_cast<uint64_t>(sm_count(device));
    // At least 16 records per thread so the per-CTA table load amortises.
    const uint64_t per_block = static_cast<uint64_t>(c.block) * 16;
    const uint64_t want = (b.n + per_block - 1) / per_block;
    uint64_t grid;
    if (k2_layout(b) == 0 || k2_layout(b) == 2 || k2_layout(b) == 4 || k2_layout(b) == 5) {
        grid = std::min(sms, want); // persistent, one CTA per SM
    } else {
        // k2_gen: < 2^16 records per CTA (the hot limbs' bound); beyond one
        // wave, a whole number of waves.
        grid = (b.n + kCtaRecords - 1) / kCtaRecords;
        grid = grid <= sms ? std::max(grid, std::min(sms, want)) : (grid + sms - 1) / sms * sms;
    }
    c.grid = static_cast<int>(std::max<uint64_t>(1, grid));
    return c;
}

bool plan_hot(int device, const DevBatch& b, const DevTable& t, const DevParams& p,
              uint32_t n_sites, uint32_t* scratch, unsigned long long* mn, unsigned long long* mx,
              int k2_grid, bool force, bool table_in_smem, cudaStream_t s, uint64_t* launches,
              cudaError_t* err) {
    (void)device;
    *err = cudaSuccess;
    if (!t.packed || n_sites == 0 || b.n == 0) return false;
    // Sample 1/64 of the batch (at most GNM_K1_SAMPLE records) in 16..256 contiguous
    // chunks of about 1024 records (one CTA each).
#ifndef GNM_K1_SAMPLE
#define GNM_K1_SAMPLE 262144
#endif
    uint64_t sample = std::min<uint64_t>(GNM_K1_SAMPLE, b.n / 64);
    const uint32_t chunks = static_cast<uint32_t>(std::min<uint64_t>(256, std::max<uint64_t>(16, sample / 1024)));
    uint32_t chunk_len = static_cast<uint32_t>(sample / chunks);
    uint32_t thr;
    if (force) {
        chunk_len = static_cast<uint32_t>(std::max<uint64_t>(1, std::min<uint64_t>(4096, b.n / chunks)));
        thr = 1;
    } else {
        if (chunk_len < 256) return false;
        // Eligible: expected to see >= 2 Forward flows per K2 CTA (a slot's
        // one flush then costs no more L2 reductions than the flows would).
        const double thr_d =
            2.0 * k2_grid * static_cast<double>(chunk_len) * chunks / static_cast<double>(b.n);
        thr = static_cast<uint32_t>(std::max(2.0, thr_d));
        if (thr > chunk_len * chunks) return false;
    }
    uint32_t* cnt = scratch;
    uint32_t* site_slot = scratch + plan_slot_offset(n_sites);
    uint32_t* hot_site = scratch + plan_hot_site_offset(n_sites);
    const uint64_t stride = std::max<uint64_t>(b.n / chunks, chunk_len);
    const uint32_t nchunks = static_cast<uint32_t>(std::min<uint64_t>(chunks, b.n / chunk_len));
    // The sample is small: probe the table through L1 rather than copying
    // it into every CTA's shared memory.
    const dim3 sg((chunk_len + 255) / 256, nchunks);
    k_sample<false><<<sg, 256, 0, s>>>(b, t.words, t.n_words, p, stride, chunk_len, cnt, mn, mx);
    k_hot_select<<<1, kSelectBlock, 0, s>>>(cnt, n_sites, thr, site_slot, hot_site);
    *launches += 2;
    if (!table_in_smem) { // K2 probes the global table: write the slots into it
        const uint32_t span = t.n_words - t.node_begin;
        const uint32_t rg = std::max<uint32_t>(1, std::min<uint32_t>((span + 255) / 256, 1024));
        k_table_slots<<<rg, 256, 0, s>>>(t.words, t.node_begin, t.leaf_begin, t.n_words, site_slot);
        *launches += 1;
    }
    *err = cudaGetLastError();
    return *err == cudaSuccess;
}

cudaError_t launch_k2(const LaunchCfg& cfg, const DevBatch& b, const DevTable& t,
                      const DevParams& p, const DevPartials& P, const DevHot& hot,
                      const DevLog& log, cudaStream_t s) {
    switch (k2_layout(b)) {
    case 0:
        launch_k2_l<0>(cfg, b, t, p, P, hot, log, s);
        break;
    case 1: launch_k2_l<1>(cfg, b, t, p, P, hot, log, s); break;
    case 2: launch_k2_l<2>(cfg, b, t, p, P, hot, log, s); break;
    case 3: launch_k2_l<3>(cfg, b, t, p, P, hot, log, s); break;
    case 5: launch_k2_l<5>(cfg, b, t, p, P, hot, log, s); break;
    default: launch_k2_l<4>(cfg, b, t, p, P, hot, log, s); break;
    }
    return cudaGetLastError();
}

uint32_t k2_regions(const LaunchCfg& cfg) { return static_cast<uint32_t>(cfg.grid) * (cfg.block / 32); }

uint32_t k2_warp_cap(const LaunchCfg& cfg, const DevBatch& b) {
    // A warp sees at most ceil(ceil(n/G) / (64 * warps)) 64-record tiles (or
    // 32-record rounds), plus the last CTA's < 64-record remainder; every
    // candidate leaves exactly one entry.
    const uint64_t warps = static_cast<uint64_t>(cfg.block / 32);
    const uint64_t per_cta = (b.n + cfg.grid - 1) / cfg.grid;
    return static_cast<uint32_t>((per_cta + 64 * warps - 1) / (64 * warps) * 64 + 128);
}

namespace {
uint32_t small_grid(int device, uint64_t items, uint32_t block) {
    const uint64_t g = (items + block - 1) / block;
    return static_cast<uint32_t>(std::max<uint64_t>(1, std::min<uint64_t>(g, static_cast<uint64_t>(sm_count(device)) * 8)));
}
} // namespace

cudaError_t launch_k3a(int device, const DevPartials& P, cudaStream_t s) {
    if (P.n_sites == 0) return cudaSuccess;
    if (cudaError_t e = cudaMemsetAsync(P.heavy_next, 0, 4, s)) return e;
    k3a_median_sb<<<small_grid(device, static_cast<uint64_t>(P.n_sites) * 4, 128), 128, 0, s>>>(P);
    return cudaGetLastError();
}

cudaError_t launch_k2b(int device, const DevPartials& P, const DevLog& log, cudaStream_t s) {
    if (log.regions == 0) return cudaSuccess;
    // Persistent: GNM_K2B_CTAS CTAs per SM, so the heavy rows flush rarely.
    const uint32_t grid = static_cast<uint32_t>(sm_count(device)) * GNM_K2B_CTAS;
    const bool wide = log.buckets != nullptr;
    if (P.n_sites <= kMapSites) {
        if (wide) k2b_fine<true, true><<<grid, 512, 0, s>>>(P, log);
        else k2b_fine<true, false><<<grid, 512, 0, s>>>(P, log);
    } else {
        if (wide) k2b_fine<false, true><<<grid, 512, 0, s>>>(P, log);
        else k2b_fine<false, false><<<grid, 512, 0, s>>>(P, log);
    }
    return cudaGetLastError();
}

cudaError_t launch_k3b(int device, const DevPartials& P, double threshold, gnm_site_stats* out,
                       int reset, cudaStream_t s) {
    auto* tallies_out = reinterpret_cast<unsigned long long*>(out + P.n_sites);
    k3b_finalize<<<small_grid(device, std::max<uint32_t>(P.n_sites, 1), 128), 128, 0, s>>>(
        P, threshold, out, tallies_out, 1, reset);
    cudaError_t e = cudaGetLastError();
    if (e || !reset) return e;
    if ((e = cudaMemsetAsync(P.coarse, 0, static_cast<size_t>(P.n_sites) * kCoarse * 4, s))) return e;
    return cudaMemsetAsync(P.fine, 0, static_cast<size_t>(P.n_sites) * kFineW * 4, s);
}

cudaError_t launch_reset(int device, const DevPartials& P, cudaStream_t s) {
    (void)device;
    return launch_init_partials(P, s);
}

cudaError_t launch_init_partials(const DevPartials& P, cudaStream_t s) {
    cudaError_t e;
    const size_t n = P.n_sites;
    if ((e = cudaMemsetAsync(P.sums, 0, (n * 4 + 4) * 8, s))) return e;
    if ((e = cudaMemsetAsync(P.mx, 0, n * 8, s))) return e;
    if ((e = cudaMemsetAsync(P.coarse, 0, n * kCoarse * 4, s))) return e;
    if ((e = cudaMemsetAsync(P.fine, 0, n * kFineW * 4, s))) return e;
    if (n)
        k_fill_u64<<<std::min<uint32_t>((P.n_sites + 255) / 256, 1024), 256, 0, s>>>(P.mn, P.n_sites,
                                                                                     kMinInitBits);
    return cudaGetLastError();
}

cudaError_t launch_hist_from_log(int device, const DevLog& log, uint32_t n_sites, uint32_t* dense,
                                 cudaStream_t s) {
    (void)n_sites;
    if (log.regions == 0) return cudaSuccess;
    k_hist_from_log<<<small_grid(device, static_cast<uint64_t>(log.regions) * 32, 256), 256, 0, s>>>(log, dense);
    return cudaGetLastError();
}

cudaError_t launch_classify(const LaunchCfg& cfg, const DevSoA& b, const DevTable& t,
                            const DevParams& p, uint32_t* out, cudaStream_t s) {
    const size_t tbytes = table_smem_bytes(t.n_words);
    if (tbytes <= kSmemTableMax)
        k_classify<true><<<cfg.grid, cfg.block, tbytes, s>>>(b, t.words, t.n_words, p, out);
    else
        k_classify<false><<<cfg.grid, cfg.block, 0, s>>>(b, t.words, t.n_words, p, out);
    return cudaGetLastError();
}

} // namespace gnm

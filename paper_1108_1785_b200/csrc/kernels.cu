// kernels.cu — sm_100a kernels of the flow-analysis hot path.
//
//   K1  k_sample, k_hot_assign, k_table_slots
//                         hot-site plan for skewed batches (see plan_hot)
//   K2  k2                classify -> attribute -> rate -> per-site aggregate
//                         (reduce_slice, rate_engine.cpp:197-240 + add :9-23)
//   K3  k3_finalize       per-site count / median / clamp / flag
//                         (finalize + stats_from + median_bps,
//                          rate_engine.cpp:42-58, 242-292; monitor.cpp:22)
//       k_classify        per-record class/site (classify/attribute :71-86, 127-146)
//
// Paths are relative to /root/reference/proj/core/src.
//
// The path is HBM-bound integer work: 32 algorithmic bytes per
// record, no tensor cores. K2 streams the six SoA columns with 128-bit
// non-allocating loads (4 records per thread per iteration), probes a
// shared-memory-resident radix table (registry.hpp), and reduces into
// order-independent integer/min/max accumulators, so the result is
// bit-identical to the reference for any grid, partitioning or GPU count.
//
// Contention: with Zipf-distributed sites the hottest site receives ~10% of
// all Forward flows, and same-address L2 atomics serialise (~1 ns each). The
// scalar sums of the hot sites (chosen per call by K1 from a 1/64 sample) are
// therefore accumulated in block-private shared memory with native 32-bit
// atomics and explicit carry propagation, and flushed once per CTA; cold
// sites and every histogram bucket go straight to L2 with RED.
#include <cuda_runtime.h>

#include <algorithm>

#include "kernels.cuh"

namespace gnm {
namespace {

constexpr uint32_t kNone = 0xFFFFFFFFu;
constexpr int kK2Block = 512;
constexpr size_t kHotBytes = kHotStride * (5 * 4 + 2 * 8);
constexpr size_t kSmemMax = 227 * 1024;
constexpr size_t kQueueBytes = (kK2Block / 32) * 64 * 16; // per-warp FwdItem queues
constexpr size_t kSmemTableMax = kSmemMax - kHotBytes - kQueueBytes - 1024;

extern __shared__ __align__(16) uint32_t g_smem[];

// ---- streaming loads (read once: do not pollute L1) ----------------------
__device__ __forceinline__ uint4 ld_stream_u4(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ uint2 ld_stream_u2(const void* p) {
    uint2 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v2.u32 {%0,%1}, [%2];"
                 : "=r"(r.x), "=r"(r.y)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ ulonglong2 ld_stream_u64x2(const void* p) {
    ulonglong2 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v2.u64 {%0,%1}, [%2];"
                 : "=l"(r.x), "=l"(r.y)
                 : "l"(p));
    return r;
}

// ---- fire-and-forget global reductions (RED, never a returning ATOM) -------
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
    const uint32_t node = table_word<kSmem>(gt, 4096u + w.y + __popc(w.x & ((1u << bit) - 1u)));
    if (node & 0x80000000u) return node & 0x7FFFFFFFu;
    return table_word<kSmem>(gt, node + ((ip >> 8) & 0xFFu));
}

// attribute (rate_engine.cpp:127-146) as one branch-free probe of both
// endpoints: the two directory words, nodes and leaf words are loaded with
// predicated selects (a uniform node reads word 0 as a dummy leaf), and the
// src value wins when both hit. Avoids the divergent src-then-dst chain.
template <bool kSmem>
__device__ __forceinline__ uint32_t lookup2(const uint32_t* __restrict__ gt, uint32_t src,
                                            uint32_t dst) {
    const uint32_t ds = src >> 16, dd = dst >> 16;
    const uint2 ws = table_pair<kSmem>(gt, ds >> 5);
    const uint2 wd = table_pair<kSmem>(gt, dd >> 5);
    const uint32_t bs = ds & 31u, bd = dd & 31u;
    const bool hs = (ws.x >> bs) & 1u, hd = (wd.x >> bd) & 1u;
    const uint32_t ns =
        hs ? table_word<kSmem>(gt, 4096u + ws.y + __popc(ws.x & ((1u << bs) - 1u))) : 0x80000000u | kNone;
    const uint32_t nd =
        hd ? table_word<kSmem>(gt, 4096u + wd.y + __popc(wd.x & ((1u << bd) - 1u))) : 0x80000000u | kNone;
    const bool us = ns & 0x80000000u, ud = nd & 0x80000000u;
    const uint32_t ls = table_word<kSmem>(gt, us ? 0u : ns + ((src >> 8) & 0xFFu));
    const uint32_t ld = table_word<kSmem>(gt, ud ? 0u : nd + ((dst >> 8) & 0xFFu));
    const uint32_t vs = us ? (hs ? (ns & 0x7FFFFFFFu) : kNone) : ls;
    const uint32_t vd = ud ? (hd ? (nd & 0x7FFFFFFFu) : kNone) : ld;
    return vs != kNone ? vs : vd;
}

template <bool kSmem>
__device__ __forceinline__ void load_table(const uint32_t* __restrict__ gt, uint32_t words) {
    if constexpr (kSmem) {
        const uint4* g4 = reinterpret_cast<const uint4*>(gt);
        uint4* s4 = reinterpret_cast<uint4*>(g_smem);
        for (uint32_t i = threadIdx.x; i < words / 4; i += blockDim.x) s4[i] = __ldg(g4 + i);
    }
}

// ---- block-private hot-site accumulators ---------------------------------
struct HotSmem {
    uint32_t* oct_lo;          // octets, 64-bit as two u32 with carry
    uint32_t* oct_hi;
    uint32_t* u0;              // micro-bps, 96-bit as three u32 with carries
    uint32_t* u1;
    uint32_t* u2;
    unsigned long long* mn;    // f64 bits
    unsigned long long* mx;
};

__device__ __forceinline__ HotSmem hot_smem(uint32_t table_words_in_smem) {
    uint32_t* base = g_smem + table_words_in_smem;
    HotSmem h;
    h.oct_lo = base;
    h.oct_hi = base + kHotStride;
    h.u0 = base + 2 * kHotStride;
    h.u1 = base + 3 * kHotStride;
    h.u2 = base + 4 * kHotStride;
    h.mn = reinterpret_cast<unsigned long long*>(base + 5 * kHotStride);
    h.mx = h.mn + kHotStride;
    return h;
}

__device__ __forceinline__ void hot_init(const HotSmem& h) {
    for (uint32_t i = threadIdx.x; i < kHotStride; i += blockDim.x) {
        h.oct_lo[i] = 0;
        h.oct_hi[i] = 0;
        h.u0[i] = 0;
        h.u1[i] = 0;
        h.u2[i] = 0;
        h.mn[i] = kMinInitBits;
        h.mx[i] = kMaxInitBits;
    }
}

// ---- per-record arithmetic -------------------------------------------------
// bucket_index (rate_engine.cpp:119-125): IEEE division, truncation.
__device__ __forceinline__ uint32_t bucket_of(double rate) {
    const double b = __ddiv_rn(rate, 10000.0);
    return b >= 10000.0 ? 10000u : static_cast<uint32_t>(b);
}

struct Tally {
    uint32_t fwd = 0, ack = 0, admin = 0, unm = 0;
};

// Exact micro-bps of one flow, rate_ubps_of (rate_engine.cpp:100-107):
// floor(octets * 8e9 / dur) as a 128-bit value (hi is non-zero only when
// dur is a few ms and octets are huge). Fast path: the f64 rate already
// approximates the quotient to ~2^-51 relative, so q0 = rz(rate * 1e6)
// lands within a few units of it; the exact integer residual then fixes
// it up. Preconditions of the fast path (product fits in u64, dur <= 2^40,
// quotient < 2^62) bound the estimate error by < 2^12 units and therefore
// the true residual by < 2^52 * 2^0 < 2^63, so the wrapped u64 residual is
// the real one; any estimate the fix-up loop cannot settle falls back to
// the exact division.
__device__ __forceinline__ void ubps_of(uint32_t oct, uint64_t dur, double rate, uint64_t& lo,
                                        uint64_t& hi) {
    hi = 0;
    if (oct <= 2305843009u) {
        const uint64_t p = static_cast<uint64_t>(oct) * 8000000000ull;
        if (dur <= (1ull << 40) && rate < 4.0e12) {
            uint64_t q = static_cast<uint64_t>(__dmul_rz(rate, 1.0e6));
            int64_t r = static_cast<int64_t>(p - q * dur);
            const int64_t d = static_cast<int64_t>(dur);
#pragma unroll 1
            for (int i = 0; i < 4 && r < 0; ++i) {
                --q;
                r += d;
            }
#pragma unroll 1
            for (int i = 0; i < 4 && r >= d; ++i) {
                ++q;
                r -= d;
            }
            if (r >= 0 && r < d) {
                lo = q;
                return;
            }
        }
        lo = p / dur;
        return;
    }
    const unsigned __int128 q = static_cast<unsigned __int128>(oct) * 8000000000ull / dur;
    lo = static_cast<uint64_t>(q);
    hi = static_cast<uint64_t>(q >> 64);
}

// A Forward flow waiting in a warp's queue: packed (slot << 20 | site), octets, duration.
struct FwdItem {
    uint32_t packed;
    uint32_t oct;
    uint64_t dur;
};
constexpr uint32_t kQueue = 64; // per-warp FwdItem capacity (< 32 left + 32 pushed)

// RateHistogram::add (rate_engine.cpp:9-23) for one Forward flow, as
// order-independent reductions:
//   hist[site][bucket] += 1                              (u32, as the reference)
//   octets and micro-bps sums                            exact integers
//   min/max of the f64 rate via u64 min/max on the bit pattern (rates > 0,
//   SURVEY.md §8a' #8); a cached read skips the atomic when it cannot win
//   (a stale value is never below the current min / above the current max).
// Called on warp-compacted items, so the arithmetic runs with full warps.
template <bool kHot>
__device__ __forceinline__ void accumulate(const FwdItem& it, const DevParams& p,
                                           const DevPartials& P, const HotSmem& h) {
    const uint32_t site = it.packed & p.site_mask;
    const uint32_t slot = kHot ? it.packed >> 20 : 0u;
    const bool hot = kHot && slot;
    // Cold sites: fetch the current min/max first (the loads overlap the
    // math), unless the context asked for unconditional min/max reductions.
    unsigned long long cur_mn = 0, cur_mx = ~0ull;
    if (!hot && !p.cold_red) {
        cur_mn = __ldcg(P.mn + site);
        cur_mx = __ldcg(P.mx + site);
    }
    const uint32_t oct = it.oct;
    // flow_rate (rate_engine.cpp:88-94): exact product, one IEEE division.
    const double rate = __ddiv_rn(8000.0 * static_cast<double>(oct), __ull2double_rn(it.dur));
    const uint32_t bucket = bucket_of(rate);
    uint64_t lo, hi;
    ubps_of(oct, it.dur, rate, lo, hi);
    red_add(P.hist + static_cast<size_t>(site) * kBuckets + bucket, 1u);
    const unsigned long long rb = static_cast<unsigned long long>(__double_as_longlong(rate));
    if (hot) {
        // 32-bit shared atomics with exact carry propagation.
        const uint32_t o = atomicAdd(h.oct_lo + slot, oct);
        if (o + oct < o) atomicAdd(h.oct_hi + slot, 1u);
        const uint32_t vl = static_cast<uint32_t>(lo), vh = static_cast<uint32_t>(lo >> 32);
        const uint32_t a = atomicAdd(h.u0 + slot, vl);
        uint32_t c2 = 0;
        if (vh) {
            const uint32_t b = atomicAdd(h.u1 + slot, vh);
            c2 = b + vh < b;
        }
        if (a + vl < a) {
            const uint32_t b = atomicAdd(h.u1 + slot, 1u);
            c2 += b == 0xFFFFFFFFu;
        }
        if (c2 | hi) atomicAdd(h.u2 + slot, c2 + static_cast<uint32_t>(hi));
        if (rb < h.mn[slot]) atomicMin(h.mn + slot, rb);
        if (rb > h.mx[slot]) atomicMax(h.mx + slot, rb);
    } else {
        unsigned long long* s = P.sums + static_cast<size_t>(site) * 4;
        red_add(s + 0, static_cast<unsigned long long>(oct));
        red_add(s + 1, lo & 0xFFFFFFFFull);
        if (lo >> 32) red_add(s + 2, lo >> 32);
        if (hi) red_add(s + 3, hi);
        if (p.cold_red || rb < cur_mn) red_min(P.mn + site, rb);
        if (p.cold_red || rb > cur_mx) red_max(P.mx + site, rb);
    }
}

// reduce_slice's per-record filter + attribution (rate_engine.cpp:199-233),
// fixed order: zero packets, pure ACK, administrative, src-first
// attribution. Returns true (and the packed site value) for Forward flows.
template <bool kSmem>
__device__ __forceinline__ bool classify(bool valid, uint32_t src, uint32_t dst, uint32_t pkts,
                                         uint32_t oct, uint64_t dur, const DevParams& p,
                                         const uint32_t* __restrict__ gt, Tally& t,
                                         uint32_t& packed) {
    if (!valid) return false;
    if (pkts == 0) {
        ++t.admin;
        return false;
    }
    if (static_cast<uint64_t>(oct) < p.ack_plus1 * pkts) {
        ++t.ack;
        return false;
    }
    if (pkts < p.min_packets || dur < p.min_duration_ms || dur == 0) {
        ++t.admin;
        return false;
    }
    uint32_t v;
    if (p.lookup_mode) {
        v = lookup<kSmem>(gt, src);
        if (v == kNone) v = lookup<kSmem>(gt, dst);
    } else {
        v = lookup2<kSmem>(gt, src, dst);
    }
    if (v == kNone) {
        ++t.unm;
        return false;
    }
    ++t.fwd;
    packed = v;
    return true;
}

// Warp-level stream compaction of Forward flows: lanes append their item to
// the warp's shared queue (ballot + popc), and every time 32 are queued the
// whole warp drains one item per lane, so accumulate() never runs with the
// ~40% lane occupancy the class mix would otherwise leave it.
template <bool kHot>
__device__ __forceinline__ void push(bool fwd, const FwdItem& it, FwdItem* q, uint32_t& qn,
                                     uint32_t lane, const DevParams& p, const DevPartials& P,
                                     const HotSmem& h) {
    const unsigned m = __ballot_sync(0xFFFFFFFFu, fwd);
    if (fwd) q[qn + __popc(m & ((1u << lane) - 1u))] = it;
    qn += __popc(m);
    if (qn >= 32) {
        __syncwarp();
        const FwdItem x = q[qn - 32 + lane];
        qn -= 32;
        __syncwarp();
        accumulate<kHot>(x, p, P, h);
    }
}

__device__ __forceinline__ void flush_tallies(const Tally& t, unsigned long long* out) {
    const uint32_t f = __reduce_add_sync(0xFFFFFFFFu, t.fwd);
    const uint32_t a = __reduce_add_sync(0xFFFFFFFFu, t.ack);
    const uint32_t d = __reduce_add_sync(0xFFFFFFFFu, t.admin);
    const uint32_t u = __reduce_add_sync(0xFFFFFFFFu, t.unm);
    if ((threadIdx.x & 31u) == 0) {
        if (f) red_add(out + 0, static_cast<unsigned long long>(f));
        if (a) red_add(out + 1, static_cast<unsigned long long>(a));
        if (d) red_add(out + 2, static_cast<unsigned long long>(d));
        if (u) red_add(out + 3, static_cast<unsigned long long>(u));
    }
}

__device__ __forceinline__ void hot_flush(const HotSmem& h, const DevHot& hot, const DevPartials& P) {
    for (uint32_t slot = 1 + threadIdx.x; slot <= hot.n_slots; slot += blockDim.x) {
        const uint64_t oct = static_cast<uint64_t>(h.oct_hi[slot]) << 32 | h.oct_lo[slot];
        if (oct == 0) continue; // untouched: every Forward flow has >= 97 octets
        const uint32_t site = __ldg(hot.hot_site + slot);
        unsigned long long* s = P.sums + static_cast<size_t>(site) * 4;
        red_add(s + 0, oct);
        red_add(s + 1, static_cast<unsigned long long>(h.u0[slot]));
        if (h.u1[slot]) red_add(s + 2, static_cast<unsigned long long>(h.u1[slot]));
        if (h.u2[slot]) red_add(s + 3, static_cast<unsigned long long>(h.u2[slot]));
        red_min(P.mn + site, h.mn[slot]);
        red_max(P.mx + site, h.mx[slot]);
    }
}

// ---- K2 ----------------------------------------------------------------------
// kLayout 0: SoA, 128-bit vector loads (all columns 16-byte aligned)
//         1: SoA, scalar loads
//         2: AoS 64-byte rows, 128-bit loads
//         3: AoS, scalar loads
// Loops are warp-uniform (each warp walks whole 32- or 128-record tiles with
// a per-lane validity flag) so the queue's warp collectives stay converged.
template <int kLayout, bool kSmem, bool kHot>
__global__ void __launch_bounds__(kK2Block, 2) k2(DevBatch b, const uint32_t* __restrict__ gt,
                                                uint32_t table_words, DevParams p, DevPartials P,
                                                DevHot hot) {
    load_table<kSmem>(gt, table_words);
    HotSmem h{};
    const uint32_t smem_words = kSmem ? table_words : 0u;
    if constexpr (kHot) {
        h = hot_smem(smem_words);
        hot_init(h);
    }
    const uint32_t lane = threadIdx.x & 31u;
    FwdItem* q = reinterpret_cast<FwdItem*>(g_smem + smem_words + (kHot ? kHotBytes / 4 : 0u)) +
                 (threadIdx.x >> 5) * kQueue;
    uint32_t qn = 0;
    __syncthreads();
    Tally t;
    const uint64_t warp_gid = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
    FwdItem it;
    if constexpr (kLayout == 0) {
        // Two records per lane per 64-record warp tile, software-pipelined:
        // the next tile's six loads are in flight while this one is
        // classified, so the load latency is not exposed at first use.
        const DevSoA& c = b.soa;
        const uint64_t n2 = c.n / 2;
        const uint64_t step = nwarps * 32;
        uint64_t base = warp_gid * 32;
        uint2 s{}, d{}, k{}, o{};
        ulonglong2 t0{}, e0{};
        auto fetch = [&](uint64_t bs, uint2& fs, uint2& fd, uint2& fk, uint2& fo, ulonglong2& ft,
                         ulonglong2& fe) {
            const uint64_t g = bs + lane;
            if (bs < n2 && g < n2) {
                fs = ld_stream_u2(c.src + 2 * g);
                fd = ld_stream_u2(c.dst + 2 * g);
                fk = ld_stream_u2(c.pkts + 2 * g);
                fo = ld_stream_u2(c.octets + 2 * g);
                ft = ld_stream_u64x2(c.start + 2 * g);
                fe = ld_stream_u64x2(c.end + 2 * g);
            }
        };
        fetch(base, s, d, k, o, t0, e0);
        for (; base < n2; base += step) {
            const bool ok = base + lane < n2;
            uint2 ns{}, nd{}, nk{}, no{};
            ulonglong2 nt{}, ne{};
            fetch(base + step, ns, nd, nk, no, nt, ne);
            bool f;
            it = FwdItem{0, o.x, e0.x - t0.x};
            f = classify<kSmem>(ok, s.x, d.x, k.x, o.x, it.dur, p, gt, t, it.packed);
            push<kHot>(f, it, q, qn, lane, p, P, h);
            it = FwdItem{0, o.y, e0.y - t0.y};
            f = classify<kSmem>(ok, s.y, d.y, k.y, o.y, it.dur, p, gt, t, it.packed);
            push<kHot>(f, it, q, qn, lane, p, P, h);
            s = ns, d = nd, k = nk, o = no, t0 = nt, e0 = ne;
        }
        // The odd tail record: the first warp of the grid.
        if (warp_gid == 0) {
            const uint64_t i = n2 * 2 + lane;
            const bool ok = i < c.n;
            it = FwdItem{0, ok ? c.octets[i] : 0u, ok ? c.end[i] - c.start[i] : 0ull};
            const bool f = classify<kSmem>(ok, ok ? c.src[i] : 0u, ok ? c.dst[i] : 0u,
                                           ok ? c.pkts[i] : 0u, it.oct, it.dur, p, gt, t, it.packed);
            push<kHot>(f, it, q, qn, lane, p, P, h);
        }
    } else {
        const uint64_t n = b.n;
        for (uint64_t base = warp_gid * 32; base < n; base += nwarps * 32) {
            const uint64_t i = base + lane;
            const bool ok = i < n;
            uint32_t src = 0, dst = 0, pkts = 0, oct = 0;
            uint64_t start = 0, end = 0;
            if (ok) {
                if constexpr (kLayout == 1) {
                    const DevSoA& c = b.soa;
                    src = c.src[i], dst = c.dst[i], pkts = c.pkts[i], oct = c.octets[i];
                    start = c.start[i], end = c.end[i];
                } else if constexpr (kLayout == 2) {
                    const unsigned char* r = static_cast<const unsigned char*>(b.rec) + i * 64;
                    const uint4 a = __ldg(reinterpret_cast<const uint4*>(r));        // src dst nexthop ifs
                    const uint4 cc = __ldg(reinterpret_cast<const uint4*>(r + 16));  // pkts octets first last
                    const ulonglong2 e = __ldg(reinterpret_cast<const ulonglong2*>(r + 48)); // start end
                    src = a.x, dst = a.y, pkts = cc.x, oct = cc.y, start = e.x, end = e.y;
                } else {
                    const unsigned char* r = static_cast<const unsigned char*>(b.rec) + i * 64;
                    const uint32_t* w = reinterpret_cast<const uint32_t*>(r);
                    const uint64_t* qq = reinterpret_cast<const uint64_t*>(r + 48);
                    src = w[0], dst = w[1], pkts = w[4], oct = w[5], start = qq[0], end = qq[1];
                }
            }
            it = FwdItem{0, oct, end - start};
            const bool f = classify<kSmem>(ok, src, dst, pkts, oct, it.dur, p, gt, t, it.packed);
            push<kHot>(f, it, q, qn, lane, p, P, h);
        }
    }
    // Drain the partial queue.
    __syncwarp();
    if (lane < qn) accumulate<kHot>(q[lane], p, P, h);
    flush_tallies(t, P.sums + static_cast<size_t>(P.n_sites) * 4);
    if constexpr (kHot) {
        __syncthreads();
        hot_flush(h, hot, P);
    }
}

// ---- K2, TMA-staged SoA variant ---------------------------------------------
// One persistent CTA per SM (kTmaBlock threads). Each CTA walks tiles
// blockIdx.x, +gridDim.x, ... of kTile records; a tile's six columns (32 KB)
// land in a shared-memory stage through cp.async.bulk (TMA bulk copies,
// evict-first in L2 so the stream does not push the L2-resident histogram and
// accumulators out), completing on the stage's mbarrier. kStages tiles are in
// flight at all times: the LAST warp to finish with a stage re-arms it with
// the CTA's next-but-(kStages-1) tile, so loads never wait for compute.
// Lane l of warp w reads record w*32+l of the tile from shared memory.
constexpr int kTmaBlock = 1024;
constexpr uint32_t kTile = 1024;
constexpr uint32_t kStageBytes = kTile * 32;
constexpr uint32_t kStages = 3;
constexpr uint32_t kChunksPerTile = kTile / 32;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ uint64_t evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes,
                                            uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

struct Stage {
    uint32_t* src;
    uint32_t* dst;
    uint32_t* pkts;
    uint32_t* oct;
    uint64_t* start;
    uint64_t* end;
};

__device__ __forceinline__ Stage stage_at(unsigned char* base, uint32_t s) {
    unsigned char* b = base + static_cast<size_t>(s) * kStageBytes;
    Stage st;
    st.src = reinterpret_cast<uint32_t*>(b);
    st.dst = st.src + kTile;
    st.pkts = st.dst + kTile;
    st.oct = st.pkts + kTile;
    st.start = reinterpret_cast<uint64_t*>(st.oct + kTile);
    st.end = st.start + kTile;
    return st;
}

// Records [first, first + count) of the 4-aligned prefix into stage st.
__device__ __forceinline__ void issue_tile(const Stage& st, const DevSoA& c, uint64_t first,
                                           uint32_t count, uint64_t* bar, uint64_t pol) {
    mbar_expect_tx(bar, count * 32u);
    tma_load_1d(st.src, c.src + first, count * 4u, bar, pol);
    tma_load_1d(st.dst, c.dst + first, count * 4u, bar, pol);
    tma_load_1d(st.pkts, c.pkts + first, count * 4u, bar, pol);
    tma_load_1d(st.oct, c.octets + first, count * 4u, bar, pol);
    tma_load_1d(st.start, c.start + first, count * 8u, bar, pol);
    tma_load_1d(st.end, c.end + first, count * 8u, bar, pol);
}

template <bool kSmem, bool kHot>
__global__ void __launch_bounds__(kTmaBlock, 1) k2_tma(DevSoA c, const uint32_t* __restrict__ gt,
                                                        uint32_t table_words, DevParams p,
                                                        DevPartials P, DevHot hot) {
    const uint32_t smem_words = kSmem ? table_words : 0u;
    load_table<kSmem>(gt, table_words);
    HotSmem h{};
    if constexpr (kHot) {
        h = hot_smem(smem_words);
        hot_init(h);
    }
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t warp = threadIdx.x >> 5;
    const uint32_t nwarps = blockDim.x >> 5;
    uint32_t* after_hot = g_smem + smem_words + (kHot ? kHotBytes / 4 : 0u);
    FwdItem* q = reinterpret_cast<FwdItem*>(after_hot) + warp * kQueue;
    unsigned char* stages = reinterpret_cast<unsigned char*>(after_hot) + nwarps * kQueue * sizeof(FwdItem);
    uint64_t* full = reinterpret_cast<uint64_t*>(stages + static_cast<size_t>(kStages) * kStageBytes);
    uint64_t* empty = full + kStages;
    uint32_t* claim = reinterpret_cast<uint32_t*>(empty + kStages);

    const uint64_t n_vec = c.n & ~3ull; // TMA-covered prefix (16-byte multiples)
    const uint64_t n_tiles = (n_vec + kTile - 1) / kTile;
    auto tile_first = [&](uint32_t local) {
        return (static_cast<uint64_t>(blockIdx.x) + static_cast<uint64_t>(local) * gridDim.x) * kTile;
    };
    auto tile_count = [&](uint64_t first) {
        return static_cast<uint32_t>(min(static_cast<uint64_t>(kTile), n_vec - first));
    };
    const uint32_t my_tiles = static_cast<uint32_t>(
        blockIdx.x < n_tiles ? (n_tiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0);
    const uint32_t my_chunks = my_tiles * kChunksPerTile;

    if (threadIdx.x == 0) {
        for (uint32_t s = 0; s < kStages; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, kChunksPerTile);
        }
        *claim = 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    Tally t;
    FwdItem it;
    uint32_t qn = 0;
    if (warp == 0) {
        // Producer: one lane keeps kStages tiles in flight. A stage is
        // re-armed once all 32 chunks of its previous tile were read
        // (empty[s] phase), so loads never wait for the accumulate() work.
        if (lane == 0) {
            const uint64_t pol = evict_first_policy();
            for (uint32_t j = 0; j < my_tiles; ++j) {
                const uint32_t s = j % kStages;
                if (j >= kStages) mbar_wait(empty + s, ((j / kStages) - 1) & 1u);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                const uint64_t f = tile_first(j);
                issue_tile(stage_at(stages, s), c, f, tile_count(f), full + s, pol);
            }
        }
        __syncwarp();
    } else {
        // Consumers claim 32-record chunks dynamically: a warp held up in
        // accumulate() never delays a stage's release. Claims can run at most
        // one tile past the loaded window (< 32 warps can be parked on an
        // unloaded tile), so every parity below names the right phase.
        for (;;) {
            uint32_t cl = 0;
            if (lane == 0) cl = atomicAdd(claim, 1u);
            cl = __shfl_sync(0xFFFFFFFFu, cl, 0);
            if (cl >= my_chunks) break;
            const uint32_t i = cl / kChunksPerTile;
            const uint32_t chunk = cl % kChunksPerTile;
            const uint32_t s = i % kStages;
            const uint32_t count = tile_count(tile_first(i));
            const Stage st = stage_at(stages, s);
            mbar_wait(full + s, (i / kStages) & 1u);
            const uint32_t k = chunk * 32 + lane;
            const bool ok = k < count;
            uint32_t src = 0, dst = 0, pkts = 0;
            it = FwdItem{0, 0, 0};
            if (ok) {
                src = st.src[k];
                dst = st.dst[k];
                pkts = st.pkts[k];
                it.oct = st.oct[k];
                it.dur = st.end[k] - st.start[k];
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(empty + s);
            const bool f = classify<kSmem>(ok, src, dst, pkts, it.oct, it.dur, p, gt, t, it.packed);
            push<kHot>(f, it, q, qn, lane, p, P, h);
        }
        // The n % 4 tail records: block 0, warp 1, direct loads.
        if (blockIdx.x == 0 && warp == 1) {
            const uint64_t r = n_vec + lane;
            const bool ok = r < c.n;
            it = FwdItem{0, ok ? c.octets[r] : 0u, ok ? c.end[r] - c.start[r] : 0ull};
            const bool f = classify<kSmem>(ok, ok ? c.src[r] : 0u, ok ? c.dst[r] : 0u,
                                           ok ? c.pkts[r] : 0u, it.oct, it.dur, p, gt, t, it.packed);
            push<kHot>(f, it, q, qn, lane, p, P, h);
        }
        __syncwarp();
        if (lane < qn) accumulate<kHot>(q[lane], p, P, h);
    }
    flush_tallies(t, P.sums + static_cast<size_t>(P.n_sites) * 4);
    if constexpr (kHot) {
        __syncthreads();
        hot_flush(h, hot, P);
    }
}

// ---- K1: hot-site plan ------------------------------------------------------
// Each block classifies one contiguous chunk of the batch and counts Forward
// flows per site.
template <bool kSmem>
__global__ void __launch_bounds__(kK2Block) k_sample(DevBatch b, const uint32_t* __restrict__ gt,
                                                      uint32_t table_words, DevParams p,
                                                      uint64_t chunk_stride, uint32_t chunk_len,
                                                      uint32_t* __restrict__ cnt) {
    load_table<kSmem>(gt, table_words);
    if constexpr (kSmem) __syncthreads();
    const uint64_t base = static_cast<uint64_t>(blockIdx.x) * chunk_stride;
    for (uint32_t j = threadIdx.x; j < chunk_len; j += blockDim.x) {
        const uint64_t i = base + j;
        uint32_t src, dst, pkts, oct;
        uint64_t start, end;
        if (b.aos) {
            const unsigned char* r = static_cast<const unsigned char*>(b.rec) + i * 64;
            const uint32_t* w = reinterpret_cast<const uint32_t*>(r);
            const uint64_t* q = reinterpret_cast<const uint64_t*>(r + 48);
            src = w[0], dst = w[1], pkts = w[4], oct = w[5], start = q[0], end = q[1];
        } else {
            src = b.soa.src[i], dst = b.soa.dst[i], pkts = b.soa.pkts[i], oct = b.soa.octets[i];
            start = b.soa.start[i], end = b.soa.end[i];
        }
        const uint64_t dur = end - start;
        if (pkts == 0 || static_cast<uint64_t>(oct) < p.ack_plus1 * pkts || pkts < p.min_packets ||
            dur < p.min_duration_ms || dur == 0)
            continue;
        uint32_t v = lookup<kSmem>(gt, src);
        if (v == kNone) v = lookup<kSmem>(gt, dst);
        if (v != kNone) atomicAdd(cnt + (v & p.site_mask), 1u);
    }
}

// Sites with at least `thr` sampled Forward flows get a slot (first come,
// first served up to kHotSlots; the numbering does not affect results).
// Resets the counts for the next call.
__global__ void k_hot_assign(uint32_t* __restrict__ cnt, uint32_t n_sites, uint32_t thr,
                             uint32_t* __restrict__ site_slot, uint32_t* __restrict__ hot_site,
                             uint32_t* __restrict__ next) {
    for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < n_sites; s += gridDim.x * blockDim.x) {
        const uint32_t c = cnt[s];
        cnt[s] = 0;
        uint32_t slot = 0;
        if (c >= thr) {
            const uint32_t k = atomicAdd(next, 1u);
            if (k < kHotSlots) {
                slot = k + 1;
                hot_site[slot] = s;
            }
        }
        site_slot[s] = slot;
    }
}

// Rewrites the slot bits of every site value in the table (nodes flagged
// uniform and leaf entries) and resets the slot counter.
__global__ void k_table_slots(uint32_t* __restrict__ words, uint32_t node_begin,
                              uint32_t leaf_begin, uint32_t end,
                              const uint32_t* __restrict__ site_slot, uint32_t* __restrict__ next) {
    const uint32_t i0 = blockIdx.x * blockDim.x + threadIdx.x;
    if (i0 == 0) *next = 0;
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

// ---- K3: per-site synthesis --------------------------------------------------
__device__ __forceinline__ uint64_t warp_sum_u64(uint64_t v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, off);
    return v;
}

// One warp per site. The site's rates all lie in [min, max], so its histogram
// is non-zero only on [bucket(min), bucket(max)] (bucket_index is monotone):
// K3 scans (and, with reset, clears) just that range.
__global__ void __launch_bounds__(256) k3_finalize(DevPartials P, double threshold,
                                                   gnm_site_stats* __restrict__ out,
                                                   unsigned long long* __restrict__ tallies_out,
                                                   int write_out, int reset) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        unsigned long long* t = P.sums + static_cast<size_t>(P.n_sites) * 4;
        if (write_out)
            for (int i = 0; i < 4; ++i) tallies_out[i] = t[i];
        if (reset)
            for (int i = 0; i < 4; ++i) t[i] = 0;
    }
    for (uint32_t site = warp; site < P.n_sites; site += nwarps) {
        const unsigned long long mxb = P.mx[site];
        const unsigned long long mnb = P.mn[site];
        if (mxb == 0) { // no Forward flow: absent from result.sites
            if (write_out && lane == 0) {
                gnm_site_stats z = {};
                out[site] = z;
            }
            continue;
        }
        const double mn = __longlong_as_double(static_cast<long long>(mnb));
        const double mx = __longlong_as_double(static_cast<long long>(mxb));
        const uint32_t b0 = bucket_of(mn), b1 = bucket_of(mx);
        unsigned int* row = P.hist + static_cast<size_t>(site) * kBuckets;
        if (write_out) {
            uint64_t c = 0;
            for (uint32_t b = b0 + lane; b <= b1; b += 32) c += row[b];
            c = warp_sum_u64(c);
            // median_bps (rate_engine.cpp:42-58): first k with cumulative >= ceil(c/2).
            const uint64_t target = (c + 1) / 2;
            uint64_t cum = 0;
            uint32_t k = kBuckets - 1;
            for (uint32_t base = b0; base <= b1; base += 32) {
                const uint32_t b = base + lane;
                uint64_t x = b <= b1 ? row[b] : 0u;
#pragma unroll
                for (int off = 1; off < 32; off <<= 1) {
                    const uint64_t y = __shfl_up_sync(0xFFFFFFFFu, x, off);
                    if (lane >= static_cast<uint32_t>(off)) x += y;
                }
                const unsigned hit = __ballot_sync(0xFFFFFFFFu, cum + x >= target);
                if (hit) {
                    k = base + static_cast<uint32_t>(__ffs(hit)) - 1u;
                    break;
                }
                cum += __shfl_sync(0xFFFFFFFFu, x, 31);
            }
            if (lane == 0) {
                double med = k == kBuckets - 1
                                 ? 100000000.0
                                 : __dadd_rn(__dmul_rn(static_cast<double>(k), 10000.0), 5000.0);
                med = med < mn ? mn : (mx < med ? mx : med); // std::clamp (stats_from :251)
                const unsigned long long* s = P.sums + static_cast<size_t>(site) * 4;
                const unsigned __int128 u = static_cast<unsigned __int128>(s[1]) +
                                            (static_cast<unsigned __int128>(s[2]) << 32) +
                                            (static_cast<unsigned __int128>(s[3]) << 64);
                gnm_site_stats o;
                o.flow_count = c;
                o.octets = s[0];
                o.rate_ubps_lo = static_cast<uint64_t>(u);
                o.rate_ubps_hi = static_cast<uint64_t>(u >> 64);
                o.min_bps = mn;
                o.max_bps = mx;
                o.avg_bps = 0; // host: double(u128)/1e6/count, libgcc rounding
                o.median_bps = med;
                o.below_threshold = med < threshold ? 1u : 0u; // monitor.cpp:22
                o.reserved = 0;
                out[site] = o;
            }
        }
        if (reset) {
            __syncwarp();
            for (uint32_t b = b0 + lane; b <= b1; b += 32) row[b] = 0;
            if (lane < 4) P.sums[static_cast<size_t>(site) * 4 + lane] = 0;
            if (lane == 0) {
                P.mn[site] = kMinInitBits;
                P.mx[site] = kMaxInitBits;
            }
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

template <int L>
cudaError_t allow_layout() {
    cudaError_t e;
    if ((e = allow_smem(k2<L, true, true>))) return e;
    if ((e = allow_smem(k2<L, true, false>))) return e;
    if ((e = allow_smem(k2<L, false, true>))) return e;
    return allow_smem(k2<L, false, false>);
}

template <int L, bool kS, bool kH>
void launch_k2_t(const LaunchCfg& cfg, const DevBatch& b, const DevTable& t, const DevParams& p,
                 const DevPartials& P, const DevHot& hot, cudaStream_t s) {
    k2<L, kS, kH><<<cfg.grid, cfg.block, cfg.smem, s>>>(b, t.words, t.n_words, p, P, hot);
}

template <int L>
void launch_k2_l(const LaunchCfg& cfg, const DevBatch& b, const DevTable& t, const DevParams& p,
                 const DevPartials& P, const DevHot& hot, cudaStream_t s) {
    const bool hh = hot.n_slots > 0;
    if (cfg.table_in_smem) {
        if (hh) launch_k2_t<L, true, true>(cfg, b, t, p, P, hot, s);
        else launch_k2_t<L, true, false>(cfg, b, t, p, P, hot, s);
    } else {
        if (hh) launch_k2_t<L, false, true>(cfg, b, t, p, P, hot, s);
        else launch_k2_t<L, false, false>(cfg, b, t, p, P, hot, s);
    }
}

size_t table_smem_bytes(uint32_t table_words) { return static_cast<size_t>(table_words) * 4; }

} // namespace

cudaError_t init_kernel_attributes() {
    cudaError_t e;
    if ((e = allow_layout<0>())) return e;
    if ((e = allow_layout<1>())) return e;
    if ((e = allow_layout<2>())) return e;
    if ((e = allow_layout<3>())) return e;
    if ((e = allow_smem(k2_tma<true, true>))) return e;
    if ((e = allow_smem(k2_tma<true, false>))) return e;
    if ((e = allow_smem(k2_tma<false, true>))) return e;
    if ((e = allow_smem(k2_tma<false, false>))) return e;
    if ((e = allow_smem(k_sample<true>))) return e;
    return allow_smem(k_classify<true>);
}

namespace {
bool soa_aligned(const DevBatch& b) {
    const DevSoA& c = b.soa;
    return !b.aos &&
           ((reinterpret_cast<uintptr_t>(c.src) | reinterpret_cast<uintptr_t>(c.dst) |
             reinterpret_cast<uintptr_t>(c.pkts) | reinterpret_cast<uintptr_t>(c.octets) |
             reinterpret_cast<uintptr_t>(c.start) | reinterpret_cast<uintptr_t>(c.end)) & 15u) == 0;
}
} // namespace

LaunchCfg k2_config(int device, const DevBatch& b, uint32_t table_words, bool hot, int* occ_cache,
                    bool allow_tma) {
    LaunchCfg c;
    const size_t tbytes = table_smem_bytes(table_words);
    const uint64_t n_tiles = ((b.n & ~3ull) + kTile - 1) / kTile;
    c.stages = 0;
    if (allow_tma && soa_aligned(b) && n_tiles > 0) {
        // TMA-staged variant: one 1024-thread CTA per SM, kStages tiles in flight.
        const size_t fixed = (hot ? kHotBytes : 0) + (kTmaBlock / 32) * kQueue * sizeof(FwdItem) +
                             kStages * kStageBytes + 2 * kStages * 8 + 16;
        if (fixed <= kSmemMax) {
            c.block = kTmaBlock;
            c.table_in_smem = tbytes + fixed <= kSmemMax;
            c.smem = fixed + (c.table_in_smem ? tbytes : 0);
            c.stages = kStages;
            c.grid = static_cast<int>(std::min<uint64_t>(sm_count(device), n_tiles));
            return c;
        }
    }
    c.block = kK2Block;
    c.table_in_smem = tbytes <= kSmemTableMax;
    c.smem = (c.table_in_smem ? tbytes : 0) + (hot ? kHotBytes : 0) + kQueueBytes;
    int per_sm = occ_cache ? occ_cache[hot ? 1 : 0] : 0;
    if (per_sm > 0) {
    } else if (c.table_in_smem)
        per_sm = hot ? occupancy(k2<0, true, true>, c.block, c.smem)
                     : occupancy(k2<0, true, false>, c.block, c.smem);
    else
        per_sm = hot ? occupancy(k2<0, false, true>, c.block, c.smem)
                     : occupancy(k2<0, false, false>, c.block, c.smem);
    if (occ_cache) occ_cache[hot ? 1 : 0] = per_sm;
    const uint64_t resident = static_cast<uint64_t>(per_sm) * sm_count(device);
    // At least 16 records per thread so the per-CTA table load amortises.
    const uint64_t per_block = static_cast<uint64_t>(c.block) * 16;
    const uint64_t want = (b.n + per_block - 1) / per_block;
    c.grid = static_cast<int>(std::max<uint64_t>(1, std::min(resident, want)));
    return c;
}

bool plan_hot(int device, const DevBatch& b, const DevTable& t, const DevParams& p,
              uint32_t n_sites, uint32_t* scratch, int k2_grid, bool force, cudaStream_t s,
              uint64_t* launches, cudaError_t* err) {
    (void)device;
    *err = cudaSuccess;
    if (!t.packed || n_sites == 0 || b.n == 0) return false;
    // Sample 1/64 of the batch (at most 256k records) in 64 contiguous chunks.
    const uint32_t chunks = 64;
    uint64_t sample = std::min<uint64_t>(262144, b.n / 64);
    uint32_t chunk_len = static_cast<uint32_t>(sample / chunks);
    uint32_t thr;
    if (force) {
        chunk_len = static_cast<uint32_t>(std::max<uint64_t>(1, std::min<uint64_t>(4096, b.n / chunks)));
        thr = 1;
    } else {
        if (chunk_len < 256) return false;
        // A site is hot when it is expected to see >= 32 Forward flows per
        // K2 CTA, so its block-private accumulator amortises the flush.
        const double thr_d =
            32.0 * k2_grid * static_cast<double>(chunk_len) * chunks / static_cast<double>(b.n);
        thr = static_cast<uint32_t>(std::max(2.0, thr_d));
        if (thr > chunk_len * chunks) return false;
    }
    uint32_t* cnt = scratch;
    uint32_t* site_slot = scratch + n_sites;
    uint32_t* hot_site = site_slot + n_sites;
    uint32_t* next = hot_site + kHotStride;
    const uint64_t stride = std::max<uint64_t>(b.n / chunks, chunk_len);
    const uint32_t nchunks = static_cast<uint32_t>(std::min<uint64_t>(chunks, b.n / chunk_len));
    const size_t tbytes = table_smem_bytes(t.n_words);
    if (tbytes <= kSmemTableMax)
        k_sample<true><<<nchunks, kK2Block, tbytes, s>>>(b, t.words, t.n_words, p, stride, chunk_len, cnt);
    else
        k_sample<false><<<nchunks, kK2Block, 0, s>>>(b, t.words, t.n_words, p, stride, chunk_len, cnt);
    const uint32_t ag = std::min<uint32_t>((n_sites + 255) / 256, 1024);
    k_hot_assign<<<ag, 256, 0, s>>>(cnt, n_sites, thr, site_slot, hot_site, next);
    const uint32_t span = t.n_words - t.node_begin;
    const uint32_t rg = std::max<uint32_t>(1, std::min<uint32_t>((span + 255) / 256, 1024));
    k_table_slots<<<rg, 256, 0, s>>>(t.words, t.node_begin, t.leaf_begin, t.n_words, site_slot, next);
    *launches += 3;
    *err = cudaGetLastError();
    return *err == cudaSuccess;
}

cudaError_t launch_k2(const LaunchCfg& cfg, const DevBatch& b, const DevTable& t,
                      const DevParams& p, const DevPartials& P, const DevHot& hot,
                      cudaStream_t s) {
    if (cfg.stages) {
        const bool hh = hot.n_slots > 0;
        if (cfg.table_in_smem) {
            if (hh) k2_tma<true, true><<<cfg.grid, cfg.block, cfg.smem, s>>>(b.soa, t.words, t.n_words, p, P, hot);
            else k2_tma<true, false><<<cfg.grid, cfg.block, cfg.smem, s>>>(b.soa, t.words, t.n_words, p, P, hot);
        } else {
            if (hh) k2_tma<false, true><<<cfg.grid, cfg.block, cfg.smem, s>>>(b.soa, t.words, t.n_words, p, P, hot);
            else k2_tma<false, false><<<cfg.grid, cfg.block, cfg.smem, s>>>(b.soa, t.words, t.n_words, p, P, hot);
        }
        return cudaGetLastError();
    }
    if (b.aos) {
        const bool vec = (reinterpret_cast<uintptr_t>(b.rec) & 15u) == 0;
        if (vec) launch_k2_l<2>(cfg, b, t, p, P, hot, s);
        else launch_k2_l<3>(cfg, b, t, p, P, hot, s);
    } else {
        const DevSoA& c = b.soa;
        const bool vec = ((reinterpret_cast<uintptr_t>(c.src) | reinterpret_cast<uintptr_t>(c.dst) |
                           reinterpret_cast<uintptr_t>(c.pkts) | reinterpret_cast<uintptr_t>(c.octets) |
                           reinterpret_cast<uintptr_t>(c.start) | reinterpret_cast<uintptr_t>(c.end)) &
                          15u) == 0;
        if (vec) launch_k2_l<0>(cfg, b, t, p, P, hot, s);
        else launch_k2_l<1>(cfg, b, t, p, P, hot, s);
    }
    return cudaGetLastError();
}

cudaError_t launch_k3(int device, const DevPartials& P, double threshold, gnm_site_stats* out,
                      int reset, cudaStream_t s) {
    const int block = 256;
    const uint64_t warps_needed = std::max<uint32_t>(P.n_sites, 1);
    const uint64_t grid = std::min<uint64_t>((warps_needed * 32 + block - 1) / block,
                                             static_cast<uint64_t>(sm_count(device)) * 8);
    auto* tallies_out = reinterpret_cast<unsigned long long*>(out + P.n_sites);
    k3_finalize<<<static_cast<unsigned>(grid), block, 0, s>>>(P, threshold, out, tallies_out, 1, reset);
    return cudaGetLastError();
}

cudaError_t launch_reset(int device, const DevPartials& P, cudaStream_t s) {
    const int block = 256;
    const uint64_t warps_needed = std::max<uint32_t>(P.n_sites, 1);
    const uint64_t grid = std::min<uint64_t>((warps_needed * 32 + block - 1) / block,
                                             static_cast<uint64_t>(sm_count(device)) * 8);
    k3_finalize<<<static_cast<unsigned>(grid), block, 0, s>>>(P, 0.0, nullptr, nullptr, 0, 1);
    return cudaGetLastError();
}

cudaError_t launch_init_partials(const DevPartials& P, cudaStream_t s) {
    cudaError_t e;
    if ((e = cudaMemsetAsync(P.sums, 0, (static_cast<size_t>(P.n_sites) * 4 + 4) * 8, s))) return e;
    if ((e = cudaMemsetAsync(P.mx, 0, static_cast<size_t>(P.n_sites) * 8, s))) return e;
    if ((e = cudaMemsetAsync(P.hist, 0, static_cast<size_t>(P.n_sites) * kBuckets * 4, s))) return e;
    if (P.n_sites)
        k_fill_u64<<<std::min<uint32_t>((P.n_sites + 255) / 256, 1024), 256, 0, s>>>(P.mn, P.n_sites,
                                                                                     kMinInitBits);
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

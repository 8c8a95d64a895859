// kernels.cu — sm_100a kernels of the flow-analysis hot path.
//
//   K2  k2_soa / k2_aos   classify -> attribute -> rate -> per-site aggregate
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
// order-independent integer/min/max accumulators in HBM/L2, so the result is
// bit-identical to the reference for any grid, partitioning or GPU count.
#include <cuda_runtime.h>

#include <algorithm>

#include "kernels.cuh"

namespace gnm {
namespace {

constexpr uint32_t kNone = 0xFFFFFFFFu;
constexpr int kK2Block = 512;

extern __shared__ __align__(16) uint32_t g_smem[];

// ---- streaming loads (read once: do not pollute L1) ----------------------
__device__ __forceinline__ uint4 ld_stream_u4(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
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
// one LDS.64 for a miss, three dependent LDS for a /24 hit.
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

template <bool kSmem>
__device__ __forceinline__ void load_table(const uint32_t* __restrict__ gt, uint32_t words) {
    if constexpr (kSmem) {
        const uint4* g4 = reinterpret_cast<const uint4*>(gt);
        uint4* s4 = reinterpret_cast<uint4*>(g_smem);
        for (uint32_t i = threadIdx.x; i < words / 4; i += blockDim.x) s4[i] = __ldg(g4 + i);
        __syncthreads();
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

// RateHistogram::add (rate_engine.cpp:9-23) for one Forward flow, as
// order-independent reductions:
//   hist[site][bucket] += 1                       (u32, as the reference)
//   octets, ubps limbs (32-bit limbs in u64 lanes) += ...   exact, carry-free
//   min/max of the f64 rate via u64 atomics on the bit pattern (rates > 0,
//   SURVEY.md §8a' #8); a cached read skips the atomic when it cannot win
//   (a stale value is never below the current min / above the current max).
__device__ __forceinline__ void accumulate(uint32_t site, uint32_t oct, uint64_t dur,
                                           const DevPartials& P) {
    // flow_rate (rate_engine.cpp:88-94): exact product, one IEEE division.
    const double rate = __ddiv_rn(8000.0 * static_cast<double>(oct), __ull2double_rn(dur));
    const uint32_t bucket = bucket_of(rate);
    // rate_ubps_of (rate_engine.cpp:100-107).
    uint64_t lo, hi = 0;
    if (oct <= 2305843009u) {
        lo = static_cast<uint64_t>(oct) * 8000000000ull / dur;
    } else {
        const unsigned __int128 q = static_cast<unsigned __int128>(oct) * 8000000000ull / dur;
        lo = static_cast<uint64_t>(q);
        hi = static_cast<uint64_t>(q >> 64);
    }
    atomicAdd(P.hist + static_cast<size_t>(site) * kBuckets + bucket, 1u);
    unsigned long long* s = P.sums + static_cast<size_t>(site) * 4;
    atomicAdd(s + 0, static_cast<unsigned long long>(oct));
    atomicAdd(s + 1, lo & 0xFFFFFFFFull);
    atomicAdd(s + 2, lo >> 32);
    if (hi) atomicAdd(s + 3, hi);
    const unsigned long long rb = static_cast<unsigned long long>(__double_as_longlong(rate));
    if (rb < P.mn[site]) atomicMin(P.mn + site, rb);
    if (rb > P.mx[site]) atomicMax(P.mx + site, rb);
}

// reduce_slice's per-record body (rate_engine.cpp:199-239), fixed order:
// zero packets, pure ACK, administrative, src-first attribution.
template <bool kSmem>
__device__ __forceinline__ void process(uint32_t src, uint32_t dst, uint32_t pkts, uint32_t oct,
                                        uint64_t start, uint64_t end, const DevParams& p,
                                        const uint32_t* __restrict__ gt, const DevPartials& P,
                                        Tally& t) {
    if (pkts == 0) {
        ++t.admin;
        return;
    }
    if (static_cast<uint64_t>(oct) < p.ack_plus1 * pkts) {
        ++t.ack;
        return;
    }
    const uint64_t dur = end - start;
    if (pkts < p.min_packets || dur < p.min_duration_ms || dur == 0) {
        ++t.admin;
        return;
    }
    uint32_t site = lookup<kSmem>(gt, src);
    if (site == kNone) site = lookup<kSmem>(gt, dst);
    if (site == kNone) {
        ++t.unm;
        return;
    }
    ++t.fwd;
    accumulate(site, oct, dur, P);
}

__device__ __forceinline__ uint32_t warp_sum_u32(uint32_t v) {
    return __reduce_add_sync(0xFFFFFFFFu, v);
}

__device__ __forceinline__ void flush_tallies(const Tally& t, unsigned long long* out) {
    const uint32_t f = warp_sum_u32(t.fwd), a = warp_sum_u32(t.ack), d = warp_sum_u32(t.admin),
                   u = warp_sum_u32(t.unm);
    if ((threadIdx.x & 31u) == 0) {
        if (f) atomicAdd(out + 0, static_cast<unsigned long long>(f));
        if (a) atomicAdd(out + 1, static_cast<unsigned long long>(a));
        if (d) atomicAdd(out + 2, static_cast<unsigned long long>(d));
        if (u) atomicAdd(out + 3, static_cast<unsigned long long>(u));
    }
}

// ---- K2 over SoA columns ----------------------------------------------------
template <bool kSmem, bool kVec>
__global__ void __launch_bounds__(kK2Block) k2_soa(DevSoA b, const uint32_t* __restrict__ gt,
                                                    uint32_t table_words, DevParams p,
                                                    DevPartials P) {
    load_table<kSmem>(gt, table_words);
    Tally t;
    const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    uint64_t done = 0;
    if constexpr (kVec) {
        const uint64_t n4 = b.n / 4;
        for (uint64_t g = tid; g < n4; g += stride) {
            const uint4 s = ld_stream_u4(b.src + 4 * g);
            const uint4 d = ld_stream_u4(b.dst + 4 * g);
            const uint4 k = ld_stream_u4(b.pkts + 4 * g);
            const uint4 o = ld_stream_u4(b.octets + 4 * g);
            const ulonglong2 t0 = ld_stream_u64x2(b.start + 4 * g);
            const ulonglong2 t1 = ld_stream_u64x2(b.start + 4 * g + 2);
            const ulonglong2 e0 = ld_stream_u64x2(b.end + 4 * g);
            const ulonglong2 e1 = ld_stream_u64x2(b.end + 4 * g + 2);
            process<kSmem>(s.x, d.x, k.x, o.x, t0.x, e0.x, p, gt, P, t);
            process<kSmem>(s.y, d.y, k.y, o.y, t0.y, e0.y, p, gt, P, t);
            process<kSmem>(s.z, d.z, k.z, o.z, t1.x, e1.x, p, gt, P, t);
            process<kSmem>(s.w, d.w, k.w, o.w, t1.y, e1.y, p, gt, P, t);
        }
        done = n4 * 4;
    }
    for (uint64_t i = done + tid; i < b.n; i += stride)
        process<kSmem>(b.src[i], b.dst[i], b.pkts[i], b.octets[i], b.start[i], b.end[i], p, gt, P, t);
    flush_tallies(t, P.sums + static_cast<size_t>(P.n_sites) * 4);
}

// ---- K2 over 64-byte flowmon::FlowRecord AoS (netflow.hpp:59-67) -----------
template <bool kSmem, bool kVec>
__global__ void __launch_bounds__(kK2Block) k2_aos(const unsigned char* __restrict__ rec,
                                                    uint64_t n, const uint32_t* __restrict__ gt,
                                                    uint32_t table_words, DevParams p,
                                                    DevPartials P) {
    load_table<kSmem>(gt, table_words);
    Tally t;
    const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = tid; i < n; i += stride) {
        const unsigned char* r = rec + i * 64;
        if constexpr (kVec) {
            const uint4 a = __ldg(reinterpret_cast<const uint4*>(r));        // src dst nexthop ifs
            const uint4 c = __ldg(reinterpret_cast<const uint4*>(r + 16));   // pkts octets first last
            const ulonglong2 e = __ldg(reinterpret_cast<const ulonglong2*>(r + 48)); // start end
            process<kSmem>(a.x, a.y, c.x, c.y, e.x, e.y, p, gt, P, t);
        } else {
            const uint32_t* w = reinterpret_cast<const uint32_t*>(r);
            const uint64_t* q = reinterpret_cast<const uint64_t*>(r + 48);
            process<kSmem>(w[0], w[1], w[4], w[5], q[0], q[1], p, gt, P, t);
        }
    }
    flush_tallies(t, P.sums + static_cast<size_t>(P.n_sites) * 4);
}

// ---- per-record classification --------------------------------------------
template <bool kSmem>
__global__ void __launch_bounds__(kK2Block) k_classify(DevSoA b, const uint32_t* __restrict__ gt,
                                                        uint32_t table_words, DevParams p,
                                                        uint32_t* __restrict__ out) {
    load_table<kSmem>(gt, table_words);
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
            uint32_t s = lookup<kSmem>(gt, b.src[i]);
            if (s == kNone) s = lookup<kSmem>(gt, b.dst[i]);
            if (s == kNone) cls = GNM_UNMATCHED;
            else {
                cls = GNM_FORWARD;
                site = s & 0x3FFFFFFFu;
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
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device);
    return n > 0 ? n : 1;
}

template <typename K>
int occupancy(K kernel, int block, size_t smem) {
    int blocks = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, kernel, block, smem);
    return blocks > 0 ? blocks : 1;
}

constexpr size_t kSmemTableMax = 200 * 1024;

template <typename K>
cudaError_t allow_smem(K kernel) {
    return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(kSmemTableMax));
}

} // namespace

cudaError_t init_kernel_attributes() {
    cudaError_t e;
    if ((e = allow_smem(k2_soa<true, true>))) return e;
    if ((e = allow_smem(k2_soa<true, false>))) return e;
    if ((e = allow_smem(k2_aos<true, true>))) return e;
    if ((e = allow_smem(k2_aos<true, false>))) return e;
    return allow_smem(k_classify<true>);
}

LaunchCfg k2_config(int device, uint64_t n, uint32_t table_words, bool aos) {
    LaunchCfg c;
    c.block = kK2Block;
    const size_t bytes = static_cast<size_t>(table_words) * 4;
    c.table_in_smem = bytes <= kSmemTableMax;
    c.smem = c.table_in_smem ? bytes : 0;
    int per_sm;
    if (aos)
        per_sm = c.table_in_smem ? occupancy(k2_aos<true, true>, c.block, c.smem)
                                 : occupancy(k2_aos<false, true>, c.block, 0);
    else
        per_sm = c.table_in_smem ? occupancy(k2_soa<true, true>, c.block, c.smem)
                                 : occupancy(k2_soa<false, true>, c.block, 0);
    const uint64_t resident = static_cast<uint64_t>(per_sm) * sm_count(device);
    // At least 16 records per thread so the per-CTA table load amortises.
    const uint64_t want = (n + static_cast<uint64_t>(c.block) * 16 - 1) / (static_cast<uint64_t>(c.block) * 16);
    c.grid = static_cast<int>(std::max<uint64_t>(1, std::min(resident, want)));
    return c;
}

cudaError_t launch_k2_soa(const LaunchCfg& cfg, const DevSoA& b, const uint32_t* table,
                          uint32_t table_words, const DevParams& p, const DevPartials& P,
                          cudaStream_t s) {
    const bool vec = ((reinterpret_cast<uintptr_t>(b.src) | reinterpret_cast<uintptr_t>(b.dst) |
                       reinterpret_cast<uintptr_t>(b.pkts) | reinterpret_cast<uintptr_t>(b.octets) |
                       reinterpret_cast<uintptr_t>(b.start) | reinterpret_cast<uintptr_t>(b.end)) &
                      15u) == 0;
    if (cfg.table_in_smem) {
        if (vec) {
            k2_soa<true, true><<<cfg.grid, cfg.block, cfg.smem, s>>>(b, table, table_words, p, P);
        } else {
            k2_soa<true, false><<<cfg.grid, cfg.block, cfg.smem, s>>>(b, table, table_words, p, P);
        }
    } else {
        if (vec) k2_soa<false, true><<<cfg.grid, cfg.block, 0, s>>>(b, table, table_words, p, P);
        else k2_soa<false, false><<<cfg.grid, cfg.block, 0, s>>>(b, table, table_words, p, P);
    }
    return cudaGetLastError();
}

cudaError_t launch_k2_aos(const LaunchCfg& cfg, const void* records, uint64_t n,
                          const uint32_t* table, uint32_t table_words, const DevParams& p,
                          const DevPartials& P, cudaStream_t s) {
    const auto* r = static_cast<const unsigned char*>(records);
    const bool vec = (reinterpret_cast<uintptr_t>(records) & 15u) == 0;
    if (cfg.table_in_smem) {
        if (vec) {
            k2_aos<true, true><<<cfg.grid, cfg.block, cfg.smem, s>>>(r, n, table, table_words, p, P);
        } else {
            k2_aos<true, false><<<cfg.grid, cfg.block, cfg.smem, s>>>(r, n, table, table_words, p, P);
        }
    } else {
        if (vec) k2_aos<false, true><<<cfg.grid, cfg.block, 0, s>>>(r, n, table, table_words, p, P);
        else k2_aos<false, false><<<cfg.grid, cfg.block, 0, s>>>(r, n, table, table_words, p, P);
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
    if (P.n_sites) k_fill_u64<<<std::min<uint32_t>((P.n_sites + 255) / 256, 1024), 256, 0, s>>>(P.mn, P.n_sites, kMinInitBits);
    return cudaGetLastError();
}

cudaError_t launch_classify(const LaunchCfg& cfg, const DevSoA& b, const uint32_t* table,
                            uint32_t table_words, const DevParams& p, uint32_t* out,
                            cudaStream_t s) {
    if (cfg.table_in_smem) {
        k_classify<true><<<cfg.grid, cfg.block, cfg.smem, s>>>(b, table, table_words, p, out);
    } else {
        k_classify<false><<<cfg.grid, cfg.block, 0, s>>>(b, table, table_words, p, out);
    }
    return cudaGetLastError();
}

} // namespace gnm

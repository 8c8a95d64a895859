// hosts.cu — per-host statistics on sm_100a.
//
// The reference keys every Forward flow's RateHistogram by (site << 32 |
// host) (reduce_slice, rate_engine.cpp:216-239), merges the per-thread
// histograms in a std::map and emits SiteResult::hosts[host] =
// stats_from(hist) (finalize, rate_engine.cpp:272-289). Paths are relative to
// /root/reference/proj/core/src.
//
// Here K2 (hosts mode) logs each Forward flow's site, bucket, host, f64 rate
// bits and exact micro-bps; at finalize this post-pass turns the log into the
// reference's rows without any per-host histogram storage:
//   H0  flat offsets: exclusive scan of the per-warp log counts;
//   H1  insert every (site, host) key into an open-addressing table and
//       flatten the log (slot, bucket, log position per flow);
//   H2  collect the distinct keys, radix-sort them: row = rank in (site,
//       host) order, i.e. the std::map's iteration order;
//   H3  per flow key = row << 14 | bucket, radix-sorted with the log position
//       as payload, so every row's flows form one run in bucket order;
//   H4  one pass over the sorted runs: count, u128 micro-bps sum, min, max
//       (segmented warp scans, one atomic per run per warp) and run starts;
//   H5  per row: the lower median is the run's element (count + 1) / 2 - 1
//       (RateHistogram::median_bps, rate_engine.cpp:42-58), clamped, avg as
//       the host rounds it (stats_from, :242-253).
#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cstdint>

#include "hosts.cuh"

namespace gnm {
namespace {

constexpr unsigned long long kEmpty = ~0ull;
constexpr uint32_t kBucketBits = 14;
constexpr uint32_t kBucketMask = (1u << kBucketBits) - 1u;

int bits_for(uint64_t n) { // smallest b with 2^b >= n (n >= 1)
    int b = 0;
    while ((1ull << b) < n) ++b;
    return b;
}

__global__ void h_total(const unsigned int* counts, const uint32_t* off, size_t n,
                        unsigned long long* total) {
    *total = n ? static_cast<unsigned long long>(off[n - 1]) + counts[n - 1] : 0ull;
}

__device__ __forceinline__ uint32_t insert_key(unsigned long long* keys, uint32_t mask, int shift,
                                               unsigned long long key) {
    uint32_t h = static_cast<uint32_t>((key * 0x9E3779B97F4A7C15ull) >> shift) & mask;
    while (true) {
        unsigned long long cur = keys[h];
        if (cur == key) return h;
        if (cur == kEmpty) {
            cur = atomicCAS(keys + h, kEmpty, key);
            if (cur == kEmpty || cur == key) return h;
        }
        h = (h + 1) & mask;
    }
}

// H1, warp per log region of one slice.
__global__ void __launch_bounds__(256) h_insert(DevLog L, const unsigned int* __restrict__ counts,
                                                const uint32_t* __restrict__ off, uint32_t entry_off,
                                                unsigned long long* keys, uint32_t mask, int shift,
                                                uint32_t* __restrict__ slot_of,
                                                uint32_t* __restrict__ bk,
                                                uint32_t* __restrict__ logpos) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < L.regions; r += nwarps) {
        const uint32_t n = counts[r];
        const uint32_t base = off[r];
        const size_t rb = static_cast<size_t>(r) * L.warp_cap;
        for (uint32_t i = lane; i < n; i += 32) {
            const size_t pos = rb + i;
            const uint32_t x = L.entries[pos];
            const uint32_t site = L.buckets ? x : x >> kLogSiteShift;
            const uint32_t b = L.buckets ? L.buckets[pos] : x & kBucketMask;
            const unsigned long long key = static_cast<unsigned long long>(site) << 32 | L.hosts[pos];
            slot_of[base + i] = insert_key(keys, mask, shift, key);
            bk[base + i] = b;
            logpos[base + i] = entry_off + static_cast<uint32_t>(pos);
        }
    }
}

// H2a: the occupied slots, in any order.
__global__ void __launch_bounds__(256) h_collect(const unsigned long long* __restrict__ keys, uint32_t cap,
                                                 unsigned long long* __restrict__ hk,
                                                 uint32_t* __restrict__ hs,
                                                 unsigned int* __restrict__ n_out) {
    const uint32_t lane = threadIdx.x & 31u;
    for (uint32_t base = blockIdx.x * blockDim.x; base < cap; base += gridDim.x * blockDim.x) {
        const uint32_t s = base + threadIdx.x;
        const unsigned long long k = s < cap ? keys[s] : kEmpty;
        const bool occ = k != kEmpty;
        const unsigned m = __ballot_sync(0xFFFFFFFFu, occ);
        uint32_t first = 0;
        if (lane == 0 && m) first = atomicAdd(n_out, __popc(m));
        first = __shfl_sync(0xFFFFFFFFu, first, 0);
        if (occ) {
            const uint32_t i = first + __popc(m & ((1u << lane) - 1u));
            hk[i] = k;
            hs[i] = s;
        }
    }
}

// H2b: slot -> row, written over the table (the keys are no longer needed).
__global__ void h_rank(const uint32_t* __restrict__ hs_sorted, uint32_t n, unsigned long long* keys) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        keys[hs_sorted[i]] = i;
}

template <typename K>
__global__ void h_keys(const uint32_t* __restrict__ slot_of, const uint32_t* __restrict__ bk, uint32_t n,
                       const unsigned long long* __restrict__ rank, K* __restrict__ sk) {
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x)
        sk[j] = static_cast<K>(rank[slot_of[j]]) << kBucketBits | bk[j];
}

// H4: acc[row] = {count, limb0, limb1, limb2, min bits, max bits}.
template <typename K>
__global__ void __launch_bounds__(256) h_reduce(const K* __restrict__ sk, const uint32_t* __restrict__ pos,
                                                uint32_t n, DevLog whole,
                                                unsigned long long* __restrict__ acc,
                                                uint32_t* __restrict__ start) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t base = blockIdx.x * blockDim.x; base < n; base += stride) {
        const uint32_t i = base + threadIdx.x;
        const bool in = i < n;
        uint64_t row = ~0ull;
        unsigned long long c = 0, l0 = 0, l1 = 0, l2 = 0, mn = kMinInitBits, mx = kMaxInitBits;
        if (in) {
            row = static_cast<uint64_t>(sk[i] >> kBucketBits);
            const uint32_t p = pos[i];
            const unsigned long long lo = whole.ulo[p];
            c = 1;
            l0 = lo & 0xFFFFFFFFull;
            l1 = lo >> 32;
            l2 = whole.uhi[p];
            mn = mx = whole.rates[p];
            if (i == 0 || static_cast<uint64_t>(sk[i - 1] >> kBucketBits) != row) start[row] = i;
        }
        // Segmented inclusive scan: runs are contiguous because rows are sorted.
#pragma unroll
        for (uint32_t d = 1; d < 32; d <<= 1) {
            const uint64_t r2 = __shfl_up_sync(0xFFFFFFFFu, row, d);
            const unsigned long long c2 = __shfl_up_sync(0xFFFFFFFFu, c, d);
            const unsigned long long a0 = __shfl_up_sync(0xFFFFFFFFu, l0, d);
            const unsigned long long a1 = __shfl_up_sync(0xFFFFFFFFu, l1, d);
            const unsigned long long a2 = __shfl_up_sync(0xFFFFFFFFu, l2, d);
            const unsigned long long m2 = __shfl_up_sync(0xFFFFFFFFu, mn, d);
            const unsigned long long x2 = __shfl_up_sync(0xFFFFFFFFu, mx, d);
            if (lane >= d && r2 == row) {
                c += c2;
                l0 += a0;
                l1 += a1;
                l2 += a2;
                mn = min(mn, m2);
                mx = max(mx, x2);
            }
        }
        const uint64_t next = __shfl_down_sync(0xFFFFFFFFu, row, 1);
        if (in && (lane == 31 || next != row)) { // run tail within this warp
            unsigned long long* a = acc + row * 6;
            atomicAdd(a + 0, c);
            atomicAdd(a + 1, l0);
            atomicAdd(a + 2, l1);
            atomicAdd(a + 3, l2);
            atomicMin(a + 4, mn);
            atomicMax(a + 5, mx);
        }
    }
}

__global__ void h_init(unsigned long long* acc, uint32_t n_rows) {
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n_rows; r += gridDim.x * blockDim.x) {
        unsigned long long* a = acc + static_cast<size_t>(r) * 6;
        a[0] = a[1] = a[2] = a[3] = 0;
        a[4] = kMinInitBits;
        a[5] = kMaxInitBits;
    }
}

// H5, thread per row.
template <typename K>
__global__ void h_final(const unsigned long long* __restrict__ acc, const uint32_t* __restrict__ start,
                        const K* __restrict__ sk, const unsigned long long* __restrict__ hk_sorted,
                        uint32_t n_rows, gnm_host_stats* __restrict__ rows) {
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n_rows; r += gridDim.x * blockDim.x) {
        const unsigned long long* a = acc + static_cast<size_t>(r) * 6;
        const uint64_t cnt = a[0];
        const unsigned __int128 u = static_cast<unsigned __int128>(a[1]) +
                                    (static_cast<unsigned __int128>(a[2]) << 32) +
                                    (static_cast<unsigned __int128>(a[3]) << 64);
        const uint32_t k = static_cast<uint32_t>(sk[start[r] + (cnt + 1) / 2 - 1] & kBucketMask);
        const double mn = __longlong_as_double(static_cast<long long>(a[4]));
        const double mx = __longlong_as_double(static_cast<long long>(a[5]));
        double med = median_of_bucket(k);
        med = med < mn ? mn : (mx < med ? mx : med);
        gnm_host_stats o;
        o.site = static_cast<uint32_t>(hk_sorted[r] >> 32);
        o.host = static_cast<uint32_t>(hk_sorted[r]);
        o.flow_count = cnt;
        o.rate_ubps_lo = static_cast<uint64_t>(u);
        o.rate_ubps_hi = static_cast<uint64_t>(u >> 64);
        o.min_bps = mn;
        o.max_bps = mx;
        o.avg_bps = avg_of(o.rate_ubps_lo, o.rate_ubps_hi, cnt);
        o.median_bps = med;
        rows[r] = o;
    }
}

template <typename K>
__global__ void h_hist(const K* __restrict__ sk, uint64_t n, uint32_t* __restrict__ dense) {
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const K k = sk[i];
        atomicAdd(dense + static_cast<size_t>(k >> kBucketBits) * kBuckets + (k & kBucketMask), 1u);
    }
}

uint32_t grid_for(int device, uint64_t n, uint32_t block) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    return static_cast<uint32_t>(std::max<uint64_t>(1, std::min<uint64_t>((n + block - 1) / block,
                                                                           static_cast<uint64_t>(std::max(sms, 1)) * 16)));
}

#define HCK(x)                                \
    do {                                      \
        const cudaError_t e_ = (x);           \
        if (e_ != cudaSuccess) return e_;     \
    } while (0)

template <typename T>
cudaError_t dalloc(T** p, size_t n, cudaStream_t s) {
    return cudaMallocAsync(reinterpret_cast<void**>(p), std::max<size_t>(n, 1) * sizeof(T), s);
}

// H3..H5 for one key width.
template <typename K>
cudaError_t sort_and_reduce(int device, uint32_t n, uint32_t n_rows, const uint32_t* slot_of, const uint32_t* bk,
                            uint32_t* logpos, const unsigned long long* rank_tab,
                            const unsigned long long* hk_sorted, const DevLog& whole, HostRows& out,
                            cudaStream_t s) {
    K *sk = nullptr, *sk2 = nullptr;
    uint32_t* pos2 = nullptr;
    HCK(dalloc(&sk, n, s));
    HCK(dalloc(&sk2, n, s));
    HCK(dalloc(&pos2, n, s));
    h_keys<K><<<grid_for(device, n, 256), 256, 0, s>>>(slot_of, bk, n, rank_tab, sk);
    HCK(cudaGetLastError());
    const int end_bit = static_cast<int>(kBucketBits) + std::max(1, bits_for(n_rows));
    size_t tb = 0;
    HCK(cub::DeviceRadixSort::SortPairs(nullptr, tb, sk, sk2, logpos, pos2, n, 0, end_bit, s));
    void* tmp = nullptr;
    HCK(cudaMallocAsync(&tmp, std::max<size_t>(tb, 1), s));
    HCK(cub::DeviceRadixSort::SortPairs(tmp, tb, sk, sk2, logpos, pos2, n, 0, end_bit, s));
    HCK(cudaFreeAsync(tmp, s));
    HCK(cudaFreeAsync(sk, s));
    unsigned long long* acc = nullptr;
    uint32_t* start = nullptr;
    HCK(dalloc(&acc, static_cast<size_t>(n_rows) * 6, s));
    HCK(dalloc(&start, n_rows, s));
    h_init<<<grid_for(device, n_rows, 256), 256, 0, s>>>(acc, n_rows);
    h_reduce<K><<<grid_for(device, n, 256), 256, 0, s>>>(sk2, pos2, n, whole, acc, start);
    HCK(cudaGetLastError());
    HCK(dalloc(&out.rows, n_rows, s));
    h_final<K><<<grid_for(device, n_rows, 128), 128, 0, s>>>(acc, start, sk2, hk_sorted, n_rows, out.rows);
    HCK(cudaGetLastError());
    HCK(cudaFreeAsync(acc, s));
    HCK(cudaFreeAsync(start, s));
    HCK(cudaFreeAsync(pos2, s));
    out.sorted = sk2;
    out.key64 = sizeof(K) == 8;
    out.n_rows = n_rows;
    out.n_flows = n;
    return cudaSuccess;
}

} // namespace

cudaError_t build_hosts(int device, const DevLog& whole, const HostSlice* slices, int n_slices,
                        const unsigned int* counts, size_t n_counts, HostRows& out, cudaStream_t s) {
    free_hosts(out, s);
    if (n_counts == 0) return cudaSuccess;
    // H0: flat offsets of every warp region's entries.
    uint32_t* off = nullptr;
    unsigned long long* scal = nullptr; // [0] total flows, [1] distinct keys
    HCK(dalloc(&off, n_counts, s));
    HCK(dalloc(&scal, 2, s));
    size_t tb = 0;
    HCK(cub::DeviceScan::ExclusiveSum(nullptr, tb, counts, off, n_counts, s));
    void* tmp = nullptr;
    HCK(cudaMallocAsync(&tmp, std::max<size_t>(tb, 1), s));
    HCK(cub::DeviceScan::ExclusiveSum(tmp, tb, counts, off, n_counts, s));
    HCK(cudaFreeAsync(tmp, s));
    HCK(cudaMemsetAsync(scal, 0, 16, s));
    h_total<<<1, 1, 0, s>>>(counts, off, n_counts, scal);
    unsigned long long h_scal[2] = {0, 0};
    HCK(cudaMemcpyAsync(h_scal, scal, 8, cudaMemcpyDeviceToHost, s));
    HCK(cudaStreamSynchronize(s));
    const uint64_t n = h_scal[0];
    if (n == 0) {
        HCK(cudaFreeAsync(off, s));
        HCK(cudaFreeAsync(scal, s));
        return cudaSuccess;
    }
    // H1: key table of at least 2 slots per flow.
    const int tbits = std::max(10, bits_for(2 * n));
    const uint32_t cap = 1u << tbits;
    unsigned long long* keys = nullptr;
    uint32_t *slot_of = nullptr, *bk = nullptr, *logpos = nullptr;
    HCK(dalloc(&keys, cap, s));
    HCK(dalloc(&slot_of, n, s));
    HCK(dalloc(&bk, n, s));
    HCK(dalloc(&logpos, n, s));
    HCK(cudaMemsetAsync(keys, 0xFF, static_cast<size_t>(cap) * 8, s));
    for (int i = 0; i < n_slices; ++i) {
        const HostSlice& sl = slices[i];
        h_insert<<<grid_for(device, static_cast<uint64_t>(sl.log.regions) * 32, 256), 256, 0, s>>>(
            sl.log, counts + sl.count_off, off + sl.count_off, static_cast<uint32_t>(sl.entry_off), keys,
            cap - 1, 64 - tbits, slot_of, bk, logpos);
        HCK(cudaGetLastError());
    }
    // H2: distinct keys in (site, host) order -> rows.
    unsigned long long *hk = nullptr, *hk_sorted = nullptr;
    uint32_t *hs = nullptr, *hs_sorted = nullptr;
    HCK(dalloc(&hk, n, s));
    HCK(dalloc(&hs, n, s));
    h_collect<<<grid_for(device, cap, 256), 256, 0, s>>>(keys, cap, hk, hs,
                                                        reinterpret_cast<unsigned int*>(scal + 1));
    HCK(cudaGetLastError());
    HCK(cudaMemcpyAsync(h_scal + 1, scal + 1, 8, cudaMemcpyDeviceToHost, s));
    HCK(cudaStreamSynchronize(s));
    const uint32_t n_rows = static_cast<uint32_t>(h_scal[1]);
    HCK(dalloc(&hk_sorted, n_rows, s));
    HCK(dalloc(&hs_sorted, n_rows, s));
    tb = 0;
    HCK(cub::DeviceRadixSort::SortPairs(nullptr, tb, hk, hk_sorted, hs, hs_sorted, n_rows, 0, 64, s));
    HCK(cudaMallocAsync(&tmp, std::max<size_t>(tb, 1), s));
    HCK(cub::DeviceRadixSort::SortPairs(tmp, tb, hk, hk_sorted, hs, hs_sorted, n_rows, 0, 64, s));
    HCK(cudaFreeAsync(tmp, s));
    h_rank<<<grid_for(device, n_rows, 256), 256, 0, s>>>(hs_sorted, n_rows, keys);
    HCK(cudaGetLastError());
    // H3..H5.
    const uint32_t n32 = static_cast<uint32_t>(n);
    if (kBucketBits + bits_for(n_rows) <= 32)
        HCK(sort_and_reduce<uint32_t>(device, n32, n_rows, slot_of, bk, logpos, keys, hk_sorted, whole, out, s));
    else
        HCK(sort_and_reduce<unsigned long long>(device, n32, n_rows, slot_of, bk, logpos, keys, hk_sorted, whole,
                                                out, s));
    for (void* p : {static_cast<void*>(off), static_cast<void*>(scal), static_cast<void*>(keys),
                    static_cast<void*>(slot_of), static_cast<void*>(bk), static_cast<void*>(logpos),
                    static_cast<void*>(hk), static_cast<void*>(hs), static_cast<void*>(hk_sorted),
                    static_cast<void*>(hs_sorted)})
        HCK(cudaFreeAsync(p, s));
    return cudaSuccess;
}

cudaError_t hosts_histograms(int device, const HostRows& h, uint32_t* dense, cudaStream_t s) {
    if (h.n_flows == 0) return cudaSuccess;
    const uint32_t g = grid_for(device, h.n_flows, 256);
    if (h.key64)
        h_hist<unsigned long long><<<g, 256, 0, s>>>(static_cast<const unsigned long long*>(h.sorted), h.n_flows,
                                                     dense);
    else
        h_hist<uint32_t><<<g, 256, 0, s>>>(static_cast<const uint32_t*>(h.sorted), h.n_flows, dense);
    return cudaGetLastError();
}

void free_hosts(HostRows& h, cudaStream_t s) {
    if (h.rows) cudaFreeAsync(h.rows, s);
    if (h.sorted) cudaFreeAsync(h.sorted, s);
    h = HostRows{};
}

} // namespace gnm

// hosts.cu — per-host statistics on sm_100a.
//
// The reference keys every Forward flow's RateHistogram by (site << 32 |
// host) (reduce_slice, rate_engine.cpp:216-239), merges the per-thread
// histograms in a std::map and emits SiteResult::hosts[host] =
// stats_from(hist) (finalize, rate_engine.cpp:272-289). Paths are relative to
// /root/reference/proj/core/src.
//
// Here K2 (hosts mode) logs each Forward flow's site, bucket, host, octets
// and duration (H1 recomputes the f64 rate and exact micro-bps, rate.cuh);
// at finalize this post-pass turns the log into the reference's rows without
// any per-host histogram storage:
//   H0  flat offsets: exclusive scan of the per-warp log counts;
//   H1  give every (site, host) key a slot: a dense id from the registry's
//       /16 directory when its non-empty /16 blocks allow (a host lies in a
//       registered /24), else an open-addressing table sized by
//       min(flows, 256 * /24 entries); accumulate the u128 micro-bps sum, min
//       and max per slot (through a per-CTA shared table for the hot slots);
//       flatten (slot, bucket) per flow;
//   H2  collect the distinct keys, radix-sort them: row = rank in (site,
//       host) order, i.e. the std::map's iteration order; every flow's slot
//       becomes its row;
//   H3  the exact lower median per row (RateHistogram::median_bps,
//       rate_engine.cpp:42-58): with rows * 628 B <= 64 MB, the sites'
//       two-round scheme (coarse counts per (super-bucket, row), each row's
//       median super-bucket, that super-bucket's 64 fine counts; all
//       L2-resident, warp-aggregated); otherwise a radix sort of the
//       row << 14 | bucket keys, where the median is the run's element
//       (count + 1) / 2 - 1;
//   H5  per row: count, clamp into [min, max], avg as the host rounds it
//       (stats_from, :242-253).
// Histograms (dense or sparse) are built from the per-flow (row, bucket)
// arrays only when asked for. Across contexts (gnm_hosts_*), H0..H2 run per
// context, the rows become the union of every context's keys, and H3/H5 run
// on partials the caller all-reduces (hosts_global_*).
#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_run_length_encode.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "hosts.cuh"
#include "rate.cuh"

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

// The post-pass kernels' dynamic shared-memory limits, set once per device
// (cudaFuncSetAttribute costs host time on every call otherwise).
cudaError_t hosts_attributes(int device);

// H0, one block: exclusive scans of the per-warp-region log counts (flow
// offsets `off`) and of their H1 work items (non-empty chunks of kInsChunk
// entries, `ioff`); out[0] = total flows, out[2 + k] = work items of slice k
// (regions [slice_off[k], slice_off[k + 1]) ).
constexpr uint32_t kOffBlock = 1024;
template <uint32_t kChunk>
__global__ void __launch_bounds__(kOffBlock) h_offsets(const unsigned int* __restrict__ counts, uint32_t n,
                                                       uint32_t* __restrict__ off, uint32_t* __restrict__ ioff,
                                                       const uint32_t* __restrict__ slice_off, uint32_t n_slices,
                                                       unsigned long long* __restrict__ out) {
    __shared__ unsigned long long wsum[kOffBlock / 32];
    __shared__ uint32_t total_items;
    const uint32_t t = threadIdx.x, lane = t & 31u, warp = t >> 5;
    const uint32_t per = (n + kOffBlock - 1) / kOffBlock;
    const uint32_t a = min(n, t * per), b = min(n, a + per);
    uint32_t f = 0, it = 0;
    for (uint32_t r = a; r < b; ++r) {
        const uint32_t c = counts[r];
        f += c;
        it += (c + kChunk - 1) / kChunk;
    }
    // (flows, items) packed in one u64: flows < 2^32, items < 2^32
    unsigned long long v = static_cast<unsigned long long>(it) << 32 | f, x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xFFFFFFFFu, x, d);
        if (lane >= static_cast<uint32_t>(d)) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    if (warp == 0) {
        unsigned long long w = wsum[lane];
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xFFFFFFFFu, w, d);
            if (lane >= static_cast<uint32_t>(d)) w += y;
        }
        wsum[lane] = w; // inclusive over warps
        if (lane == 31) {
            out[0] = static_cast<uint32_t>(w);
            total_items = static_cast<uint32_t>(w >> 32);
        }
    }
    __syncthreads();
    unsigned long long e = x - v + (warp ? wsum[warp - 1] : 0ull); // exclusive prefix of this thread
    uint32_t fo = static_cast<uint32_t>(e), io = static_cast<uint32_t>(e >> 32);
    for (uint32_t r = a; r < b; ++r) {
        const uint32_t c = counts[r];
        off[r] = fo;
        ioff[r] = io;
        fo += c;
        io += (c + kChunk - 1) / kChunk;
    }
    __syncthreads(); // ioff written by the block is visible to the block
    for (uint32_t k = t; k < n_slices; k += kOffBlock) {
        const uint32_t s0 = slice_off[k], s1 = k + 1 < n_slices ? slice_off[k + 1] : n;
        out[2 + k] = (s1 < n ? ioff[s1] : total_items) - (s0 < n ? ioff[s0] : total_items);
    }
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

// H1, warp per work item (a non-empty chunk of kInsChunk entries of one
// warp region, numbered by h_offsets); each lane takes 4 consecutive entries
// per step (LDG.128 on the u32 columns) and the four table probes are issued
// before any is resolved.
// acc[slot] = {limb0, limb1, limb2, ~min bits, max bits} in L2 (zero at
// start: the min is kept complemented). Heavy hosts would serialise on their
// slot's L2 atomics, so each CTA folds flows into a shared table of kAgg
// entries first (one CTA of 1024 threads per SM, 192 KB); a flow whose slot
// has no entry goes to L2 directly. The table starts with the batch's hot
// slots (h_hot_sample / h_hot_pick: per entry the most frequent sampled slot
// hashing to it); an entry left empty goes to the first slot hashed to it.
// An entry keeps micro-bps below 2^48 as three 16-bit limbs in u32 counters
// (native, non-returning shared atomics). A CTA takes a contiguous range of
// at most kInsItemsPerCta work items of at most kInsChunk flows, i.e. fewer
// than 2^16 adds per limb, so no counter can wrap and no add has to return
// its value. Per-entry f32 bounds (rounded outward) filter the L2 min/max
// reductions: a stale bound only costs an extra one.
// Dense ids: the slot is computed, not probed; whether it is occupied is
// read back from its max-rate accumulator (every flow's rate is > 0), and
// its key is rebuilt from the id in h_collect_dense -- no per-flow key
// traffic at all.
#ifndef GNM_INS_BLOCK
#define GNM_INS_BLOCK 1024
#endif
constexpr uint32_t kInsBlock = GNM_INS_BLOCK;
#ifndef GNM_INS_AGG_BITS
#define GNM_INS_AGG_BITS 13
#endif
constexpr uint32_t kAggBits = GNM_INS_AGG_BITS;
constexpr uint32_t kAgg = 1u << kAggBits;
// GNM_INS_EXACT: the entry keeps the exact min/max rate bits (u64, moved by
// shared CAS loops, which fire only when the bound improves) and reduces them
// into L2 once at the flush, instead of f32 filters that reduce every
// improvement as it happens (~2 ln k reductions for k flows of the entry).
#ifndef GNM_INS_EXACT
#define GNM_INS_EXACT 0
#endif
constexpr size_t kInsSmem = kAgg * (GNM_INS_EXACT ? 8 + 8 + 3 * 4 + 4 : 4 + 4 + 3 * 4 + 4); // 192 KB at 8192
#ifndef GNM_INS_CTAS_PER_SM
#define GNM_INS_CTAS_PER_SM 1
#endif
#ifndef GNM_INS_CHUNK
#define GNM_INS_CHUNK 512
#endif
constexpr uint32_t kInsChunk = GNM_INS_CHUNK;
constexpr uint32_t kInsItemsPerCta = 65535u / kInsChunk; // items * chunk < 2^16 adds per limb

__device__ __forceinline__ void red_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("red.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void red_max_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("red.global.max.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

struct AggSmem {
#if GNM_INS_EXACT
    unsigned long long* nmn; // ~(smallest rate bits) of the entry's flows in this CTA (0: none)
    unsigned long long* mx;  // largest rate bits (0: none)
#else
    float* mn; // >= the smallest rate this CTA reduced into L2 for the entry (+inf: none)
    float* mx; // <= the largest
#endif
    uint32_t* key;
    uint32_t* limb; // [3][kAgg]
};

__device__ __forceinline__ void agg_flush(const AggSmem& t, uint32_t e, unsigned long long* a) {
    const uint32_t x0 = atomicExch(t.limb + e, 0u), x1 = atomicExch(t.limb + kAgg + e, 0u);
    const uint32_t x2 = atomicExch(t.limb + 2 * kAgg + e, 0u);
    if (x0 | x1) red_u64(a + 0, static_cast<unsigned long long>(x0) + (static_cast<unsigned long long>(x1) << 16));
    if (x2) red_u64(a + 1, x2);
#if GNM_INS_EXACT
    if (const unsigned long long m = t.mx[e]) {
        red_max_u64(a + 3, t.nmn[e]);
        red_max_u64(a + 4, m);
    }
#endif
}

__device__ __forceinline__ uint32_t agg_entry(uint32_t slot) { return (slot * 2654435761u) >> (32 - kAggBits); }

// One flow's contribution (any lane, no warp-level grouping). An entry left
// empty by the preload (h_hot_pick) goes to the first slot hashed to it.
__device__ __forceinline__ void fold(uint32_t slot, unsigned long long lo, uint32_t hi, unsigned long long rate,
                                     const AggSmem& t, unsigned long long* acc) {
    unsigned long long* a = acc + static_cast<size_t>(slot) * 5;
    const uint32_t e = agg_entry(slot);
    uint32_t cur = t.key[e];
    if (cur == 0xFFFFFFFFu) cur = atomicCAS(t.key + e, 0xFFFFFFFFu, slot);
    if ((cur == 0xFFFFFFFFu || cur == slot) && hi == 0 && lo < (1ull << 48)) {
        atomicAdd(t.limb + e, static_cast<uint32_t>(lo) & 0xFFFFu);
        atomicAdd(t.limb + kAgg + e, static_cast<uint32_t>(lo) >> 16);
        atomicAdd(t.limb + 2 * kAgg + e, static_cast<uint32_t>(lo >> 32));
#if GNM_INS_EXACT
        if (~rate > t.nmn[e]) atomicMax(t.nmn + e, ~rate);
        if (rate > t.mx[e]) atomicMax(t.mx + e, rate);
#else
        // Bounds move by shared atomics on the f32 bits (positive floats
        // order as integers), only after their reduction was issued.
        const double r = __longlong_as_double(static_cast<long long>(rate));
        if (r < static_cast<double>(t.mn[e])) {
            red_max_u64(a + 3, ~rate);
            atomicMin(reinterpret_cast<int*>(t.mn + e), __float_as_int(__double2float_ru(r)));
        }
        if (r > static_cast<double>(t.mx[e])) {
            red_max_u64(a + 4, rate);
            atomicMax(reinterpret_cast<int*>(t.mx + e), __float_as_int(__double2float_rd(r)));
        }
#endif
    } else {
        red_u64(a + 0, lo & 0xFFFFFFFFull);
        red_u64(a + 1, lo >> 32);
        if (hi) red_u64(a + 2, hi); // micro-bps >= 2^64: rare
        red_max_u64(a + 3, ~rate);
        red_max_u64(a + 4, rate);
    }
}

// Dense id of a host whose /16 is in the registry directory (its /24 is
// registered): rank of the /16 << 16 | its low 16 bits, bit-reversed so
// that the hosts of one /24 (one site, often hot) land 256 entries apart
// instead of in the same L2 sectors.
__device__ __forceinline__ uint32_t dense_id(uint32_t host, const uint2* __restrict__ dir) {
    const uint32_t d = host >> 16;
    const uint2 pr = __ldg(dir + (d >> 5));
    return (pr.y + __popc(pr.x & ((1u << (d & 31u)) - 1u))) << 16 | __brev(host << 16);
}

// Hot-slot preload (dense ids). Which hosts are heavy is a property of the
// batch, not of a CTA's share of it, so instead of first-come entries (most
// taken by hosts a CTA sees once) every CTA's table starts with the same
// set: the slots of a sample of the log, counted, and per table entry the
// most frequent sampled slot hashing to it.
// The sample is the first `take` entries of every warp region: K2's warps
// log the flows of tiles spread over the whole batch, so the regions' heads
// are a sample of the batch, read with coalesced loads. Heavy slots recur
// within a CTA's regions, so each CTA counts them in a shared table first
// (first come; a slot without an entry goes to L2 directly): plain
// per-sample L2 atomics serialise on the hottest slots' counters.
constexpr uint32_t kSampleAggBits = 12, kSampleAgg = 1u << kSampleAggBits;
constexpr uint32_t kSampleHead = 512; // entries per region (one slice)
__global__ void __launch_bounds__(1024) h_hot_sample(DevLog L, const unsigned int* __restrict__ counts,
                                                     const uint2* __restrict__ dir, uint32_t take,
                                                     uint32_t* __restrict__ cnt) {
    __shared__ uint32_t skey[kSampleAgg], scnt[kSampleAgg];
    for (uint32_t i = threadIdx.x; i < kSampleAgg; i += blockDim.x) {
        skey[i] = 0xFFFFFFFFu;
        scnt[i] = 0;
    }
    __syncthreads();
    const uint32_t r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31u;
    if (r < L.regions) {
        const uint32_t n = min(__ldg(counts + r), take);
        const unsigned int* h = L.hosts + static_cast<size_t>(r) * L.warp_cap;
        for (uint32_t i = lane * 4; i < n; i += 128) {
            const uint4 x = __ldcs(reinterpret_cast<const uint4*>(h + i));
            const uint32_t hs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                if (i + q >= n) break;
                const uint32_t sl = dense_id(hs[q], dir);
                const uint32_t e = (sl * 2654435761u) >> (32 - kSampleAggBits);
                uint32_t cur = skey[e];
                if (cur == 0xFFFFFFFFu) cur = atomicCAS(skey + e, 0xFFFFFFFFu, sl);
                if (cur == 0xFFFFFFFFu || cur == sl) atomicAdd(scnt + e, 1u);
                else atomicAdd(cnt + sl, 1u);
            }
        }
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < kSampleAgg; i += blockDim.x)
        if (scnt[i]) atomicAdd(cnt + skey[i], scnt[i]);
}

__global__ void h_hot_pick(const uint32_t* __restrict__ cnt, uint32_t cap, unsigned long long* __restrict__ table) {
    for (uint32_t sl = blockIdx.x * blockDim.x + threadIdx.x; sl < cap; sl += gridDim.x * blockDim.x) {
        const uint32_t c = cnt[sl];
        if (c >= 2) atomicMax(table + agg_entry(sl), static_cast<unsigned long long>(c) << 32 | sl);
    }
}

template <bool kDense, bool kPre>
__global__ void __launch_bounds__(kInsBlock, GNM_INS_CTAS_PER_SM) h_insert(
    DevLog L, const unsigned int* __restrict__ counts, const uint32_t* __restrict__ off,
    const uint32_t* __restrict__ ioff, uint32_t items, const uint2* __restrict__ dir,
    unsigned long long* keys, uint32_t mask, int shift, unsigned long long* __restrict__ acc,
    uint32_t* __restrict__ slot_of, uint32_t* __restrict__ bk, const unsigned long long* __restrict__ hot) {
    extern __shared__ __align__(16) unsigned char h_smem[];
    AggSmem t;
#if GNM_INS_EXACT
    t.nmn = reinterpret_cast<unsigned long long*>(h_smem);
    t.mx = t.nmn + kAgg;
    t.key = reinterpret_cast<uint32_t*>(t.mx + kAgg);
#else
    t.mn = reinterpret_cast<float*>(h_smem);
    t.mx = t.mn + kAgg;
    t.key = reinterpret_cast<uint32_t*>(t.mx + kAgg);
#endif
    t.limb = t.key + kAgg;
    for (uint32_t i = threadIdx.x; i < kAgg; i += blockDim.x) {
#if GNM_INS_EXACT
        t.nmn[i] = 0;
        t.mx[i] = 0;
#else
        t.mn[i] = __int_as_float(0x7F800000); // +inf
        t.mx[i] = 0.0f;
#endif
        if constexpr (kPre) {
            const unsigned long long h = hot[i];
            t.key[i] = h ? static_cast<uint32_t>(h) : 0xFFFFFFFFu;
        } else {
            t.key[i] = 0xFFFFFFFFu;
        }
#pragma unroll
        for (int f = 0; f < 3; ++f) t.limb[f * kAgg + i] = 0;
    }
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31u;
    // this CTA's contiguous range of the slice's `items` work items (the
    // non-empty chunks, numbered by ioff; <= kInsItemsPerCta, see above)
    const uint32_t ibase = ioff[0];
    const uint32_t i0 = static_cast<uint32_t>(static_cast<uint64_t>(items) * blockIdx.x / gridDim.x);
    const uint32_t i1 = static_cast<uint32_t>(static_cast<uint64_t>(items) * (blockIdx.x + 1) / gridDim.x);
    uint32_t r = 0;
    {
        // the region of this warp's first item: the last r with ioff[r] <= item
        const uint32_t w0 = ibase + i0 + (threadIdx.x >> 5);
        uint32_t lo = 0, hi = L.regions; // ioff[lo] <= w0 < ioff[hi] (ioff[regions] = end)
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (__ldg(ioff + mid) <= w0) lo = mid;
            else hi = mid;
        }
        r = lo;
    }
    for (uint32_t w = i0 + (threadIdx.x >> 5); w < i1; w += blockDim.x >> 5) {
        while (r + 1 < L.regions && __ldg(ioff + r + 1) <= ibase + w) ++r;
        const uint32_t c0 = (ibase + w - __ldg(ioff + r)) * kInsChunk;
        const uint32_t n = min(counts[r], c0 + kInsChunk);
        const uint32_t base = off[r];
        const size_t rb = static_cast<size_t>(r) * L.warp_cap;
        for (uint32_t i = c0 + lane * 4; i < n; i += 128) {
            const size_t pos = rb + i;
            const uint4 x = __ldcs(reinterpret_cast<const uint4*>(L.entries + pos));
            const uint4 hst = __ldcs(reinterpret_cast<const uint4*>(L.hosts + pos));
            const uint4 bb = L.buckets ? __ldcs(reinterpret_cast<const uint4*>(L.buckets + pos)) : make_uint4(0, 0, 0, 0);
            const uint4 oc = __ldcs(reinterpret_cast<const uint4*>(L.octs + pos));
            const ulonglong2 du01 = __ldcs(reinterpret_cast<const ulonglong2*>(L.durs + pos));
            const ulonglong2 du23 = __ldcs(reinterpret_cast<const ulonglong2*>(L.durs + pos + 2));
            const uint32_t xs[4] = {x.x, x.y, x.z, x.w}, hs[4] = {hst.x, hst.y, hst.z, hst.w};
            const uint32_t bs[4] = {bb.x, bb.y, bb.z, bb.w};
            // flow_rate and rate_ubps_of again (rate.cuh: the same arithmetic
            // as K2, so the same bits), from the logged octets and duration
            const uint32_t os[4] = {oc.x, oc.y, oc.z, oc.w};
            const unsigned long long ds[4] = {du01.x, du01.y, du23.x, du23.y};
            unsigned long long los[4], rts[4];
            uint32_t us[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const double rate = flow_rate_dev(os[q], ds[q]);
                uint64_t lo, hi;
                ubps_of(os[q], ds[q], rate, lo, hi);
                los[q] = lo;
                us[q] = static_cast<uint32_t>(hi);
                rts[q] = static_cast<unsigned long long>(__double_as_longlong(rate));
            }
            unsigned long long key[4], first[4];
            uint32_t h0[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) { // dense ids, or issue the four first probes
                const uint32_t site = L.buckets ? xs[q] : xs[q] >> kLogSiteShift;
                key[q] = static_cast<unsigned long long>(site) << 32 | hs[q];
                if constexpr (kDense) {
                    h0[q] = dense_id(hs[q], dir);
                    first[q] = 0;
                } else {
                    h0[q] = static_cast<uint32_t>((key[q] * 0x9E3779B97F4A7C15ull) >> shift) & mask;
                    first[q] = i + q < n ? keys[h0[q]] : 0ull;
                }
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                if (i + q >= n) break;
                uint32_t slot;
                if constexpr (kDense) {
                    slot = h0[q];
                } else {
                    slot = first[q] == key[q] ? h0[q] : insert_key(keys, mask, shift, key[q]);
                }
                slot_of[base + i + q] = slot;
                bk[base + i + q] = L.buckets ? bs[q] : xs[q] & kBucketMask;
                fold(slot, los[q], us[q], rts[q], t, acc);
            }
        }
    }
    __syncthreads();
    for (uint32_t e = threadIdx.x; e < kAgg; e += blockDim.x) {
        const uint32_t slot = t.key[e];
        if (slot == 0xFFFFFFFFu) continue;
        unsigned long long* a = acc + static_cast<size_t>(slot) * 5;
        agg_flush(t, e, a);
        // the cached bounds were reduced into L2 when they were set
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

// Dense ids: the /16 block of each rank (the inverse of the directory's
// rank-of-/16), for rebuilding a slot's host address.
__global__ void h_prefix_of_rank(const uint2* __restrict__ dir, uint32_t* __restrict__ prefix) {
    const uint32_t d = blockIdx.x * blockDim.x + threadIdx.x;
    if (d >= 65536u) return;
    const uint2 pr = __ldg(dir + (d >> 5));
    if ((pr.x >> (d & 31u)) & 1u) prefix[pr.y + __popc(pr.x & ((1u << (d & 31u)) - 1u))] = d;
}

// H2a (dense ids): the occupied slots (max-rate accumulator set: every
// Forward rate is > 0) and their keys rebuilt from the id: host = the /16 of
// the rank | the un-reversed low 16 bits, site = the registry's /24 entry
// (words: the device table, site values masked by site_mask).
__global__ void __launch_bounds__(256) h_collect_dense(const unsigned long long* __restrict__ acc, uint32_t cap,
                                                       const uint32_t* __restrict__ prefix,
                                                       const uint32_t* __restrict__ words, uint32_t site_mask,
                                                       unsigned long long* __restrict__ hk, uint32_t* __restrict__ hs,
                                                       unsigned int* __restrict__ n_out) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint2* dir = reinterpret_cast<const uint2*>(words);
    for (uint32_t base = blockIdx.x * blockDim.x; base < cap; base += gridDim.x * blockDim.x) {
        const uint32_t s = base + threadIdx.x;
        const bool occ = s < cap && acc[static_cast<size_t>(s) * 5 + 4] != 0ull;
        unsigned long long k = 0;
        if (occ) {
            const uint32_t ip = __ldg(prefix + (s >> 16)) << 16 | (__brev(s & 0xFFFFu) >> 16);
            const uint32_t d = ip >> 16;
            const uint2 pr = __ldg(dir + (d >> 5));
            const uint32_t node = __ldg(words + 4096u + pr.y + __popc(pr.x & ((1u << (d & 31u)) - 1u)));
            const uint32_t v = (node & 0x80000000u) ? node & 0x7FFFFFFFu : __ldg(words + node + ((ip >> 8) & 0xFFu));
            k = static_cast<unsigned long long>(v & site_mask) << 32 | ip;
        }
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

// ---- per-row exact lower median, two rounds (rows * 628 B L2-resident) -------
// The sites' scheme (kernels.cuh): coarse counts per (super-bucket, row),
// super-bucket-major; each row's median super-bucket and the median's rank
// in it; the fine counts of that super-bucket only. Lanes of a warp that
// carry the same (row, super-bucket) or (row, bucket) add once, together.
constexpr uint32_t kCoarseH = 157, kFineH = 64;
constexpr size_t kTwoRoundBytes = 64ull << 20;

// Hot (row, super-bucket) pairs would serialise on one L2 counter, so each
// CTA counts into a shared table first (first come, first served; a pair
// whose entry is taken goes to L2 directly) and flushes it once.
#ifndef GNM_HC_AGG_BITS
#define GNM_HC_AGG_BITS 13
#endif
#ifndef GNM_HC_CTAS_PER_SM
#define GNM_HC_CTAS_PER_SM 3
#endif
constexpr uint32_t kCoarseAggBits = GNM_HC_AGG_BITS;
constexpr uint32_t kCoarseAgg = 1u << kCoarseAggBits;
constexpr size_t kCoarseSmem = static_cast<size_t>(kCoarseAgg) * 8;
// With `rank`, also turns every flow's slot into its row (in place).
// Each thread takes four consecutive flows per step (LDG.128 of the slot and
// bucket columns) and issues their four rank gathers before using any: the
// gathers are dependent, L2-latency-bound loads.
__device__ __forceinline__ void coarse_one(uint32_t r, uint32_t sb, uint32_t n_rows, uint32_t* tkey, uint32_t* tcnt,
                                           uint32_t* __restrict__ coarse) {
    const uint32_t key = r << 8 | sb; // rows < 2^24 on this path (rows * 628 B <= 64 MB)
    const uint32_t e = (key * 2654435761u) >> (32 - kCoarseAggBits);
    uint32_t cur = tkey[e];
    if (cur == 0xFFFFFFFFu) cur = atomicCAS(tkey + e, 0xFFFFFFFFu, key);
    if (cur == 0xFFFFFFFFu || cur == key)
        atomicAdd(tcnt + e, 1u);
    else
        atomicAdd(coarse + static_cast<size_t>(sb) * n_rows + r, 1u);
}

// kPack (local two-round path, rows < 2^18): instead of writing every
// flow's row over its slot, write row << 14 | bucket over its bucket, so
// h_fine (and any histogram export) reads one u32 column per flow, not two.
template <bool kPack>
__global__ void __launch_bounds__(512) h_coarse(uint32_t* __restrict__ row, uint32_t* __restrict__ bk,
                                                uint32_t n, uint32_t n_rows, const unsigned long long* __restrict__ rank,
                                                uint32_t* __restrict__ coarse) {
    extern __shared__ uint32_t hc_smem[];
    uint32_t* tkey = hc_smem;
    uint32_t* tcnt = hc_smem + kCoarseAgg;
    for (uint32_t i = threadIdx.x; i < kCoarseAgg; i += blockDim.x) {
        tkey[i] = 0xFFFFFFFFu;
        tcnt[i] = 0;
    }
    __syncthreads();
    const uint32_t n4 = n / 4; // row and bk are cudaMallocAsync bases: 16-byte aligned
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n4; j += gridDim.x * blockDim.x) {
        uint4 rw = __ldcs(reinterpret_cast<const uint4*>(row) + j);
        const uint4 bw = __ldcs(reinterpret_cast<const uint4*>(bk) + j);
        if (rank) {
            const unsigned long long a = rank[rw.x], b = rank[rw.y], c = rank[rw.z], d = rank[rw.w];
            rw = make_uint4(static_cast<uint32_t>(a), static_cast<uint32_t>(b), static_cast<uint32_t>(c),
                            static_cast<uint32_t>(d));
            if constexpr (kPack)
                __stcs(reinterpret_cast<uint4*>(bk) + j,
                       make_uint4(rw.x << kBucketBits | bw.x, rw.y << kBucketBits | bw.y, rw.z << kBucketBits | bw.z,
                                  rw.w << kBucketBits | bw.w));
            else
                __stcs(reinterpret_cast<uint4*>(row) + j, rw);
        }
        coarse_one(rw.x, bw.x >> 6, n_rows, tkey, tcnt, coarse);
        coarse_one(rw.y, bw.y >> 6, n_rows, tkey, tcnt, coarse);
        coarse_one(rw.z, bw.z >> 6, n_rows, tkey, tcnt, coarse);
        coarse_one(rw.w, bw.w >> 6, n_rows, tkey, tcnt, coarse);
    }
    for (uint32_t j = n4 * 4 + blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        const uint32_t r = rank ? static_cast<uint32_t>(rank[row[j]]) : row[j];
        const uint32_t b = bk[j];
        if (rank) {
            if constexpr (kPack) bk[j] = r << kBucketBits | b;
            else row[j] = r;
        }
        coarse_one(r, b >> 6, n_rows, tkey, tcnt, coarse);
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < kCoarseAgg; i += blockDim.x)
        if (tcnt[i]) atomicAdd(coarse + static_cast<size_t>(tkey[i] & 0xFFu) * n_rows + (tkey[i] >> 8), tcnt[i]);
}

__global__ void h_msb(const uint32_t* __restrict__ coarse, uint32_t n_rows, uint32_t* __restrict__ msb,
                      uint32_t* __restrict__ mrank, uint32_t* __restrict__ cnt) {
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n_rows; r += gridDim.x * blockDim.x) {
        uint32_t total = 0;
        for (uint32_t sb = 0; sb < kCoarseH; ++sb) total += coarse[static_cast<size_t>(sb) * n_rows + r];
        const uint32_t target = (total + 1) / 2; // RateHistogram::median_bps (rate_engine.cpp:47)
        uint32_t cum = 0, m = 0, k = 0;
        for (uint32_t sb = 0; sb < kCoarseH; ++sb) {
            const uint32_t c = coarse[static_cast<size_t>(sb) * n_rows + r];
            if (cum + c >= target) {
                m = sb;
                k = target - cum;
                break;
            }
            cum += c;
        }
        msb[r] = m;
        mrank[r] = k;
        cnt[r] = total;
    }
}

// Four consecutive flows per lane per step, their msb gathers issued
// together; lanes carrying the same (row, bucket) add once.
template <bool kPacked> // bk holds row << 14 | bucket (row unused)
__global__ void __launch_bounds__(256) h_fine(const uint32_t* __restrict__ row, const uint32_t* __restrict__ bk,
                                              uint32_t n, const uint32_t* __restrict__ msb,
                                              uint32_t* __restrict__ fine) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t n4 = (n + 3) / 4;
    for (uint32_t base = blockIdx.x * blockDim.x; base < n4; base += gridDim.x * blockDim.x) {
        const uint32_t j = base + threadIdx.x;
        uint32_t rs[4] = {0, 0, 0, 0}, bs[4] = {0, 0, 0, 0}, ms[4];
        bool in[4] = {false, false, false, false};
        if (4 * j + 3 < n) {
            const uint4 bw = __ldcs(reinterpret_cast<const uint4*>(bk) + j);
            bs[0] = bw.x, bs[1] = bw.y, bs[2] = bw.z, bs[3] = bw.w;
            if constexpr (!kPacked) {
                const uint4 rw = __ldcs(reinterpret_cast<const uint4*>(row) + j);
                rs[0] = rw.x, rs[1] = rw.y, rs[2] = rw.z, rs[3] = rw.w;
            }
            in[0] = in[1] = in[2] = in[3] = true;
        } else {
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (4 * j + q < n) {
                    if constexpr (!kPacked) rs[q] = row[4 * j + q];
                    bs[q] = bk[4 * j + q];
                    in[q] = true;
                }
        }
        if constexpr (kPacked) {
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                rs[q] = bs[q] >> kBucketBits;
                bs[q] &= kBucketMask;
            }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) ms[q] = in[q] ? __ldg(msb + rs[q]) : 0xFFFFFFFFu;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const bool hit = (bs[q] >> 6) == ms[q];
            const unsigned long long key =
                hit ? (static_cast<unsigned long long>(rs[q]) << 8 | (bs[q] & 63u)) : ~0ull;
            const unsigned m = __match_any_sync(0xFFFFFFFFu, key);
            if (hit && lane == static_cast<uint32_t>(__ffs(m) - 1))
                atomicAdd(fine + static_cast<size_t>(rs[q]) * kFineH + (bs[q] & 63u), __popc(m));
        }
    }
}

// H5 (two-round), thread per row: the exact bucket from the fine counts.
__global__ void h_final2(const unsigned long long* __restrict__ acc, const uint32_t* __restrict__ cnt,
                         const uint32_t* __restrict__ msb, const uint32_t* __restrict__ mrank,
                         const uint32_t* __restrict__ fine, const unsigned long long* __restrict__ hk_sorted,
                         const uint32_t* __restrict__ hs_sorted, uint32_t n_rows, gnm_host_stats* __restrict__ rows) {
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n_rows; r += gridDim.x * blockDim.x) {
        const uint32_t* f = fine + static_cast<size_t>(r) * kFineH;
        uint32_t cum = 0, k = msb[r] * kFineH + kFineH - 1;
        const uint32_t want = mrank[r];
        for (uint32_t q = 0; q < kFineH; ++q) {
            cum += f[q];
            if (cum >= want) {
                k = msb[r] * kFineH + q;
                break;
            }
        }
        const unsigned long long* a = acc + static_cast<size_t>(hs_sorted[r]) * 5;
        const unsigned __int128 u = static_cast<unsigned __int128>(a[0]) +
                                    (static_cast<unsigned __int128>(a[1]) << 32) +
                                    (static_cast<unsigned __int128>(a[2]) << 64);
        const double mn = __longlong_as_double(static_cast<long long>(~a[3]));
        const double mx = __longlong_as_double(static_cast<long long>(a[4]));
        double med = median_of_bucket(k);
        med = med < mn ? mn : (mx < med ? mx : med);
        gnm_host_stats o;
        o.site = static_cast<uint32_t>(hk_sorted[r] >> 32);
        o.host = static_cast<uint32_t>(hk_sorted[r]);
        o.flow_count = cnt[r];
        o.rate_ubps_lo = static_cast<uint64_t>(u);
        o.rate_ubps_hi = static_cast<uint64_t>(u >> 64);
        o.min_bps = mn;
        o.max_bps = mx;
        o.avg_bps = avg_of(o.rate_ubps_lo, o.rate_ubps_hi, o.flow_count);
        o.median_bps = med;
        rows[r] = o;
    }
}

// ---- per-row median from sorted (row, bucket) keys (many rows) -------------------
template <typename K>
__global__ void h_keys(const uint32_t* __restrict__ row, const uint32_t* __restrict__ bk, uint32_t n,
                       K* __restrict__ sk, bool packed) {
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x)
        sk[j] = packed ? static_cast<K>(bk[j]) : static_cast<K>(row[j]) << kBucketBits | bk[j];
}

// h_to_rows + h_keys in one pass: every flow's slot becomes its row (in
// place) and its (row, bucket) sort key is written.
template <typename K>
__global__ void h_rows_keys(uint32_t* __restrict__ row, const uint32_t* __restrict__ bk, uint32_t n,
                            const unsigned long long* __restrict__ rank, K* __restrict__ sk) {
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        const uint32_t r = static_cast<uint32_t>(rank[row[j]]);
        row[j] = r;
        sk[j] = static_cast<K>(r) << kBucketBits | bk[j];
    }
}

// start[row] = first position of the row's run; start[n_rows] = n.
template <typename K>
__global__ void h_starts(const K* __restrict__ sk, uint32_t n, uint32_t n_rows, uint32_t* __restrict__ start) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const K row = sk[i] >> kBucketBits;
        if (i == 0 || (sk[i - 1] >> kBucketBits) != row) start[row] = i;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) start[n_rows] = n;
}

// H5 (sorted), thread per row: the lower median is the run's element
// (count + 1) / 2 - 1.
template <typename K>
__global__ void h_final(const unsigned long long* __restrict__ acc, const uint32_t* __restrict__ start,
                        const K* __restrict__ sk, const unsigned long long* __restrict__ hk_sorted,
                        const uint32_t* __restrict__ hs_sorted, uint32_t n_rows,
                        gnm_host_stats* __restrict__ rows) {
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n_rows; r += gridDim.x * blockDim.x) {
        const unsigned long long* a = acc + static_cast<size_t>(hs_sorted[r]) * 5;
        const uint32_t s0 = start[r];
        const uint64_t cnt = start[r + 1] - s0;
        const unsigned __int128 u = static_cast<unsigned __int128>(a[0]) +
                                    (static_cast<unsigned __int128>(a[1]) << 32) +
                                    (static_cast<unsigned __int128>(a[2]) << 64);
        const uint32_t k = static_cast<uint32_t>(sk[s0 + (cnt + 1) / 2 - 1] & kBucketMask);
        const double mn = __longlong_as_double(static_cast<long long>(~a[3]));
        const double mx = __longlong_as_double(static_cast<long long>(a[4]));
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

__global__ void h_hist(const uint32_t* __restrict__ row, const uint32_t* __restrict__ bk, uint64_t n,
                       uint32_t* __restrict__ dense, bool packed) {
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint32_t b = bk[i];
        const uint32_t r = packed ? b >> kBucketBits : row[i];
        atomicAdd(dense + static_cast<size_t>(r) * kBuckets + (b & kBucketMask), 1u);
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

// Stream-ordered temporaries released when the scope ends, on every path.
struct Scratch {
    cudaStream_t s;
    std::vector<void*> held;
    explicit Scratch(cudaStream_t st) : s(st) {}
    Scratch(const Scratch&) = delete;
    Scratch& operator=(const Scratch&) = delete;
    ~Scratch() {
        for (void* q : held) cudaFreeAsync(q, s);
    }
    template <typename T>
    cudaError_t get(T** p, size_t n) {
        const cudaError_t e = dalloc(p, n, s);
        if (e == cudaSuccess) held.push_back(*p);
        return e;
    }
};

// h.sorted: every flow's (row, bucket) key in (row, bucket) order.
// With `rank`, h.row_of still holds H1 slots and becomes rows on the way.
template <typename K>
cudaError_t sort_keys(int device, HostRows& h, cudaStream_t s, const unsigned long long* rank = nullptr) {
    Scratch tmp_(s);
    const uint32_t n = static_cast<uint32_t>(h.n_flows);
    K *sk = nullptr, *sk2 = nullptr;
    HCK(tmp_.get(&sk, n));
    HCK(dalloc(&sk2, n, s));
    h.sorted = sk2; // owned by `h` from here (free_hosts)
    if (rank)
        h_rows_keys<K><<<grid_for(device, n, 256), 256, 0, s>>>(h.row_of, h.bkt, n, rank, sk);
    else
        h_keys<K><<<grid_for(device, n, 256), 256, 0, s>>>(h.row_of, h.bkt, n, sk, h.packed);
    HCK(cudaGetLastError());
    const int end_bit = static_cast<int>(kBucketBits) + std::max(1, bits_for(h.n_rows));
    size_t tb = 0;
    HCK(cub::DeviceRadixSort::SortKeys(nullptr, tb, sk, sk2, n, 0, end_bit, s));
    unsigned char* tmp = nullptr;
    HCK(tmp_.get(&tmp, tb));
    return cub::DeviceRadixSort::SortKeys(tmp, tb, sk, sk2, n, 0, end_bit, s);
}

cudaError_t ensure_sorted(int device, HostRows& h, cudaStream_t s) {
    if (h.sorted || h.n_flows == 0) return cudaSuccess;
    return h.key64 ? sort_keys<unsigned long long>(device, h, s) : sort_keys<uint32_t>(device, h, s);
}

template <typename K>
cudaError_t finish_sorted(int device, HostRows& h, const unsigned long long* rank, const unsigned long long* acc,
                          const unsigned long long* hk_sorted, const uint32_t* hs_sorted, cudaStream_t s) {
    Scratch tmp_(s);
    if (!h.sorted && h.n_flows) HCK(sort_keys<K>(device, h, s, rank));
    const uint32_t n = static_cast<uint32_t>(h.n_flows);
    uint32_t* start = nullptr;
    HCK(tmp_.get(&start, static_cast<size_t>(h.n_rows) + 1));
    const K* sk = static_cast<const K*>(h.sorted);
    h_starts<K><<<grid_for(device, n, 256), 256, 0, s>>>(sk, n, static_cast<uint32_t>(h.n_rows), start);
    HCK(cudaGetLastError());
    h_final<K><<<grid_for(device, h.n_rows, 128), 128, 0, s>>>(acc, start, sk, hk_sorted, hs_sorted,
                                                               static_cast<uint32_t>(h.n_rows), h.rows);
    return cudaGetLastError();
}

cudaError_t finish_two_round(int device, HostRows& h, const unsigned long long* rank, const unsigned long long* acc,
                             const unsigned long long* hk_sorted, const uint32_t* hs_sorted, cudaStream_t s) {
    Scratch tmp_(s);
    if ((reinterpret_cast<uintptr_t>(h.row_of) | reinterpret_cast<uintptr_t>(h.bkt)) & 15u)
        return cudaErrorMisalignedAddress; // h_coarse / h_fine read them as uint4
    const uint32_t n = static_cast<uint32_t>(h.n_flows), nr = static_cast<uint32_t>(h.n_rows);
    uint32_t *coarse = nullptr, *msb = nullptr, *mrank = nullptr, *cnt = nullptr, *fine = nullptr;
    HCK(tmp_.get(&coarse, static_cast<size_t>(nr) * kCoarseH));
    HCK(tmp_.get(&msb, nr));
    HCK(tmp_.get(&mrank, nr));
    HCK(tmp_.get(&cnt, nr));
    HCK(tmp_.get(&fine, static_cast<size_t>(nr) * kFineH));
    HCK(cudaMemsetAsync(coarse, 0, static_cast<size_t>(nr) * kCoarseH * 4, s));
    HCK(cudaMemsetAsync(fine, 0, static_cast<size_t>(nr) * kFineH * 4, s));
    HCK(hosts_attributes(device));
    int sms = 0;
    HCK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    const uint32_t cg = static_cast<uint32_t>(std::max<uint64_t>(
        1, std::min<uint64_t>((n + 511) / 512, static_cast<uint64_t>(sms) * GNM_HC_CTAS_PER_SM)));
    // rows < 2^18 here (rows * 628 B <= 64 MB): pack them into the bucket column
    const bool pack = rank && nr < (1u << (32 - kBucketBits));
    if (pack) h_coarse<true><<<cg, 512, kCoarseSmem, s>>>(h.row_of, h.bkt, n, nr, rank, coarse);
    else h_coarse<false><<<cg, 512, kCoarseSmem, s>>>(h.row_of, h.bkt, n, nr, rank, coarse);
    h.packed = pack;
    h_msb<<<grid_for(device, nr, 128), 128, 0, s>>>(coarse, nr, msb, mrank, cnt);
    if (pack) h_fine<true><<<grid_for(device, (n + 3) / 4, 256), 256, 0, s>>>(h.row_of, h.bkt, n, msb, fine);
    else h_fine<false><<<grid_for(device, (n + 3) / 4, 256), 256, 0, s>>>(h.row_of, h.bkt, n, msb, fine);
    h_final2<<<grid_for(device, nr, 128), 128, 0, s>>>(acc, cnt, msb, mrank, fine, hk_sorted, hs_sorted, nr, h.rows);
    return cudaGetLastError();
}

cudaError_t hosts_attributes(int device) {
    static std::atomic<uint64_t> done{0}; // one bit per device ordinal (< 64)
    const uint64_t bit = device >= 0 && device < 64 ? 1ull << device : 0ull;
    if (bit && (done.load(std::memory_order_acquire) & bit)) return cudaSuccess;
    HCK(cudaFuncSetAttribute(h_coarse<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kCoarseSmem)));
    HCK(cudaFuncSetAttribute(h_coarse<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kCoarseSmem)));
    HCK(cudaFuncSetAttribute(h_insert<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(kInsSmem)));
    HCK(cudaFuncSetAttribute(h_insert<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(kInsSmem)));
    done.fetch_or(bit, std::memory_order_release);
    return cudaSuccess;
}

} // namespace

cudaError_t build_hosts_local(int device, const HostSlice* slices, int n_slices, const unsigned int* counts,
                              size_t n_counts, uint64_t max_keys, uint32_t n_sites, const uint32_t* dir, uint32_t n16,
                              bool packed, HostRows& out, HostLocal& loc, cudaStream_t s) {
    free_hosts(out, s);
    free_local(loc, s);
    loc.ready = true;
    if (n_counts == 0) return cudaSuccess;
    Scratch tmp_(s);
    // H0: flat offsets of every warp region's entries, H1 work items per slice.
    uint32_t *off = nullptr, *ioff = nullptr, *slice_off = nullptr;
    unsigned long long* scal = nullptr; // [0] total flows, [1] distinct keys, [2 + k] items of slice k
    HCK(tmp_.get(&off, n_counts));
    HCK(tmp_.get(&ioff, n_counts));
    HCK(tmp_.get(&slice_off, n_slices));
    HCK(tmp_.get(&scal, 2 + n_slices));
    std::vector<uint32_t> h_slice_off(n_slices);
    for (int i = 0; i < n_slices; ++i) h_slice_off[i] = static_cast<uint32_t>(slices[i].count_off);
    HCK(cudaMemcpyAsync(slice_off, h_slice_off.data(), n_slices * 4, cudaMemcpyHostToDevice, s));
    HCK(cudaMemsetAsync(scal, 0, (2 + n_slices) * 8, s));
    h_offsets<kInsChunk><<<1, kOffBlock, 0, s>>>(counts, static_cast<uint32_t>(n_counts), off, ioff, slice_off,
                                                 static_cast<uint32_t>(n_slices), scal);
    std::vector<unsigned long long> h_scal(2 + n_slices, 0);
    HCK(cudaMemcpyAsync(h_scal.data(), scal, h_scal.size() * 8, cudaMemcpyDeviceToHost, s));
    HCK(cudaStreamSynchronize(s));
    const uint64_t n = h_scal[0];
    if (n == 0) return cudaSuccess;
    HCK(hosts_attributes(device));
    int sms = 0;
    HCK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    // H1: dense ids when the registry's /16 blocks allow (every host lies in
    // a registered /24, so rank-of-/16 << 16 | low 16 bits is unique and
    // needs no probe), else an open-addressing table of at least two slots
    // per possible key.
    const bool dense = dir && n16 && (static_cast<uint64_t>(n16) << 16) <= (1ull << 24);
    const int tbits = std::max(10, bits_for(2 * std::max<uint64_t>(1, std::min(n, max_keys))));
    const uint32_t cap = dense ? n16 << 16 : 1u << tbits;
    HCK(dalloc(&loc.table, cap, s)); // owned by `loc` (free_local)
    HCK(dalloc(&loc.acc, static_cast<size_t>(cap) * 5, s));
    loc.cap = cap;
    HCK(dalloc(&out.row_of, n, s)); // slots first, rows later; owned by `out`
    HCK(dalloc(&out.bkt, n, s));
    out.n_flows = n;
    if (!dense) HCK(cudaMemsetAsync(loc.table, 0xFF, static_cast<size_t>(cap) * 8, s));
    HCK(cudaMemsetAsync(loc.acc, 0, static_cast<size_t>(cap) * 40, s));
    unsigned long long* hot = nullptr; // dense ids: the preloaded hot slots of every H1 table
    if (dense) {
        uint32_t* cnt = nullptr;
        HCK(tmp_.get(&cnt, cap));
        HCK(tmp_.get(&hot, kAgg));
        HCK(cudaMemsetAsync(cnt, 0, static_cast<size_t>(cap) * 4, s));
        HCK(cudaMemsetAsync(hot, 0, static_cast<size_t>(kAgg) * 8, s));
        const uint32_t take = std::max<uint32_t>(32, (kSampleHead / n_slices) & ~3u);
        for (int i = 0; i < n_slices; ++i)
            h_hot_sample<<<(slices[i].log.regions + 31) / 32, 1024, 0, s>>>(
                slices[i].log, counts + slices[i].count_off, reinterpret_cast<const uint2*>(dir), take, cnt);
        h_hot_pick<<<grid_for(device, cap, 256), 256, 0, s>>>(cnt, cap, hot);
        HCK(cudaGetLastError());
    }
    for (int i = 0; i < n_slices; ++i) {
        const HostSlice& sl = slices[i];
        // At least four CTAs per SM, and enough CTAs that none takes more
        // than kInsItemsPerCta items (the limbs' no-wrap bound).
        const uint64_t items = h_scal[2 + i];
        if (items == 0) continue;
        const uint64_t g = std::max<uint64_t>((items + kInsItemsPerCta - 1) / kInsItemsPerCta,
                                              std::min<uint64_t>(items, static_cast<uint64_t>(GNM_INS_CTAS_PER_SM) * sms));
        if (dense)
            h_insert<true, true><<<static_cast<uint32_t>(g), kInsBlock, kInsSmem, s>>>(
                sl.log, counts + sl.count_off, off + sl.count_off, ioff + sl.count_off, static_cast<uint32_t>(items),
                reinterpret_cast<const uint2*>(dir), loc.table,
                cap - 1, 64 - tbits, loc.acc, out.row_of, out.bkt, hot);
        else
            h_insert<false, false><<<static_cast<uint32_t>(g), kInsBlock, kInsSmem, s>>>(
                sl.log, counts + sl.count_off, off + sl.count_off, ioff + sl.count_off, static_cast<uint32_t>(items),
                nullptr, loc.table, cap - 1, 64 - tbits, loc.acc,
                out.row_of, out.bkt, nullptr);
        HCK(cudaGetLastError());
    }
    // H2: distinct keys in (site, host) order -> rows.
    unsigned long long* hk = nullptr;
    uint32_t* hs = nullptr;
    const uint64_t kcap = std::min<uint64_t>(n, cap);
    HCK(tmp_.get(&hk, kcap));
    HCK(tmp_.get(&hs, kcap));
    if (dense) {
        uint32_t* prefix = nullptr;
        HCK(tmp_.get(&prefix, n16));
        h_prefix_of_rank<<<256, 256, 0, s>>>(reinterpret_cast<const uint2*>(dir), prefix);
        h_collect_dense<<<grid_for(device, cap, 256), 256, 0, s>>>(loc.acc, cap, prefix, dir,
                                                                  packed ? 0xFFFFFu : 0x7FFFFFFFu, hk, hs,
                                                                  reinterpret_cast<unsigned int*>(scal + 1));
    } else {
        h_collect<<<grid_for(device, cap, 256), 256, 0, s>>>(loc.table, cap, hk, hs,
                                                            reinterpret_cast<unsigned int*>(scal + 1));
    }
    HCK(cudaGetLastError());
    HCK(cudaMemcpyAsync(h_scal.data() + 1, scal + 1, 8, cudaMemcpyDeviceToHost, s));
    HCK(cudaStreamSynchronize(s));
    const uint32_t n_rows = static_cast<uint32_t>(h_scal[1]);
    HCK(dalloc(&loc.hk_sorted, n_rows, s));
    HCK(dalloc(&loc.hs_sorted, n_rows, s));
    size_t tb = 0;
    // keys are site << 32 | host: only the site's bits above the host sort
    const int end_bit = 32 + std::max(1, bits_for(std::max<uint64_t>(n_sites, 1)));
    HCK(cub::DeviceRadixSort::SortPairs(nullptr, tb, hk, loc.hk_sorted, hs, loc.hs_sorted, n_rows, 0, end_bit, s));
    unsigned char* tmp2 = nullptr;
    HCK(tmp_.get(&tmp2, tb));
    HCK(cub::DeviceRadixSort::SortPairs(tmp2, tb, hk, loc.hk_sorted, hs, loc.hs_sorted, n_rows, 0, end_bit, s));
    h_rank<<<grid_for(device, n_rows, 256), 256, 0, s>>>(loc.hs_sorted, n_rows, loc.table);
    HCK(cudaGetLastError());
    out.n_rows = n_rows;
    out.key64 = kBucketBits + bits_for(n_rows) > 32;
    return cudaSuccess;
}

// The median scheme for `rows` rows: the L2-resident two-round counts
// (rows * 628 B <= 64 MB) or the sort. GNM_HOSTS_MEDIAN=sort|two forces one
// (measurement; both are exact).
static bool two_round_median(uint32_t rows) {
    static const int force = [] {
        const char* e = std::getenv("GNM_HOSTS_MEDIAN");
        if (!e) return 0;
        return std::strcmp(e, "sort") == 0 ? 1 : (std::strcmp(e, "two") == 0 ? 2 : 0);
    }();
    if (force == 1) return false;
    if (force == 2) return rows < (1u << 24); // h_coarse's key packs the row in 24 bits
    return static_cast<size_t>(rows) * kCoarseH * 4 <= kTwoRoundBytes;
}

cudaError_t finish_hosts(int device, HostRows& out, HostLocal& loc, cudaStream_t s) {
    cudaError_t e = cudaSuccess;
    if (out.n_flows) {
        const uint32_t n_rows = static_cast<uint32_t>(out.n_rows);
        e = dalloc(&out.rows, n_rows, s);
        // H3..H5: the exact lower median per row (slots become rows on the way).
        if (e == cudaSuccess) {
            if (two_round_median(n_rows)) {
                e = finish_two_round(device, out, loc.table, loc.acc, loc.hk_sorted, loc.hs_sorted, s);
            } else {
                e = out.key64 ? finish_sorted<unsigned long long>(device, out, loc.table, loc.acc, loc.hk_sorted,
                                                                  loc.hs_sorted, s)
                              : finish_sorted<uint32_t>(device, out, loc.table, loc.acc, loc.hk_sorted,
                                                        loc.hs_sorted, s);
            }
        }
    }
    free_local(loc, s);
    return e;
}

cudaError_t build_hosts(int device, const HostSlice* slices, int n_slices, const unsigned int* counts,
                        size_t n_counts, uint64_t max_keys, HostRows& out, cudaStream_t s) {
    HostLocal loc;
    const cudaError_t e =
        build_hosts_local(device, slices, n_slices, counts, n_counts, max_keys, 0xFFFFFFFFu, nullptr, 0, true, out,
                          loc, s);
    if (e != cudaSuccess) {
        free_local(loc, s);
        return e;
    }
    return finish_hosts(device, out, loc, s);
}

// ---- cross-context combine ---------------------------------------------------------
namespace {
// Local row -> its index in the sorted union (every local key is in it).
__global__ void g_map(const unsigned long long* __restrict__ local, uint32_t n_local,
                      const unsigned long long* __restrict__ global, uint32_t n_global, uint32_t* __restrict__ map) {
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n_local; r += gridDim.x * blockDim.x) {
        const unsigned long long k = local[r];
        uint32_t lo = 0, hi = n_global;
        while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (global[mid] < k) lo = mid + 1;
            else hi = mid;
        }
        map[r] = lo;
    }
}

__global__ void g_init_min(unsigned long long* __restrict__ mn, uint32_t n) {
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) mn[r] = kMinInitBits;
}

__global__ void g_fill(const uint32_t* __restrict__ map, const uint32_t* __restrict__ hs_sorted, uint32_t n_local,
                       const unsigned long long* __restrict__ acc, unsigned long long* __restrict__ sums,
                       unsigned long long* __restrict__ mn, unsigned long long* __restrict__ mx) {
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n_local; r += gridDim.x * blockDim.x) {
        const unsigned long long* a = acc + static_cast<size_t>(hs_sorted[r]) * 5;
        const uint32_t g = map[r];
        sums[static_cast<size_t>(g) * 3 + 0] = a[0];
        sums[static_cast<size_t>(g) * 3 + 1] = a[1];
        sums[static_cast<size_t>(g) * 3 + 2] = a[2];
        mn[g] = ~a[3]; // the slot keeps its min complemented
        mx[g] = a[4];
    }
}

// Every flow's slot -> its global row.
__global__ void g_rows(uint32_t* __restrict__ row, uint32_t n, const unsigned long long* __restrict__ table,
                       const uint32_t* __restrict__ map) {
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x)
        row[j] = map[static_cast<uint32_t>(table[row[j]])];
}

__global__ void g_final(const unsigned long long* __restrict__ keys, const unsigned long long* __restrict__ sums,
                        const unsigned long long* __restrict__ mn, const unsigned long long* __restrict__ mx,
                        const uint32_t* __restrict__ cnt, const uint32_t* __restrict__ msb,
                        const uint32_t* __restrict__ mrank, const uint32_t* __restrict__ fine, uint32_t n,
                        gnm_host_stats* __restrict__ rows) {
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
        const uint32_t* f = fine + static_cast<size_t>(r) * kFineH;
        uint32_t cum = 0, k = msb[r] * kFineH + kFineH - 1;
        for (uint32_t q = 0; q < kFineH; ++q) {
            cum += f[q];
            if (cum >= mrank[r]) {
                k = msb[r] * kFineH + q;
                break;
            }
        }
        const unsigned long long* a = sums + static_cast<size_t>(r) * 3;
        const unsigned __int128 u = static_cast<unsigned __int128>(a[0]) +
                                    (static_cast<unsigned __int128>(a[1]) << 32) +
                                    (static_cast<unsigned __int128>(a[2]) << 64);
        const double lo_b = __longlong_as_double(static_cast<long long>(mn[r]));
        const double hi_b = __longlong_as_double(static_cast<long long>(mx[r]));
        double med = median_of_bucket(k);
        med = med < lo_b ? lo_b : (hi_b < med ? hi_b : med);
        gnm_host_stats o;
        o.site = static_cast<uint32_t>(keys[r] >> 32);
        o.host = static_cast<uint32_t>(keys[r]);
        o.flow_count = cnt[r];
        o.rate_ubps_lo = static_cast<uint64_t>(u);
        o.rate_ubps_hi = static_cast<uint64_t>(u >> 64);
        o.min_bps = lo_b;
        o.max_bps = hi_b;
        o.avg_bps = avg_of(o.rate_ubps_lo, o.rate_ubps_hi, o.flow_count);
        o.median_bps = med;
        rows[r] = o;
    }
}
} // namespace

cudaError_t hosts_global_begin(int device, HostRows& out, const HostLocal& loc, const unsigned long long* keys,
                               uint64_t n, HostGlobal& g, cudaStream_t s) {
    free_global(g, s);
    if (n >= (1ull << 24)) return cudaErrorInvalidValue; // the coarse pass keys rows in 24 bits
    g.n = n;
    const size_t ng = std::max<uint64_t>(n, 1);
    HCK(dalloc(&g.keys, ng, s));
    HCK(dalloc(&g.local_to_global, std::max<uint64_t>(out.n_rows, 1), s));
    HCK(dalloc(&g.sums, ng * 3, s));
    HCK(dalloc(&g.min, ng, s));
    HCK(dalloc(&g.max, ng, s));
    HCK(dalloc(&g.coarse, ng * kCoarseH, s));
    HCK(dalloc(&g.fine, ng * kFineH, s));
    HCK(dalloc(&g.msb, ng, s));
    HCK(dalloc(&g.mrank, ng, s));
    HCK(dalloc(&g.cnt, ng, s));
    if (n) HCK(cudaMemcpyAsync(g.keys, keys, n * 8, cudaMemcpyDeviceToDevice, s));
    HCK(cudaMemsetAsync(g.sums, 0, ng * 24, s));
    g_init_min<<<grid_for(device, ng, 256), 256, 0, s>>>(g.min, static_cast<uint32_t>(ng));
    HCK(cudaMemsetAsync(g.max, 0, ng * 8, s));
    HCK(cudaMemsetAsync(g.coarse, 0, ng * kCoarseH * 4, s));
    HCK(cudaMemsetAsync(g.fine, 0, ng * kFineH * 4, s));
    const uint32_t nl = static_cast<uint32_t>(out.n_rows);
    if (nl) {
        g_map<<<grid_for(device, nl, 256), 256, 0, s>>>(loc.hk_sorted, nl, g.keys, static_cast<uint32_t>(n),
                                                        g.local_to_global);
        g_fill<<<grid_for(device, nl, 256), 256, 0, s>>>(g.local_to_global, loc.hs_sorted, nl, loc.acc, g.sums,
                                                         g.min, g.max);
        const uint32_t nf = static_cast<uint32_t>(out.n_flows);
        g_rows<<<grid_for(device, nf, 256), 256, 0, s>>>(out.row_of, nf, loc.table, g.local_to_global);
        HCK(hosts_attributes(device));
        h_coarse<false><<<grid_for(device, nf, 512), 512, kCoarseSmem, s>>>(out.row_of, out.bkt, nf, static_cast<uint32_t>(n),
                                                           nullptr, g.coarse);
        HCK(cudaGetLastError());
    }
    out.global = true;
    return cudaSuccess;
}

cudaError_t hosts_global_prepare(int device, const HostRows& out, HostGlobal& g, cudaStream_t s) {
    const uint32_t n = static_cast<uint32_t>(g.n), nf = static_cast<uint32_t>(out.n_flows);
    if (n) h_msb<<<grid_for(device, n, 128), 128, 0, s>>>(g.coarse, n, g.msb, g.mrank, g.cnt);
    if (nf) h_fine<false><<<grid_for(device, (nf + 3) / 4, 256), 256, 0, s>>>(out.row_of, out.bkt, nf, g.msb, g.fine);
    g.prepared = true;
    return cudaGetLastError();
}

cudaError_t hosts_key_union(int device, const unsigned long long* all, uint64_t n, unsigned long long* out,
                            uint64_t* n_out, cudaStream_t s) {
    (void)device;
    *n_out = 0;
    if (n == 0) return cudaSuccess;
    Scratch tmp_(s);
    unsigned long long* sorted = nullptr;
    uint64_t* d_n = nullptr;
    HCK(tmp_.get(&sorted, n));
    HCK(tmp_.get(&d_n, 1));
    size_t tb = 0, tb2 = 0;
    HCK(cub::DeviceRadixSort::SortKeys(nullptr, tb, all, sorted, n, 0, 64, s));
    HCK(cub::DeviceSelect::Unique(nullptr, tb2, sorted, out, d_n, n, s));
    unsigned char* tmp = nullptr;
    HCK(tmp_.get(&tmp, std::max(tb, tb2)));
    HCK(cub::DeviceRadixSort::SortKeys(tmp, tb, all, sorted, n, 0, 64, s));
    HCK(cub::DeviceSelect::Unique(tmp, tb2, sorted, out, d_n, n, s));
    uint64_t m = 0;
    HCK(cudaMemcpyAsync(&m, d_n, 8, cudaMemcpyDeviceToHost, s));
    HCK(cudaStreamSynchronize(s));
    unsigned long long last = 0;
    if (m) {
        HCK(cudaMemcpyAsync(&last, out + m - 1, 8, cudaMemcpyDeviceToHost, s));
        HCK(cudaStreamSynchronize(s));
    }
    *n_out = m - (m && last == kEmpty ? 1 : 0); // the all-gather's padding sorts last
    return cudaSuccess;
}

cudaError_t hosts_global_finish(int device, HostRows& out, HostGlobal& g, cudaStream_t s) {
    if (out.rows) cudaFreeAsync(out.rows, s);
    out.rows = nullptr;
    // row_of now holds global rows: any sorted / sparse form of the local
    // rows is stale, and the (row, bucket) key width follows the union
    for (void* p : {out.sorted, out.sp_keys, static_cast<void*>(out.sp_counts)})
        if (p) cudaFreeAsync(p, s);
    out.sorted = out.sp_keys = nullptr;
    out.sp_counts = nullptr;
    out.n_sparse = ~0ull;
    out.key64 = kBucketBits + bits_for(std::max<uint64_t>(g.n, 1)) > 32;
    const uint32_t n = static_cast<uint32_t>(g.n);
    HCK(dalloc(&out.rows, std::max<uint32_t>(n, 1), s));
    if (n)
        g_final<<<grid_for(device, n, 128), 128, 0, s>>>(g.keys, g.sums, g.min, g.max, g.cnt, g.msb, g.mrank,
                                                         g.fine, n, out.rows);
    out.n_rows = n;
    return cudaGetLastError();
}

void free_local(HostLocal& loc, cudaStream_t s) {
    for (void* p : {static_cast<void*>(loc.table), static_cast<void*>(loc.acc), static_cast<void*>(loc.hk_sorted),
                    static_cast<void*>(loc.hs_sorted)})
        if (p) cudaFreeAsync(p, s);
    loc = HostLocal{};
}

void free_global(HostGlobal& g, cudaStream_t s) {
    for (void* p : {static_cast<void*>(g.keys), static_cast<void*>(g.local_to_global), static_cast<void*>(g.sums),
                    static_cast<void*>(g.min), static_cast<void*>(g.max), static_cast<void*>(g.coarse),
                    static_cast<void*>(g.fine), static_cast<void*>(g.msb), static_cast<void*>(g.mrank),
                    static_cast<void*>(g.cnt)})
        if (p) cudaFreeAsync(p, s);
    g = HostGlobal{};
}

cudaError_t hosts_histograms(int device, const HostRows& h, uint32_t* dense, cudaStream_t s) {
    if (h.n_flows == 0) return cudaSuccess;
    h_hist<<<grid_for(device, h.n_flows, 256), 256, 0, s>>>(h.row_of, h.bkt, h.n_flows, dense, h.packed);
    return cudaGetLastError();
}

namespace {
template <typename K>
cudaError_t rle(HostRows& h, cudaStream_t s) {
    const K* in = static_cast<const K*>(h.sorted);
    Scratch tmp_(s);
    K* keys = nullptr;
    uint64_t* d_n = nullptr;
    HCK(dalloc(&keys, h.n_flows, s));
    h.sp_keys = keys; // owned by `h` from here (free_hosts)
    HCK(dalloc(&h.sp_counts, h.n_flows, s));
    HCK(tmp_.get(&d_n, 1));
    size_t tb = 0;
    HCK(cub::DeviceRunLengthEncode::Encode(nullptr, tb, in, keys, h.sp_counts, d_n, h.n_flows, s));
    unsigned char* tmp = nullptr;
    HCK(tmp_.get(&tmp, tb));
    HCK(cub::DeviceRunLengthEncode::Encode(tmp, tb, in, keys, h.sp_counts, d_n, h.n_flows, s));
    uint64_t n = 0;
    HCK(cudaMemcpyAsync(&n, d_n, 8, cudaMemcpyDeviceToHost, s));
    HCK(cudaStreamSynchronize(s));
    h.n_sparse = n;
    return cudaSuccess;
}

template <typename K>
__global__ void h_split(const K* __restrict__ keys, uint64_t n, uint32_t* __restrict__ rows,
                        uint32_t* __restrict__ buckets) {
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        rows[i] = static_cast<uint32_t>(keys[i] >> kBucketBits);
        buckets[i] = static_cast<uint32_t>(keys[i] & kBucketMask);
    }
}
} // namespace

cudaError_t hosts_sparse(int device, HostRows& h, uint64_t* n, cudaStream_t s) {
    if (h.n_sparse == ~0ull) {
        if (h.n_flows == 0) {
            h.n_sparse = 0;
        } else {
            HCK(ensure_sorted(device, h, s)); // the two-round median needs no sort; histograms do
            HCK(h.key64 ? rle<unsigned long long>(h, s) : rle<uint32_t>(h, s));
        }
    }
    *n = h.n_sparse;
    return cudaSuccess;
}

cudaError_t hosts_sparse_export(int device, const HostRows& h, uint32_t* rows, uint32_t* buckets, uint32_t* counts,
                                cudaStream_t s) {
    if (h.n_sparse == 0 || h.n_sparse == ~0ull) return cudaSuccess;
    const uint32_t g = grid_for(device, h.n_sparse, 256);
    if (h.key64)
        h_split<<<g, 256, 0, s>>>(static_cast<const unsigned long long*>(h.sp_keys), h.n_sparse, rows, buckets);
    else
        h_split<<<g, 256, 0, s>>>(static_cast<const uint32_t*>(h.sp_keys), h.n_sparse, rows, buckets);
    HCK(cudaGetLastError());
    return cudaMemcpyAsync(counts, h.sp_counts, h.n_sparse * 4, cudaMemcpyDeviceToDevice, s);
}

void free_hosts(HostRows& h, cudaStream_t s) {
    for (void* p : {static_cast<void*>(h.rows), h.sorted, h.sp_keys, static_cast<void*>(h.sp_counts),
                    static_cast<void*>(h.row_of), static_cast<void*>(h.bkt)})
        if (p) cudaFreeAsync(p, s);
    h = HostRows{};
}

} // namespace gnm

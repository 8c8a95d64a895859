// kernels.cuh — launch interface of the sm_100a kernels (kernels.cu).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "gnetmon.h"

namespace gnm {

constexpr uint32_t kBuckets = 10001;
// Exact lower median by two-round selection instead of dense 10001-bucket
// histograms:
//   round 1  coarse counts per (site, super-bucket), super-bucket = bucket >> 6
//            (157 of them; bucket 10000 -> 156), kept by K2 in a 6 MB
//            L2-resident array (sb-major: coarse[sb * n_sites + site]);
//   round 2  each site's median super-bucket is found from the coarse
//            counts (K3a); the fine counts of just that super-bucket (64
//            buckets) are rebuilt from K2's per-flow log (K2b); K3b walks
//            them to the exact bucket.
// The log holds one entry per candidate flow: site << 14 | bucket (or a
// skip marker), plus a second u32 array of buckets for registries of >=
// 2^18 sites. Dense histograms, when asked for, are rebuilt from the log.
constexpr uint32_t kCoarse = 157;
constexpr uint32_t kFineW = 64;
constexpr uint32_t kLogSkip = 0xFFFFFFFFu;
constexpr uint32_t kLogSiteShift = 14;
constexpr uint32_t kLogPackedSites = 1u << 18;
constexpr uint64_t kMinInitBits = 0x7FF0000000000000ull; // +inf: empty min
constexpr uint64_t kMaxInitBits = 0;                     // +0.0: empty max (rates are > 0)
constexpr uint32_t kHotSlots = 2047;  // block-private accumulators for hot sites (11 slot bits)
constexpr uint32_t kHotStride = 2048; // kHotSlots + 1 (slot 0 = cold)

#ifdef __CUDACC__
// stats_from's avg (rate_engine.cpp:250; sum_bps rate_engine.hpp:62):
// (double(u128 sum) / 1e6) / double(count), each step rounded to nearest
// even like the host (libgcc __floatuntidf): a sum of >= 2^64 keeps its top
// 64 bits with the shifted-out bits folded into a sticky LSB, which rounds
// to 53 bits exactly as the 128-bit value would, then scales by 2^shift.
__device__ __forceinline__ double avg_of(uint64_t lo, uint64_t hi, uint64_t count) {
    double sum;
    if (hi == 0) {
        sum = __ull2double_rn(lo);
    } else {
        const int lz = __clzll(static_cast<long long>(hi));
        const int sh = 64 - lz;
        const uint64_t top = (hi << lz) | (lo >> sh);
        const uint64_t sticky = (lo << lz) != 0 ? 1u : 0u;
        sum = ldexp(__ull2double_rn(top | sticky), sh);
    }
    return __ddiv_rn(__ddiv_rn(sum, 1e6), __ull2double_rn(count));
}

// median_bps (rate_engine.cpp:42-58) of lower-median bucket k, before the
// clamp into [min, max] (stats_from :251).
__device__ __forceinline__ double median_of_bucket(uint32_t k) {
    return k == kBuckets - 1 ? 100000000.0 : __dadd_rn(__dmul_rn(static_cast<double>(k), 10000.0), 5000.0);
}
#endif

// Hot-site plan scratch (u32 words): per-site sample counts (padded to a
// multiple of 4: read as 16-byte vectors), site -> slot, slot -> site.
inline size_t plan_slot_offset(uint32_t n_sites) { return (static_cast<size_t>(n_sites) + 3) / 4 * 4; }
inline size_t plan_hot_site_offset(uint32_t n_sites) { return plan_slot_offset(n_sites) + n_sites; }
inline size_t plan_scratch_words(uint32_t n_sites) { return plan_hot_site_offset(n_sites) + kHotStride + 1; }

struct DevParams {
    uint64_t ack_plus1;       // ack_avg_size_max + 1, u64 (rate_engine.cpp:78)
    uint32_t min_packets;
    uint32_t min_duration_ms;
    uint32_t min_packets1;    // max(min_packets, 1): folds d_pkts == 0 (:75) into one compare
    uint32_t min_duration1;   // max(min_duration_ms, 1): folds duration == 0 (:81)
    uint32_t site_mask;       // kPackedSiteMask, or 0x7FFFFFFF for wide tables
    uint32_t wide_log;        // registry >= kLogPackedSites sites: log buckets in their own array
    uint32_t windowed;        // 1: analyze only records with end_ms in [win_lo, win_hi)
    uint64_t win_lo;          //    (FlowStore::snapshot, flow_store.cpp:75), fused into K1/K2
    uint64_t win_hi;
    uint32_t ablation;        // GNM_K2_ABLATION builds only (tools/ablation.sh); 0 otherwise
};

// Device partial accumulators of one context (layout in gnetmon.h, gnm_partials).
struct DevPartials {
    unsigned long long* sums; // [n_sites*4 + 4]
    unsigned long long* mn;   // f64 bits
    unsigned long long* mx;   // f64 bits
    unsigned int* coarse;     // [kCoarse * n_sites], sb-major
    unsigned int* fine;       // [n_sites * kFineW]: the median super-bucket's buckets
    unsigned int* msb;        // [n_sites]: median super-bucket (K3a, low 8 bits; 0xFF if
                              // empty) | K2b heavy-row index << 8 (0xFFFFFF: none)
    unsigned int* mrank;      // [n_sites]: rank of the lower median within it (1-based)
    unsigned long long* cnt;  // [n_sites]: flow count (K3a)
    unsigned int* heavy_next; // K3a's heavy-row counter, then the site of each heavy row
    unsigned short* map16;    // [n_sites + 8]: K3a's (median super-bucket | heavy row << 8) for K2b
    uint32_t n_sites;
};

// One K2 launch's slice of the log: per-warp regions of warp_cap entries
// (region = blockIdx * warps + warp), each warp's entry count in counts[].
struct DevLog {
    unsigned int* entries;
    unsigned int* buckets; // wide registries only (>= kLogPackedSites sites), else null
    unsigned int* counts;
    uint32_t warp_cap;
    uint32_t regions;
    // Hosts mode (gnm_ctx_set_hosts), else null: per entry the matched host
    // IP, the flow's octets and duration (H1 recomputes the f64 rate and the
    // exact micro-bps from them: 16 bytes per flow instead of 24); indexed
    // like `entries` from this slice's base.
    unsigned int* hosts;
    unsigned int* octs;
    unsigned long long* durs;
};

// Per-call hot-site plan: slot -> site (slots 1..n_slots), 0 slots = off.
struct DevHot {
    const uint32_t* hot_site;
    uint32_t n_slots;
    // With the table in shared memory, K2 applies the plan's slot numbers
    // (site -> slot) while loading it (no k_table_slots pass); null otherwise.
    const uint32_t* site_slot;
    uint32_t node_begin, leaf_begin;
};

struct DevSoA {
    const uint32_t* src;
    const uint32_t* dst;
    const uint32_t* pkts;
    const uint32_t* octets;
    const uint64_t* start;
    const uint64_t* end;
    uint64_t n;
    // Loader-compacted batches (non-windowed host SoA input): the duration
    // end - start as u32, computed on the host, in place of start/end (which
    // are then null). K2 layout 5.
    const uint32_t* dur32 = nullptr;
};

// A batch is SoA columns or 64-byte flowmon::FlowRecord AoS rows.
struct DevBatch {
    bool aos;
    bool archive; // aos rows are FLOWARC1 entries (big-endian, flow_store.cpp:144-165)
    DevSoA soa;
    const void* rec;
    uint64_t n;
};

struct DevTable {
    uint32_t* words;
    uint32_t n_words;     // padded to a multiple of 4
    uint32_t node_begin;
    uint32_t leaf_begin;
    bool packed;
};

struct LaunchCfg {
    int grid;
    int block;
    size_t smem;
    bool table_in_smem;
};

// Once per device: opt the shared-memory kernels into large dynamic smem.
cudaError_t init_kernel_attributes();

// Occupancy-derived launch configuration for K2 over n records.
// occ_cache[hot] memoises blocks/SM (0 = unknown) for this table size.
LaunchCfg k2_config(int device, const DevBatch& b, uint32_t table_words, bool hot, int* occ_cache,
                    bool hosts = false);

// K1 (optional, skewed batches): sample the batch, pick the hot sites and
// write their slots into the table words; the sampled Forward flows' rates
// also go into the partials' min/max (`mn`, `mx`), which seed K2's hot-slot
// caches. Returns false when the batch is
// too small for block-private accumulation to pay; `scratch` holds
// n_sites u32 counts (zero at rest), n_sites u32 site->slot and kHotStride
// u32 slot->site.
bool plan_hot(int device, const DevBatch& b, const DevTable& t, const DevParams& p,
              uint32_t n_sites, uint32_t* scratch, unsigned long long* mn, unsigned long long* mx,
              int k2_grid, bool force, bool table_in_smem, cudaStream_t s, uint64_t* launches,
              cudaError_t* err);

// Entries one warp region must hold for a launch of `cfg` over b (>= the
// warp's records, rounded up to the 32-entry drain granularity).
uint32_t k2_warp_cap(const LaunchCfg& cfg, const DevBatch& b);
uint32_t k2_regions(const LaunchCfg& cfg);
cudaError_t launch_k2(const LaunchCfg& cfg, const DevBatch& b, const DevTable& t,
                      const DevParams& p, const DevPartials& P, const DevHot& hot,
                      const DevLog& log, cudaStream_t s);
// K3a: per-site flow count -> median super-bucket and rank (round 1).
cudaError_t launch_k3a(int device, const DevPartials& P, cudaStream_t s);
// K2b: fine counts of every site's median super-bucket from one launch's log (round 2).
cudaError_t launch_k2b(int device, const DevPartials& P, const DevLog& log, cudaStream_t s);
// K3b: exact median, clamp, flag and the site table; reset != 0 clears the
// partials (sums, min/max, coarse, fine).
cudaError_t launch_k3b(int device, const DevPartials& P, double threshold, gnm_site_stats* out,
                       int reset, cudaStream_t s);
cudaError_t launch_reset(int device, const DevPartials& P, cudaStream_t s);
cudaError_t launch_init_partials(const DevPartials& P, cudaStream_t s);
// Dense [n_sites][10001] histograms (RateHistogram::buckets_ order) from one
// launch's log, added into `dense` (device memory, zeroed by the caller).
cudaError_t launch_hist_from_log(int device, const DevLog& log, uint32_t n_sites, uint32_t* dense,
                                 cudaStream_t s);
cudaError_t launch_classify(const LaunchCfg& cfg, const DevSoA& b, const DevTable& t,
                            const DevParams& p, uint32_t* out, cudaStream_t s);

} // namespace gnm

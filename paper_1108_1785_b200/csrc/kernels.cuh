// kernels.cuh — launch interface of the sm_100a kernels (kernels.cu).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "gnetmon.h"

namespace gnm {

constexpr uint32_t kBuckets = 10001;
// Per-site histograms, sector-blocked and bucket-major: the 8 buckets of
// one 32-byte sector belong to one site (the sector footprint of a site's
// touched buckets is the same as a site-major row), while consecutive
// 8-bucket groups of a site lie n_sites * 32 B apart. A hot site's buckets
// therefore spread over every L2 slice instead of the few slices a 40 KB
// row would map to (same-slice RED contention, profiles/round1).
constexpr uint32_t kBucketGroups = (kBuckets + 7) / 8; // 1251
constexpr uint32_t kHistStride = kBucketGroups * 8;   // words per site
__host__ __device__ inline size_t hist_index(uint32_t site, uint32_t bucket, uint32_t n_sites) {
    return (static_cast<size_t>(bucket >> 3) * n_sites + site) * 8 + (bucket & 7u);
}
constexpr uint64_t kMinInitBits = 0x7FF0000000000000ull; // +inf: empty min
constexpr uint64_t kMaxInitBits = 0;                     // +0.0: empty max (rates are > 0)
constexpr uint32_t kHotSlots = 512;   // block-private accumulators for hot sites
constexpr uint32_t kHotStride = 520;  // kHotSlots + 1 (slot 0 = cold), padded

struct DevParams {
    uint64_t ack_plus1;       // ack_avg_size_max + 1, u64 (rate_engine.cpp:78)
    uint32_t min_packets;
    uint32_t min_duration_ms;
    uint32_t min_packets1;    // max(min_packets, 1): folds d_pkts == 0 (:75) into one compare
    uint32_t min_duration1;   // max(min_duration_ms, 1): folds duration == 0 (:81)
    uint32_t site_mask;       // kPackedSiteMask, or 0x7FFFFFFF for wide tables
    uint32_t ablation;        // GNM_K2_ABLATION builds only (tools/ablation.sh); 0 otherwise
};

// Device partial accumulators of one context (layout in gnetmon.h, gnm_partials).
struct DevPartials {
    unsigned long long* sums; // [n_sites*4 + 4]
    unsigned long long* mn;   // f64 bits
    unsigned long long* mx;   // f64 bits
    unsigned int* hist;       // [n_sites * 10001]
    uint32_t n_sites;
};

// Per-call hot-site plan: slot -> site (slots 1..n_slots), 0 slots = off.
struct DevHot {
    const uint32_t* hot_site;
    uint32_t n_slots;
};

struct DevSoA {
    const uint32_t* src;
    const uint32_t* dst;
    const uint32_t* pkts;
    const uint32_t* octets;
    const uint64_t* start;
    const uint64_t* end;
    uint64_t n;
};

// A batch is SoA columns or 64-byte flowmon::FlowRecord AoS rows.
struct DevBatch {
    bool aos;
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
    int variant; // aligned SoA: 0 register double-buffered loads, 1 TMA L2 prefetch,
                 // 2 TMA bulk copies into per-warp shared-memory rings
};

// Once per device: opt the shared-memory kernels into large dynamic smem.
cudaError_t init_kernel_attributes();

// Occupancy-derived launch configuration for K2 over n records.
// occ_cache[hot] memoises blocks/SM (0 = unknown) for this table size.
LaunchCfg k2_config(int device, const DevBatch& b, uint32_t table_words, bool hot, int* occ_cache,
                    int variant = 0);

// K1 (optional, skewed batches): sample the batch, pick the hot sites and
// write their slots into the table words. Returns false when the batch is
// too small for block-private accumulation to pay; `scratch` holds
// n_sites u32 counts (zero at rest), n_sites u32 site->slot and kHotStride
// u32 slot->site.
bool plan_hot(int device, const DevBatch& b, const DevTable& t, const DevParams& p,
              uint32_t n_sites, uint32_t* scratch, int k2_grid, bool force, cudaStream_t s,
              uint64_t* launches, cudaError_t* err);

cudaError_t launch_k2(const LaunchCfg& cfg, const DevBatch& b, const DevTable& t,
                      const DevParams& p, const DevPartials& P, const DevHot& hot,
                      cudaStream_t s);
// K3: per-site count/median/flag; reset != 0 also clears the partials.
cudaError_t launch_k3(int device, const DevPartials& P, double threshold, gnm_site_stats* out,
                      int reset, cudaStream_t s);
cudaError_t launch_reset(int device, const DevPartials& P, cudaStream_t s);
cudaError_t launch_init_partials(const DevPartials& P, cudaStream_t s);
// Dense [n_sites][10001] copy of the blocked histograms (the reference's
// RateHistogram::buckets_ order) into `dense` (device memory).
cudaError_t launch_hist_export(const DevPartials& P, uint32_t* dense, cudaStream_t s);
cudaError_t launch_classify(const LaunchCfg& cfg, const DevSoA& b, const DevTable& t,
                            const DevParams& p, uint32_t* out, cudaStream_t s);

} // namespace gnm

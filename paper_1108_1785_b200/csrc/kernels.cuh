// kernels.cuh — launch interface of the sm_100a kernels (kernels.cu).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "gnetmon.h"

namespace gnm {

constexpr uint32_t kBuckets = 10001;
constexpr uint64_t kMinInitBits = 0x7FF0000000000000ull; // +inf: empty min
constexpr uint64_t kMaxInitBits = 0;                     // +0.0: empty max (rates are > 0)

struct DevParams {
    uint64_t ack_plus1;       // ack_avg_size_max + 1, u64 (rate_engine.cpp:78)
    uint32_t min_packets;
    uint32_t min_duration_ms;
};

// Device partial accumulators of one context (layout in gnetmon.h, gnm_partials).
struct DevPartials {
    unsigned long long* sums; // [n_sites*4 + 4]
    unsigned long long* mn;   // f64 bits
    unsigned long long* mx;   // f64 bits
    unsigned int* hist;       // [n_sites * 10001]
    uint32_t n_sites;
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

struct LaunchCfg {
    int grid;
    int block;
    size_t smem;
    bool table_in_smem;
};

// Once per device: opt the shared-memory-table kernels into > 48 KB smem.
cudaError_t init_kernel_attributes();

// Occupancy-derived launch configuration for K2 over n records with a table
// of `table_words` u32.
LaunchCfg k2_config(int device, uint64_t n, uint32_t table_words, bool aos);

cudaError_t launch_k2_soa(const LaunchCfg& cfg, const DevSoA& b, const uint32_t* table,
                          uint32_t table_words, const DevParams& p, const DevPartials& P,
                          cudaStream_t s);
cudaError_t launch_k2_aos(const LaunchCfg& cfg, const void* records, uint64_t n,
                          const uint32_t* table, uint32_t table_words, const DevParams& p,
                          const DevPartials& P, cudaStream_t s);
// K3: per-site count/median/flag; reset != 0 also clears the partials.
cudaError_t launch_k3(int device, const DevPartials& P, double threshold, gnm_site_stats* out,
                      int reset, cudaStream_t s);
cudaError_t launch_reset(int device, const DevPartials& P, cudaStream_t s);
cudaError_t launch_init_partials(const DevPartials& P, cudaStream_t s);
cudaError_t launch_classify(const LaunchCfg& cfg, const DevSoA& b, const uint32_t* table,
                            uint32_t table_words, const DevParams& p, uint32_t* out,
                            cudaStream_t s);

} // namespace gnm

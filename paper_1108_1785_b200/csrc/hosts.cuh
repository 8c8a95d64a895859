// hosts.cuh — per-host statistics post-pass (hosts.cu), SURVEY.md §8f next #1.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "kernels.cuh"

namespace gnm {

// One K2 launch's slice of the hosts-mode log (the DevLog K2 wrote) and where
// it sits in the context's concatenated log and per-warp counts.
struct HostSlice {
    DevLog log;
    size_t entry_off; // first entry of the slice in the whole log
    size_t count_off; // first per-warp count of the slice
};

// Device results of one post-pass; owned by the caller's context, released
// with free_hosts. row_of/bkt keep every flow's (row, bucket) for the
// optional histogram exports.
struct HostRows {
    gnm_host_stats* rows = nullptr;
    uint64_t n_rows = 0;
    uint32_t* row_of = nullptr; // per flow: its row (stale H1 slots when `packed`)
    uint32_t* bkt = nullptr;    // per flow: its bucket, or row << 14 | bucket when `packed`
    bool packed = false;        // the local two-round median packed the rows into bkt (rows < 2^18)
    uint64_t n_flows = 0;
    void* sorted = nullptr;     // (row << 14 | bucket) keys in order, u32 or u64 per key64; on demand
    bool key64 = false;
    bool global = false;        // rows are a cross-context union: histograms would be local only
    // Sparse histograms (run-length encoding of `sorted`), built on demand.
    void* sp_keys = nullptr; // unique (row << 14 | bucket), same width as `sorted`
    uint32_t* sp_counts = nullptr;
    uint64_t n_sparse = ~0ull; // ~0: not built yet
};

// The local phase's state, kept for the cross-GPU combine (H0..H2 done).
struct HostLocal {
    unsigned long long* table = nullptr;     // slot -> local row (after H2)
    unsigned long long* acc = nullptr;       // per slot {limb0, limb1, limb2, ~min, max}
    unsigned long long* hk_sorted = nullptr; // local distinct keys (site << 32 | host), sorted
    uint32_t* hs_sorted = nullptr;           // local row -> slot
    uint32_t cap = 0;
    bool ready = false;
};

// Global rows of a multi-context combine (gnm_hosts_*): every rank's
// partials indexed by the union of all ranks' keys, reduced by the caller
// (sums / coarse / fine: SUM; min: MIN; max: MAX -- f64 bits, +inf / 0
// where a rank saw no flow of the row).
struct HostGlobal {
    unsigned long long* keys = nullptr; // [n] sorted union of keys
    uint32_t* local_to_global = nullptr;
    unsigned long long* sums = nullptr; // [n * 3] micro-bps limbs
    unsigned long long* min = nullptr;  // [n] min rate bits
    unsigned long long* max = nullptr;  // [n]
    uint32_t* coarse = nullptr;         // [157 * n] super-bucket-major
    uint32_t* fine = nullptr;           // [n * 64]
    uint32_t* msb = nullptr;
    uint32_t* mrank = nullptr;
    uint32_t* cnt = nullptr;
    uint64_t n = 0;
    bool prepared = false;
};

// Local phase (H0..H2): flat per-flow (slot, bucket), per-slot sums, the
// sorted local keys; `out.n_rows` = local rows. Then either finish_hosts
// (this context's rows) or the global combine below.
// dir / n16: the device registry table's /16 directory and its non-empty
// /16 count (dense host ids when n16 << 16 <= 2^24), or null / 0 (hashing).
cudaError_t build_hosts_local(int device, const HostSlice* slices, int n_slices, const unsigned int* counts,
                              size_t n_counts, uint64_t max_keys, uint32_t n_sites, const uint32_t* dir, uint32_t n16,
                              bool packed, HostRows& out, HostLocal& loc, cudaStream_t s);
cudaError_t finish_hosts(int device, HostRows& out, HostLocal& loc, cudaStream_t s);
// Global combine: begin (map local rows into the union, fill sums/min/max
// and coarse counts), [caller all-reduces], prepare (each row's median
// super-bucket, this context's fine counts), [caller all-reduces fine],
// finish (rows of the union in out.rows).
cudaError_t hosts_global_begin(int device, HostRows& out, const HostLocal& loc, const unsigned long long* keys,
                               uint64_t n, HostGlobal& g, cudaStream_t s);
// Sorted union (duplicates and the kEmpty padding dropped) of n keys
// all-gathered from every rank; out holds up to n keys. Synchronises s.
cudaError_t hosts_key_union(int device, const unsigned long long* all, uint64_t n, unsigned long long* out,
                            uint64_t* n_out, cudaStream_t s);
cudaError_t hosts_global_prepare(int device, const HostRows& out, HostGlobal& g, cudaStream_t s);
cudaError_t hosts_global_finish(int device, HostRows& out, HostGlobal& g, cudaStream_t s);
void free_local(HostLocal& loc, cudaStream_t s);
void free_global(HostGlobal& g, cudaStream_t s);

// Builds the per-host rows from the log slices and all per-warp counts.
// max_keys bounds the distinct (site, host) keys (256 per registry /24
// entry). Synchronises `s` twice (to size the tables).
cudaError_t build_hosts(int device, const HostSlice* slices, int n_slices,
                        const unsigned int* counts, size_t n_counts, uint64_t max_keys, HostRows& out,
                        cudaStream_t s);

// Dense [n_rows][kBuckets] histograms of the rows (device buffer, zeroed by the caller).
cudaError_t hosts_histograms(int device, const HostRows& h, uint32_t* dense, cudaStream_t s);

// Sparse histograms: the non-zero (row, bucket) counts in (row, bucket)
// order. hosts_sparse builds them (once per result) and returns their count
// (synchronises `s`); hosts_sparse_export writes them to device arrays.
cudaError_t hosts_sparse(int device, HostRows& h, uint64_t* n, cudaStream_t s);
cudaError_t hosts_sparse_export(int device, const HostRows& h, uint32_t* rows, uint32_t* buckets, uint32_t* counts,
                                cudaStream_t s);

void free_hosts(HostRows& h, cudaStream_t s);

} // namespace gnm

/*
 * gnetmon.h — C-ABI boundary of the B200-native G-NetMon flow-analysis hot path.
 *
 * This is the drop-in boundary for the reference's analytics layer
 * (flowmon, /root/reference/proj). Every entry point below names the
 * reference interface it replaces (file:line relative to
 * /root/reference/proj/core). No C++ types, no exceptions and no torch types
 * cross this boundary: plain pointers, sizes and an int status, plus a
 * thread-local last-error string (gnm_last_error).
 *
 * Hot path:  classify -> attribute -> rate -> per-site
 * aggregate (K1 plan + K2, sm_100a) -> per-site median/avg/flag (K3a, K2b,
 * K3b: the two-round exact median, sm_100a) -> streak rule (host).
 * Around it (§8f): per-host rows (gnm_ctx_set_hosts), the snapshot window
 * fused into K2 (gnm_*_window), NetFlow v5 decode (gnm_decode_netflow) and
 * FLOWARC1 archives (gnm_decode_archive, gnm_*_archive).
 */
#ifndef GNETMON_H
#define GNETMON_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GNM_ABI_VERSION 4

/* rate_engine.hpp:18-20 */
#define GNM_BUCKET_COUNT 10001
#define GNM_BUCKET_WIDTH_BPS 10000.0
#define GNM_RATE_CAP_BPS 100000000.0
/* monitor.hpp:15 */
#define GNM_DEFAULT_WARN_THRESHOLD_BPS 1000000.0

#define GNM_NO_SITE 0xFFFFFFFFu

/* Status codes. The reference throws; these map its exception kinds. */
typedef enum gnm_status {
    GNM_OK = 0,
    GNM_ERR_INVALID_ARGUMENT = 1,
    GNM_ERR_OVERLAP = 2,        /* CatalogError::Kind::Overlap      site_catalog.hpp:18 */
    GNM_ERR_INVALID_CIDR = 3,   /* CatalogError::Kind::InvalidCidr  site_catalog.hpp:18 */
    GNM_ERR_CUDA = 4,           /* any CUDA runtime error */
    GNM_ERR_OUT_OF_MEMORY = 5,  /* std::bad_alloc / cudaErrorMemoryAllocation */
    GNM_ERR_ZERO_DURATION = 6,  /* RateError::Kind::ZeroDuration    rate_engine.hpp:37 */
    GNM_ERR_EMPTY_HISTOGRAM = 7,/* RateError::Kind::EmptyHistogram  rate_engine.hpp:37 */
    GNM_ERR_NO_DEVICE = 8,      /* no CUDA device: there is no CPU fallback */
    GNM_ERR_CAPACITY = 9,       /* caller buffer too small */
    GNM_ERR_BAD_MAGIC = 10,     /* ArchiveError::Kind::BadMagic          flow_store.hpp:24 */
    GNM_ERR_BAD_VERSION = 11,   /* ArchiveError::Kind::BadVersion */
    GNM_ERR_TRUNCATED = 12,     /* ArchiveError::Kind::TruncatedArchive (incl. trailing bytes) */
    GNM_ERR_COMM = 13           /* NCCL / communicator failure (multi-GPU combine) */
} gnm_status;

/* FlowClass (rate_engine.hpp:31), same ordinal values. */
typedef enum gnm_flow_class {
    GNM_FORWARD = 0,
    GNM_PURE_ACK = 1,
    GNM_ADMINISTRATIVE = 2,
    GNM_UNMATCHED = 3
} gnm_flow_class;

/* Thread-local message of the last failing call on this thread. */
const char* gnm_last_error(void);
int gnm_abi_version(void);

/* ---- FilterParams (rate_engine.hpp:22-29) ------------------------------- */
typedef struct gnm_filter_params {
    uint32_t ack_avg_size_max; /* default 96  */
    uint32_t min_packets;      /* default 20  */
    uint32_t min_duration_ms;  /* default 100 */
    uint32_t workers;          /* accepted, ignored: the GPU grid is the worker pool */
} gnm_filter_params;

void gnm_filter_params_default(gnm_filter_params* out);

/* ---- Site registry: replaces SiteCatalog (site_catalog.hpp:50-97) -------- */
typedef struct gnm_cidr {
    uint32_t addr;      /* host byte order, as Cidr::addr (site_catalog.hpp:32) */
    int32_t prefix_len; /* 1..32 */
} gnm_cidr;

typedef struct gnm_registry gnm_registry;

/* Cidr::parse (site_catalog.cpp:48-66). GNM_ERR_INVALID_CIDR on bad text. */
int gnm_cidr_parse(const char* text, gnm_cidr* out);
/* parse_ipv4 (site_catalog.cpp:10-40). */
int gnm_ipv4_parse(const char* text, uint32_t* out);

int gnm_registry_create(gnm_registry** out);
void gnm_registry_destroy(gnm_registry* reg);
/* SiteCatalog::register_site (site_catalog.cpp:90-121): expands each CIDR
 * into /24 tiles (longer prefixes round up to the enclosing /24), rejects
 * overlap with GNM_ERR_OVERLAP and leaves the registry unchanged on error.
 * Site ids are dense registration indices. */
int gnm_registry_register_site(gnm_registry* reg, const char* name, const gnm_cidr* cidrs,
                               size_t n_cidrs, uint32_t* out_site_id);
/* SiteCatalog::lookup (site_catalog.hpp:99-112); GNM_NO_SITE when absent. */
uint32_t gnm_registry_lookup(const gnm_registry* reg, uint32_t ip);
/* SiteCatalog::sequential_lookup (site_catalog.hpp:114-122). */
uint32_t gnm_registry_sequential_lookup(const gnm_registry* reg, uint32_t ip);
size_t gnm_registry_site_count(const gnm_registry* reg);
size_t gnm_registry_entry_count(const gnm_registry* reg);
/* SiteCatalog::entries (site_catalog.hpp:77): (prefix24, site) in insertion
 * order. Writes min(cap, entry_count) pairs. */
size_t gnm_registry_entries(const gnm_registry* reg, uint32_t* prefix24, uint32_t* site,
                            size_t cap);
/* SiteCatalog::site(id).name; NULL when out of range. */
const char* gnm_registry_site_name(const gnm_registry* reg, uint32_t site);
/* Bumped by every successful registration (device copies re-upload lazily). */
uint64_t gnm_registry_version(const gnm_registry* reg);

/* ---- Flow batches ---------------------------------------------------------
 * The hot columns of flowmon::FlowRecord (netflow.hpp:59-67): src_addr@0,
 * dst_addr@4, d_pkts@16, d_octets@20, start_ms@48, end_ms@56. */
typedef enum gnm_mem { GNM_MEM_HOST = 0, GNM_MEM_DEVICE = 1 } gnm_mem;

typedef struct gnm_batch_soa {
    const uint32_t* src_addr;
    const uint32_t* dst_addr;
    const uint32_t* d_pkts;
    const uint32_t* d_octets;
    const uint64_t* start_ms;
    const uint64_t* end_ms;
    uint64_t n;
    int32_t mem; /* gnm_mem */
} gnm_batch_soa;

/* 64-byte records in the exact flowmon::FlowRecord layout (netflow.hpp:59-67). */
typedef struct gnm_batch_aos {
    const void* records;
    uint64_t n;
    int32_t mem; /* gnm_mem */
} gnm_batch_aos;

#define GNM_FLOW_RECORD_BYTES 64

/* ---- Results: replaces AnalysisResult's site level (rate_engine.hpp:76-119) */
typedef struct gnm_site_stats {
    uint64_t flow_count;    /* RateStats::flow_count; 0 => site absent from result.sites */
    uint64_t octets;        /* sum of d_octets over Forward flows (north_star byte sum) */
    uint64_t rate_ubps_lo;  /* exact u128 sum of per-flow micro-bps (RateHistogram::sum_ubps_) */
    uint64_t rate_ubps_hi;
    double min_bps;         /* RateStats, rate_engine.cpp:242-253 */
    double max_bps;
    double avg_bps;         /* double(u128 sum) / 1e6 / count, host-converted like libgcc */
    double median_bps;      /* bucket-midpoint lower median, clamped into [min,max] */
    uint32_t below_threshold; /* median_bps < threshold_bps (K3 flag), 0 when empty */
    uint32_t reserved;
} gnm_site_stats;

typedef struct gnm_tallies { /* ClassTallies rate_engine.hpp:101-110 */
    uint64_t forward;
    uint64_t pure_ack;
    uint64_t administrative;
    uint64_t unmatched;
} gnm_tallies;

typedef struct gnm_result {
    /* inputs */
    uint64_t window_start_ms; /* copied through, no filtering (rate_engine.cpp:257-258) */
    uint64_t window_end_ms;
    double threshold_bps;     /* for below_threshold; GNM_DEFAULT_WARN_THRESHOLD_BPS */
    uint32_t sites_capacity;  /* rows available in sites[] (and histograms[]) */
    gnm_site_stats* sites;    /* caller-owned host array; row = SiteId */
    uint32_t* histograms;     /* optional caller-owned host [capacity * 10001]; NULL skips */
    /* outputs */
    uint32_t n_sites;         /* registry site count at call time (rows written) */
    gnm_tallies tallies;
} gnm_result;

/* Per-host statistics: one row per (site, host) of SiteResult::hosts
 * (rate_engine.hpp:84-99; finalize, rate_engine.cpp:272-289). The host is
 * the flow's matched endpoint: src_addr when the src lookup hits, else
 * dst_addr (reduce_slice, rate_engine.cpp:216-232). */
typedef struct gnm_host_stats {
    uint32_t site;
    uint32_t host;          /* IPv4, host order */
    uint64_t flow_count;    /* RateStats of the host's histogram (stats_from) */
    uint64_t rate_ubps_lo;  /* exact u128 sum of per-flow micro-bps */
    uint64_t rate_ubps_hi;
    double min_bps;
    double max_bps;
    double avg_bps;
    double median_bps;      /* lower median, clamped into [min,max] */
} gnm_host_stats;

/* ---- Device context -------------------------------------------------------- */
typedef struct gnm_ctx gnm_ctx;

/* One context per host thread and GPU; calls on a context are serialized. */
int gnm_ctx_create(int device, gnm_ctx** out);
void gnm_ctx_destroy(gnm_ctx* ctx);
/* Use an external cudaStream_t (NULL = the context's own stream). */
int gnm_ctx_set_stream(gnm_ctx* ctx, void* cuda_stream);
void* gnm_ctx_stream(gnm_ctx* ctx);
/* Host-batch loader chunk (records per pinned double-buffer half). */
int gnm_ctx_set_chunk_records(gnm_ctx* ctx, uint64_t records);
/* Block-private accumulation of hot (heavily hit) sites:
 * GNM_HOT_AUTO (default) plans it per batch from a 1/64 sample when the batch
 * is large and skewed enough; GNM_HOT_OFF never; GNM_HOT_FORCE always (every
 * sampled site up to the slot capacity; a test hook). Results are identical
 * in every mode. */
#define GNM_HOT_OFF 0
#define GNM_HOT_AUTO 1
#define GNM_HOT_FORCE 2
int gnm_ctx_set_hot_mode(gnm_ctx* ctx, int mode);
/* CUDA graphs (default on): a gnm_analyze / gnm_analyze_window call on a
 * DEVICE batch that repeats the previous call's inputs (column pointers,
 * size, registry and version, parameters, window, threshold, hot mode)
 * replays one captured graph of the whole device phase instead of launching
 * its kernels one by one. Results are identical; the batch's contents may
 * change between calls. Not used with timing, per-host mode or histograms. */
int gnm_ctx_set_graphs(gnm_ctx* ctx, int enable);
/* Per-host mode (off by default): K2 also logs each Forward flow's host,
 * rate and micro-bps, and every finalize then builds the per-host rows,
 * sorted by (site, host) like the reference's std::map iteration. Only
 * between accumulations. The rows reflect this context's own accumulation
 * (per-host results are not part of the cross-GPU partials). */
int gnm_ctx_set_hosts(gnm_ctx* ctx, int enable);
/* Rows of the last finalize in per-host mode (0 otherwise). */
uint64_t gnm_host_count(gnm_ctx* ctx);
/* Copy the last finalize's rows into out[capacity] (GNM_ERR_CAPACITY when
 * short) and, when `histograms` is non-NULL, each row's RateHistogram
 * buckets (HostResult::histogram) into histograms[capacity * 10001]. Valid
 * until the next finalize or reset. */
int gnm_host_results(gnm_ctx* ctx, gnm_host_stats* out, uint64_t capacity, uint32_t* histograms);
/* The same histograms in sparse form: the non-zero (row, bucket) counts in
 * (row, bucket) order; row indexes the gnm_host_results rows. With rows ==
 * NULL only *n_entries is set (a query); otherwise GNM_ERR_CAPACITY when
 * capacity < *n_entries. Host arrays. */
int gnm_host_histogram_entries(gnm_ctx* ctx, uint32_t* rows, uint32_t* buckets, uint32_t* counts,
                               uint64_t capacity, uint64_t* n_entries);

/* Per-host rows across GPUs (hosts mode): the two-round protocol of
 * gnm_partials applied to (site, host) rows. Per rank, after gnm_accumulate:
 *   gnm_hosts_local_keys      this context's distinct keys (site << 32 | host),
 *                             sorted, as a device array of *n u64;
 *   [caller: the sorted union of every rank's keys, on this device]
 *   gnm_hosts_set_keys        partials of the union: sums u64[3n] (micro-bps
 *                             in 32-bit limbs) SUM, min f64[n] MIN (+inf
 *                             where this rank has no flow of the row), max
 *                             f64[n] MAX, coarse u32[157n] (super-bucket-
 *                             major) SUM;
 *   [caller: all-reduce them]
 *   gnm_hosts_prepare_median  each row's median super-bucket; fine u32[64n]
 *                             counts this rank's flows inside it;
 *   [caller: all-reduce fine]
 *   gnm_finalize              rows of the union (gnm_host_results; no
 *                             histograms for combined rows).
 * The union may hold up to 2^24 - 1 rows. */
typedef struct gnm_host_partials {
    uint64_t* sums;
    double* min;
    double* max;
    uint32_t* coarse;
    uint32_t* fine;
    uint64_t n;
} gnm_host_partials;
int gnm_hosts_local_keys(gnm_ctx* ctx, const gnm_registry* reg, const uint64_t** keys, uint64_t* n);
int gnm_hosts_set_keys(gnm_ctx* ctx, const uint64_t* keys, uint64_t n, gnm_host_partials* out);
int gnm_hosts_prepare_median(gnm_ctx* ctx);

/* aggregate() (rate_engine.cpp:335-347) + the K3 site synthesis
 * (finalize/stats_from, rate_engine.cpp:242-292) in one synchronous call.
 * Results are identical for any batch split (commutative monoid). */
int gnm_analyze(gnm_ctx* ctx, const gnm_registry* reg, const gnm_filter_params* params,
                const gnm_batch_soa* batch, gnm_result* result);
int gnm_analyze_aos(gnm_ctx* ctx, const gnm_registry* reg, const gnm_filter_params* params,
                    const gnm_batch_aos* batch, gnm_result* result);

/* Split form, for streaming and multi-GPU: accumulate any number of batches
 * into the context's device partials (K2, asynchronous on the context
 * stream), optionally all-reduce the partials across GPUs, then finalize
 * (K3 + result D2H + partial reset; synchronous). */
int gnm_accumulate(gnm_ctx* ctx, const gnm_registry* reg, const gnm_filter_params* params,
                   const gnm_batch_soa* batch);
/* FlowStore::snapshot(window_start_ms, window_end_ms) fused into the
 * accumulation (flow_store.cpp:62-80): only records with end_ms in
 * [window_start_ms, window_end_ms) are classified or counted, as if the
 * reference's aggregate ran on the snapshot's copy. */
int gnm_accumulate_window(gnm_ctx* ctx, const gnm_registry* reg, const gnm_filter_params* params,
                          const gnm_batch_soa* batch, uint64_t window_start_ms,
                          uint64_t window_end_ms);
int gnm_accumulate_window_aos(gnm_ctx* ctx, const gnm_registry* reg, const gnm_filter_params* params,
                              const gnm_batch_aos* batch, uint64_t window_start_ms,
                              uint64_t window_end_ms);
/* snapshot(result->window_start_ms, result->window_end_ms) + aggregate + finalize in one call:
 * monitor.cpp:109-120 (run_cycle) on the GPU. */
int gnm_analyze_window(gnm_ctx* ctx, const gnm_registry* reg, const gnm_filter_params* params,
                       const gnm_batch_soa* batch, gnm_result* result);
int gnm_accumulate_aos(gnm_ctx* ctx, const gnm_registry* reg, const gnm_filter_params* params,
                       const gnm_batch_aos* batch);
/* GNM_ERR_CAPACITY (after the rows are written) when one accumulation held
 * 2^32 or more Forward flows: the u32 coarse counts could have wrapped. */
int gnm_finalize(gnm_ctx* ctx, const gnm_registry* reg, gnm_result* result);
/* Drop accumulated partials without producing a result. */
int gnm_reset(gnm_ctx* ctx);

/* Device partials of the current accumulation, for a cross-GPU all-reduce
 * (SURVEY.md §8e). All are device pointers on the context's device.
 *   sums:   uint64 [n_sites*4 + 4]   reduce SUM  (per site: octets, ubps limb0,
 *           limb1, limb2 (32-bit limbs); then tallies fwd, ack, admin, unmatched)
 *   min:    float64 [n_sites]        reduce MIN  (+inf when empty)
 *   max:    float64 [n_sites]        reduce MAX  (0 when empty)
 *   coarse: uint32 [157*n_sites]     reduce SUM  flows per (super-bucket, site),
 *           super-bucket = bucket >> 6, index sb*n_sites + site
 *   fine:   uint32 [n_sites*64]      reduce SUM  the median super-bucket's
 *           64 bucket counts; valid after gnm_prepare_median
 * The exact median is a two-round selection. Multi-GPU protocol, per rank:
 *   gnm_accumulate (own shard) -> all-reduce sums/min/max/coarse ->
 *   gnm_prepare_median (finds the global median super-bucket, counts this
 *   rank's flows inside it) -> all-reduce fine -> gnm_finalize.
 * A single context just calls gnm_finalize, which prepares itself. */
typedef struct gnm_partials {
    uint64_t* sums;
    double* min_bps;
    double* max_bps;
    uint32_t* coarse;
    uint32_t* fine;
    uint64_t n_sites;
    uint64_t sums_count;
    uint64_t coarse_count;
    uint64_t fine_count;
} gnm_partials;
int gnm_get_partials(gnm_ctx* ctx, const gnm_registry* reg, gnm_partials* out);
/* Round 2 of the median on this context's log (see gnm_partials); no further
 * gnm_accumulate until gnm_finalize or gnm_reset. Not with a communicator
 * (gnm_ctx_comm_init), whose finalize runs both rounds itself. */
int gnm_prepare_median(gnm_ctx* ctx, const gnm_registry* reg);

/* ---- Multi-GPU inside the library ---------------------------
 * Records shard by index across the GPUs -- rank i of N takes
 * [n*i/N, n*(i+1)/N), the reference's worker boundaries (rate_engine.cpp:
 * 341-344) -- and the per-site partials combine in two rounds of NCCL
 * all-reduces over NVLink (round 1: sums and coarse counts SUM, min MIN, max
 * MAX, as one ncclGroupStart/End call; round 2: the median super-buckets'
 * fine counts SUM), enqueued on the context's stream between K2 and K3b.
 * With a communicator attached, gnm_finalize / gnm_analyze* run the combine
 * themselves: every rank returns the same global result. In per-host mode
 * the ranks' (site, host) keys are all-gathered into their sorted union
 * first; the host rows are then global, and a rank's host histograms
 * (gnm_host_results / gnm_host_histogram_entries) count that rank's own
 * flows over the global rows (gnm_group_host_histogram_entries sums them).
 * NCCL (libnccl.so.2) is loaded on first use. */

#define GNM_COMM_ID_BYTES 128 /* sizeof(ncclUniqueId) */

/* One process per GPU: rank 0 creates the id, the caller distributes it to
 * every rank out of band, and each rank attaches its context (the calls
 * block until all N ranks have joined). */
int gnm_comm_unique_id(unsigned char out[GNM_COMM_ID_BYTES]);
int gnm_ctx_comm_init(gnm_ctx* ctx, int nranks, int rank, const unsigned char id[GNM_COMM_ID_BYTES]);
/* Detach (and destroy) the context's communicator. */
int gnm_ctx_comm_destroy(gnm_ctx* ctx);
/* Ranks in the context's communicator (1 without one). */
int gnm_ctx_comm_size(gnm_ctx* ctx);

/* One process driving N GPUs: one context per device and one NCCL clique
 * (ncclCommInitAll). GNM_GROUP_LOOPBACK exchanges through host memory
 * instead -- a test hook that runs the same orchestration with several
 * ranks on one device (NCCL rejects two ranks on one GPU). */
typedef struct gnm_group gnm_group;
#define GNM_GROUP_NCCL 0
#define GNM_GROUP_LOOPBACK 1
int gnm_group_create(const int* devices, int n_devices, int kind, gnm_group** out);
void gnm_group_destroy(gnm_group* group);
int gnm_group_size(const gnm_group* group);
/* Rank i's context (per-context settings: hosts mode, hot mode, chunking). */
gnm_ctx* gnm_group_ctx(gnm_group* group, int rank);
/* aggregate over the group's GPUs: shard i of the batch to rank i, every
 * rank accumulates its shard and finalizes with the combine (one host
 * thread per rank); `result` receives the global rows. Host or device
 * batches (device batches must be readable from every rank's GPU). If a
 * rank fails, the group's communicators are aborted (no rank is left
 * blocked in a collective), the root cause is returned, and later calls on
 * the group fail with GNM_ERR_COMM. */
int gnm_group_analyze(gnm_group* group, const gnm_registry* reg, const gnm_filter_params* params,
                      const gnm_batch_soa* batch, gnm_result* result);
int gnm_group_analyze_aos(gnm_group* group, const gnm_registry* reg, const gnm_filter_params* params,
                          const gnm_batch_aos* batch, gnm_result* result);
/* Per-host rows of the last group analysis (hosts mode on every rank's
 * context): the global rows, and their histograms summed over the ranks as
 * sparse (row, bucket, count) entries in (row, bucket) order. */
uint64_t gnm_group_host_count(gnm_group* group);
int gnm_group_host_results(gnm_group* group, gnm_host_stats* out, uint64_t capacity);
int gnm_group_host_histogram_entries(gnm_group* group, uint32_t* rows, uint32_t* buckets, uint32_t* counts,
                                     uint64_t capacity, uint64_t* n_entries);

/* Per-record classification (classify/attribute, rate_engine.cpp:71-86,
 * 127-146): out[i] = class << 30 | (site & 0x3FFFFFFF), site = 0x3FFFFFFF
 * unless Forward. `out` is a host or device pointer per out_mem. */
int gnm_classify(gnm_ctx* ctx, const gnm_registry* reg, const gnm_filter_params* params,
                 const gnm_batch_soa* batch, uint32_t* out, int32_t out_mem);

/* Device time of the last analyze/accumulate/finalize, from CUDA events on
 * the context stream. */
typedef struct gnm_timing {
    double accumulate_ms; /* K2 (sum over launches since the last finalize) */
    double finalize_ms;   /* K3a + K2b + K3b */
    double h2d_ms;        /* loader copies (host batches) */
    uint64_t k2_launches;
    uint64_t kernel_launches; /* every kernel this library launched since ctx creation */
    uint64_t records;         /* records accumulated since the last finalize */
    double plan_ms;           /* K1 hot-site planning (sample, assign, table slots) */
    /* Running totals since timing was last enabled, over every finalize:
     * K1, K2 and finalize device time, and the number of finalizes. */
    double total_plan_ms;
    double total_accumulate_ms;
    double total_finalize_ms;
    uint64_t total_finalizes;
    uint64_t total_k2_launches;
    /* bytes the loader has copied host -> device since ctx creation (host
     * batches; non-windowed SoA batches send a u32 duration in place of the
     * two u64 timestamps: 20 bytes per record instead of 32) */
    uint64_t h2d_bytes;
} gnm_timing;
int gnm_ctx_timing(gnm_ctx* ctx, gnm_timing* out);
/* 1 = record CUDA events around every kernel (default 0); enabling resets
 * the running totals. */
int gnm_ctx_enable_timing(gnm_ctx* ctx, int enable);

/* ---- NetFlow v5 ingest: Collector::ingest_datagram, batched ---------------
 * (collector.cpp:101-129; decode_packet netflow.cpp:78-113, resolve_times
 * :150-161; paths relative to /root/reference/proj/core/src). Decodes n
 * datagrams on the GPU: datagram i is bytes [offsets[i], offsets[i+1]) of
 * `datagrams` (both in memory `in_mem`). A datagram the reference would
 * reject with CodecError is dropped (status 1 bad version, 2 truncated,
 * 3 bad count; 0 ok); records with d_pkts == 0 or d_octets < d_pkts are
 * rejected as the collector does; the rest are written as 64-byte
 * flowmon::FlowRecord rows (netflow.hpp:59-67) to `out_records` (memory
 * `out_mem`, `capacity` rows) in datagram order, then record order -- the
 * order the collector appends them to the FlowStore. `status` (optional)
 * is a host array of n bytes. GNM_ERR_CAPACITY when the accepted records
 * do not fit. */
typedef struct gnm_netflow_stats {
    uint64_t datagrams;
    uint64_t decode_errors;    /* CollectorMetrics::decode_errors */
    uint64_t records_rejected; /* CollectorMetrics::records_rejected */
    uint64_t records_accepted; /* records written */
} gnm_netflow_stats;
int gnm_decode_netflow(gnm_ctx* ctx, const uint8_t* datagrams, uint64_t bytes, const uint64_t* offsets,
                       uint64_t n, int32_t in_mem, void* out_records, uint64_t capacity, int32_t out_mem,
                       uint8_t* status, gnm_netflow_stats* stats);

/* ---- FLOWARC1 archives (flow_store.cpp:144-207) ---------------------------
 * An archive in memory (host or device, device buffers 4-byte aligned):
 * "FLOWARC1", be32 version 1, be64 count, then count 64-byte big-endian
 * entries (be64 start_ms, be64 end_ms, 48-byte raw record). The header and
 * length checks are FlowStore::load's, as status codes.
 * gnm_decode_archive: FlowStore::load -> FlowRecord rows (64 B) in
 *   `out_records` (memory `out_mem`, `capacity` rows); *n_out = count.
 * gnm_accumulate_archive / gnm_analyze_archive: aggregate over the
 *   archive's records with K2 reading the entries in place (no decode pass;
 *   host archives stream through the chunked H2D loader). */
int gnm_decode_archive(gnm_ctx* ctx, const uint8_t* bytes, uint64_t len, int32_t in_mem, void* out_records,
                       uint64_t capacity, int32_t out_mem, uint64_t* n_out);
int gnm_accumulate_archive(gnm_ctx* ctx, const gnm_registry* reg, const gnm_filter_params* params,
                           const uint8_t* bytes, uint64_t len, int32_t mem);
int gnm_analyze_archive(gnm_ctx* ctx, const gnm_registry* reg, const gnm_filter_params* params,
                        const uint8_t* bytes, uint64_t len, int32_t mem, gnm_result* result);

/* ---- Warning rule: evaluate_warnings (monitor.cpp:13-34) ----------------- */
typedef struct gnm_warning_state gnm_warning_state;
typedef struct gnm_warning {
    uint32_t site;
    uint32_t consecutive_bad_hours;
    double median_bps;
} gnm_warning;

int gnm_warning_state_create(gnm_warning_state** out);
void gnm_warning_state_destroy(gnm_warning_state* st);
uint32_t gnm_warning_state_streak(const gnm_warning_state* st, uint32_t site);
/* For every site with flow_count > 0 (ascending SiteId, as std::map
 * iteration): median < threshold extends the streak, else resets it; every
 * site at streak >= 2 warns. Zero-flow sites are frozen. Writes up to cap
 * warnings and the total count to *n_out. */
int gnm_evaluate_warnings(const gnm_result* result, gnm_warning_state* st, double threshold_bps,
                          gnm_warning* out, size_t cap, size_t* n_out);

#ifdef __cplusplus
}
#endif

#endif /* GNETMON_H */

// capi.cu — the extern "C" boundary (include/gnetmon.h): registry, device
// context, pinned double-buffered loader, K2/K3 orchestration and the
// host-side streak rule. No exceptions cross the ABI; every entry point
// returns a gnm_status and leaves a thread-local message on failure.
//
// There is no CPU fallback: without a CUDA device gnm_ctx_create fails with
// GNM_ERR_NO_DEVICE and nothing else can run.
#include <cuda_runtime.h>

#include <algorithm>
#include <mutex>
#include <functional>
#include <condition_variable>
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <new>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "comm.hpp"
#include "gnetmon.h"
#include "kernels.cuh"
#include "hosts.cuh"
#include "netflow.cuh"
#include "registry.hpp"

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

struct CudaError : std::runtime_error {
    explicit CudaError(const std::string& m) : std::runtime_error(m) {}
};

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        if (e == cudaErrorMemoryAllocation) throw std::bad_alloc();
        throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
    }
}

template <typename F>
int guarded(F&& f) {
    try {
        return f();
    } catch (const CudaError& e) {
        return fail(GNM_ERR_CUDA, e.what());
    } catch (const gnm::CommError& e) {
        return fail(GNM_ERR_COMM, e.what());
    } catch (const std::bad_alloc&) {
        return fail(GNM_ERR_OUT_OF_MEMORY, "out of memory");
    } catch (const std::exception& e) {
        return fail(GNM_ERR_INVALID_ARGUMENT, e.what());
    }
}

} // namespace

struct gnm_registry {
    gnm::Registry r;
};

struct gnm_warning_state {
    std::map<uint32_t, uint32_t> streaks; // WarningState (monitor.hpp:20-37)
};

struct EventPair {
    cudaEvent_t a = nullptr, b = nullptr;
};

// Persistent host workers for the loader's staging work (parallel_for):
// run(nt, fn) executes fn(t, nt) for t = 0..nt-1 and returns when all are
// done; the caller takes t = 0 and then claims any task no worker has
// started yet. A loader chunk is a millisecond or two of copying, and a
// condition-variable wake-up costs tens to hundreds of microseconds, so an
// idle worker spins on the run counter for kSpin before it sleeps.
inline void cpu_relax() {
#if defined(__x86_64__) || defined(__i386__)
    __builtin_ia32_pause();
#endif
}

class WorkerPool {
public:
    explicit WorkerPool(unsigned n) {
        for (unsigned i = 0; i < n; ++i) th_.emplace_back([this, i] { loop(i); });
    }
    ~WorkerPool() {
        {
            std::lock_guard<std::mutex> l(m_);
            stop_.store(true);
        }
        cv_.notify_all();
        for (auto& t : th_) t.join();
    }
    size_t size() const { return th_.size(); }
    template <typename F>
    void run(unsigned nt, F& fn) {
        if (nt <= 1) {
            fn(0u, 1u);
            return;
        }
        job_ = [&fn](unsigned t, unsigned n) { fn(t, n); };
        done_.store(0);
        // state = run id (24 bits) | nt (8 bits) | next task (32 bits); one
        // fetch_add claims a task of exactly the run it belongs to
        last_nt_.store(nt);
        run_id_ = (run_id_ + 1) & 0xFFFFFFu;
        state_.store(static_cast<uint64_t>(run_id_) << 40 | static_cast<uint64_t>(nt) << 32 | 1u);
        if (sleepers_.load() > 0) {
            std::lock_guard<std::mutex> l(m_);
            cv_.notify_all();
        }
        fn(0u, nt);
        for (;;) { // help with tasks nobody has claimed
            const uint64_t st = state_.fetch_add(1);
            const unsigned t = static_cast<unsigned>(st);
            if (t >= nt) break;
            fn(t, nt);
            done_.fetch_add(1);
        }
        for (unsigned k = 0; done_.load() != nt - 1; ++k) {
            cpu_relax();
            if (k > 4096) std::this_thread::yield();
        }
        job_ = nullptr;
    }

private:
    // GNM_POOL_SPIN_US overrides the spin before sleeping (0: sleep at once)
    const std::chrono::microseconds kSpin{[] {
        const char* e = std::getenv("GNM_POOL_SPIN_US");
        return e ? std::atol(e) : 3000L;
    }()};
    // Worker `index` spins only if the last run used that many threads: a
    // small run (the result copy) leaves the rest of a loader-sized pool
    // asleep instead of spinning on the cores the caller's host work needs.
    void loop(unsigned index) {
        uint32_t seen = 0;
        for (;;) {
            uint64_t st = state_.load();
            if (static_cast<uint32_t>(st >> 40) == seen) {
                const bool spin = index + 1 < last_nt_.load();
                const auto t0 = std::chrono::steady_clock::now();
                for (unsigned k = 1;; ++k) {
                    cpu_relax(); // leave the core's other hardware thread its issue slots
                    st = state_.load();
                    if (static_cast<uint32_t>(st >> 40) != seen || stop_.load()) break;
                    if (!spin || ((k & 1023u) == 0 && std::chrono::steady_clock::now() - t0 > kSpin)) {
                        std::unique_lock<std::mutex> l(m_);
                        sleepers_.fetch_add(1);
                        cv_.wait(l, [&] { return static_cast<uint32_t>(state_.load() >> 40) != seen || stop_.load(); });
                        sleepers_.fetch_sub(1);
                        st = state_.load();
                        break;
                    }
                }
            }
            if (stop_.load()) return;
            for (;;) {
                // a claim belongs to the run it was taken from (a newer run's
                // task is that run's to execute: its caller waits for it)
                const uint64_t c = state_.fetch_add(1);
                const unsigned t = static_cast<unsigned>(c), n = static_cast<unsigned>(c >> 32) & 0xFFu;
                seen = static_cast<uint32_t>(c >> 40);
                if (t >= n) break;
                job_(t, n);
                done_.fetch_add(1);
            }
        }
    }
    std::vector<std::thread> th_;
    std::mutex m_;
    std::condition_variable cv_;
    std::function<void(unsigned, unsigned)> job_;
    std::atomic<uint64_t> state_{0};
    std::atomic<unsigned> done_{0};
    std::atomic<int> sleepers_{0};
    std::atomic<unsigned> last_nt_{0};
    std::atomic<bool> stop_{false};
    uint32_t run_id_ = 0;
};

struct gnm_ctx {
    int device = 0;
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;
    cudaStream_t copy_stream = nullptr;

    // registry cache (device table)
    const gnm_registry* reg = nullptr;
    uint64_t reg_version = ~0ull;
    uint32_t* d_table = nullptr;
    size_t table_cap_words = 0;
    gnm::DevTable table{};
    int hot_mode = GNM_HOT_AUTO;

    // partials
    gnm::DevPartials P{};
    // per-flow log of the current accumulation (round 2 of the median):
    // entries (and, for wide registries, buckets) in per-launch slices
    struct LogSlice {
        size_t entry_off, count_off;
        uint32_t warp_cap, regions;
    };
    unsigned int* d_log = nullptr;
    unsigned int* d_logb = nullptr;
    size_t log_cap = 0, log_used = 0;
    size_t logb_cap = 0; // d_logb grows only for wide registries: its own capacity
    bool log_wide = false;
    unsigned int* d_counts = nullptr;
    size_t counts_cap = 0, counts_used = 0;
    std::vector<LogSlice> slices;
    // hosts mode (gnm_ctx_set_hosts): per-entry host, octets, duration
    bool hosts = false;
    unsigned int* d_lhost = nullptr;
    unsigned int* d_loct = nullptr;
    unsigned long long* d_ldur = nullptr;
    size_t lhost_cap = 0;
    gnm::HostRows hrows;
    gnm::HostLocal hlocal;   // hosts local phase done (gnm_hosts_local_keys)
    gnm::HostGlobal hglobal; // cross-context rows (gnm_hosts_set_keys)

    // CUDA graph of a repeated device-batch analysis (analyze_graphed)
    bool graphs = true;
    struct GraphKey {
        const void* cols[6];
        uint64_t n;
        const gnm_registry* reg;
        uint64_t version;
        gnm_filter_params params;
        uint64_t win_lo, win_hi;
        int windowed;
        double threshold;
        int hot_mode;
        uint32_t n_sites;
        uint64_t alloc_gen;
        int aos;
        bool operator==(const GraphKey& o) const { return std::memcmp(this, &o, sizeof o) == 0; }
    };
    struct GraphEntry {
        GraphKey key;
        cudaGraphExec_t exec = nullptr;
        uint64_t kernels = 0; // kernels per replay (launch accounting)
        uint64_t last_use = 0;
    };
    std::vector<GraphEntry> graph_cache; // up to kGraphCache recent input sets
    uint64_t graph_clock = 0;
    // Bumped whenever a buffer or baked-in size a captured graph refers to
    // changes (table upload, partials, log, output staging).
    uint64_t alloc_gen = 0;
    bool capturing = false; // inside analyze_graphed's stream capture: no (re)allocation allowed

    bool prepared = false; // K3a + K2b ran (gnm_prepare_median) for this accumulation
    uint32_t* d_scratch = nullptr; // hot-site plan: counts, site->slot, slot->site, counter
    uint32_t partial_cap = 0;
    bool accumulating = false;
    const gnm_registry* acc_reg = nullptr;
    uint64_t acc_version = 0;

    // finalize output staging: n_sites rows + 32 B of tallies
    gnm_site_stats* d_out = nullptr;
    gnm_site_stats* h_out = nullptr;
    size_t out_cap_rows = 0;

    // loader: two device slots of `chunk` records, pinned host staging
    uint64_t chunk = 1ull << 22;
    unsigned char* d_stage[2] = {nullptr, nullptr};
    unsigned char* h_stage[2] = {nullptr, nullptr};
    size_t stage_bytes = 0;
    size_t h_stage_bytes = 0;
    cudaEvent_t ev_h2d[2] = {nullptr, nullptr};
    cudaEvent_t ev_k2[2] = {nullptr, nullptr};

    // timing
    bool timing = false;
    std::vector<EventPair> pool;
    std::vector<EventPair> k2_pairs, k3_pairs, h2d_pairs, plan_pairs;
    double acc_ms = 0, fin_ms = 0, h2d_ms = 0, plan_ms = 0;
    double tot_plan_ms = 0, tot_acc_ms = 0, tot_fin_ms = 0;
    uint64_t tot_finalizes = 0, tot_k2 = 0, k2_since_fin = 0;
    int occ[2] = {0, 0}; // K2 blocks/SM (cold, hot) for the current table size
    uint64_t k2_launches = 0, kernel_launches = 0, records = 0;
    uint64_t h2d_bytes = 0; // loader copies since creation (gnm_timing)
    unsigned stage_share = 1; // contexts loading at once in this process (a group's size)
    std::unique_ptr<WorkerPool> pool_workers; // the loader's host threads (parallel_for)

    // multi-GPU: with a communicator, gnm_finalize runs the two-round
    // combine across the ranks itself (gnm_ctx_comm_init / gnm_group_*)
    std::unique_ptr<gnm::Comm> comm;
    bool discard_hist_out = false; // group ranks > 0: join the histogram all-reduce, keep no copy
};

namespace {

EventPair take_pair(gnm_ctx* c) {
    if (!c->pool.empty()) {
        EventPair p = c->pool.back();
        c->pool.pop_back();
        return p;
    }
    EventPair p;
    ck(cudaEventCreate(&p.a), "cudaEventCreate");
    ck(cudaEventCreate(&p.b), "cudaEventCreate");
    return p;
}

double drain_pairs(gnm_ctx* c, std::vector<EventPair>& v) {
    double total = 0;
    for (EventPair& p : v) {
        float ms = 0;
        ck(cudaEventSynchronize(p.b), "cudaEventSynchronize");
        ck(cudaEventElapsedTime(&ms, p.a, p.b), "cudaEventElapsedTime");
        total += ms;
        c->pool.push_back(p);
    }
    v.clear();
    return total;
}

gnm::DevParams dev_params(const gnm_ctx* c, const gnm_filter_params* p) {
    gnm_filter_params d;
    gnm_filter_params_default(&d);
    if (!p) p = &d;
    gnm::DevParams q;
    q.ack_plus1 = static_cast<uint64_t>(p->ack_avg_size_max) + 1;
    q.min_packets = p->min_packets;
    q.min_duration_ms = p->min_duration_ms;
    q.site_mask = c->table.packed ? gnm::kPackedSiteMask : 0x7FFFFFFFu;
    q.min_packets1 = std::max<uint32_t>(p->min_packets, 1);
    q.min_duration1 = std::max<uint32_t>(p->min_duration_ms, 1);
    q.wide_log = c->P.n_sites >= gnm::kLogPackedSites;
    q.windowed = 0;
    q.win_lo = q.win_hi = 0;
    q.ablation = 0;
#ifdef GNM_K2_ABLATION
    if (const char* a = std::getenv("GNM_K2_ABLATION")) q.ablation = static_cast<uint32_t>(std::atoi(a));
#endif
    return q;
}

// Upload the registry's device table when the context has not seen this
// registry version (the catalog is rebuilt on update).
void ensure_table(gnm_ctx* c, const gnm_registry* reg) {
    if (c->reg == reg && c->reg_version == reg->r.version() && c->d_table) return;
    gnm::DeviceTable t = reg->r.compile_device_table();
    while (t.words.size() % 4) t.words.push_back(0); // uint4 smem copy
    if (t.words.size() > c->table_cap_words) {
        if (c->d_table) ck(cudaFree(c->d_table), "cudaFree");
        c->d_table = nullptr;
        ck(cudaMalloc(&c->d_table, t.words.size() * 4), "cudaMalloc(table)");
        c->table_cap_words = t.words.size();
    }
    // The previous table may still be read by queued kernels.
    ck(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");
    ck(cudaMemcpy(c->d_table, t.words.data(), t.words.size() * 4, cudaMemcpyHostToDevice),
       "cudaMemcpy(table)");
    c->table.words = c->d_table;
    c->table.n_words = static_cast<uint32_t>(t.words.size());
    c->table.node_begin = t.node_begin;
    c->table.leaf_begin = t.leaf_begin;
    c->table.packed = t.packed;
    c->occ[0] = c->occ[1] = 0;
    c->reg = reg;
    c->reg_version = reg->r.version();
    c->alloc_gen += 1;
}

// Partials sized for the registry's site count; all-zero (min=+inf) at rest.
void ensure_partials(gnm_ctx* c, uint32_t n_sites) {
    if (n_sites > c->partial_cap || !c->P.sums) {
        ck(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");
        if (c->P.sums) {
            cudaFree(c->P.sums);
            cudaFree(c->P.mn);
            cudaFree(c->P.mx);
            cudaFree(c->P.coarse);
            cudaFree(c->P.fine);
            cudaFree(c->P.msb);
            cudaFree(c->P.mrank);
            cudaFree(c->P.cnt);
            cudaFree(c->P.heavy_next);
            cudaFree(c->P.map16);
            cudaFree(c->d_scratch);
            c->d_scratch = nullptr;
        }
        c->P = gnm::DevPartials{};
        const uint32_t cap = std::max<uint32_t>(n_sites, 1);
        ck(cudaMalloc(&c->P.sums, (static_cast<size_t>(cap) * 4 + 4) * 8), "cudaMalloc(sums)");
        ck(cudaMalloc(&c->P.mn, static_cast<size_t>(cap) * 8), "cudaMalloc(min)");
        ck(cudaMalloc(&c->P.mx, static_cast<size_t>(cap) * 8), "cudaMalloc(max)");
        ck(cudaMalloc(&c->P.coarse, static_cast<size_t>(cap) * gnm::kCoarse * 4), "cudaMalloc(coarse)");
        ck(cudaMalloc(&c->P.fine, static_cast<size_t>(cap) * gnm::kFineW * 4), "cudaMalloc(fine)");
        ck(cudaMalloc(&c->P.msb, static_cast<size_t>(cap) * 4), "cudaMalloc(msb)");
        ck(cudaMalloc(&c->P.mrank, static_cast<size_t>(cap) * 4), "cudaMalloc(mrank)");
        ck(cudaMalloc(&c->P.cnt, static_cast<size_t>(cap) * 8), "cudaMalloc(cnt)");
        ck(cudaMalloc(&c->P.heavy_next, 4 * (1 + 64)), "cudaMalloc(heavy)"); // counter, row -> site
        const size_t map_bytes = (static_cast<size_t>(cap) + 8) * 2; // whole 16-byte vectors
        ck(cudaMalloc(&c->P.map16, map_bytes), "cudaMalloc(map16)");
        ck(cudaMemsetAsync(c->P.map16, 0, map_bytes, c->stream), "cudaMemsetAsync(map16)");
        const size_t scratch_words = gnm::plan_scratch_words(cap);
        ck(cudaMalloc(&c->d_scratch, scratch_words * 4), "cudaMalloc(scratch)");
        ck(cudaMemsetAsync(c->d_scratch, 0, scratch_words * 4, c->stream), "cudaMemsetAsync");
        c->P.n_sites = cap;
        ck(gnm::launch_init_partials(c->P, c->stream), "init partials");
        c->kernel_launches += 1;
        c->partial_cap = cap;
        c->alloc_gen += 1;
    }
    if (c->P.n_sites != n_sites) {
        // Tallies live after the last site row: move them (zero at rest).
        c->P.n_sites = n_sites;
        ck(cudaMemsetAsync(c->P.sums + static_cast<size_t>(n_sites) * 4, 0, 32, c->stream),
           "cudaMemsetAsync");
        c->alloc_gen += 1;
        // The hot-plan layout depends on n_sites: start from zero counts.
        ck(cudaMemsetAsync(c->d_scratch, 0, gnm::plan_scratch_words(c->partial_cap) * 4, c->stream),
           "cudaMemsetAsync(scratch)");
    }
}

void ensure_out(gnm_ctx* c, uint32_t n_sites) {
    const size_t rows = static_cast<size_t>(n_sites) + 1; // + tallies
    if (rows <= c->out_cap_rows) return;
    if (c->capturing) throw CudaError("cudaMalloc(out): no allocation during graph capture");
    ck(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");
    if (c->d_out) cudaFree(c->d_out);
    if (c->h_out) cudaFreeHost(c->h_out);
    c->d_out = nullptr;
    c->h_out = nullptr;
    ck(cudaMalloc(&c->d_out, rows * sizeof(gnm_site_stats)), "cudaMalloc(out)");
    // The last row holds only the 32 bytes of tallies; the rest stays zero.
    ck(cudaMemset(c->d_out, 0, rows * sizeof(gnm_site_stats)), "cudaMemset(out)");
    ck(cudaMallocHost(&c->h_out, rows * sizeof(gnm_site_stats)), "cudaMallocHost(out)");
    c->out_cap_rows = rows;
    c->alloc_gen += 1;
}

void ensure_stage(gnm_ctx* c, size_t bytes_per_slot, bool need_host) {
    if (bytes_per_slot > c->stage_bytes) {
        ck(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");
        ck(cudaStreamSynchronize(c->copy_stream), "cudaStreamSynchronize");
        for (int i = 0; i < 2; ++i) {
            if (c->d_stage[i]) cudaFree(c->d_stage[i]);
            c->d_stage[i] = nullptr;
        }
        for (int i = 0; i < 2; ++i) ck(cudaMalloc(&c->d_stage[i], bytes_per_slot), "cudaMalloc(stage)");
        c->stage_bytes = bytes_per_slot;
    }
    if (need_host && bytes_per_slot > c->h_stage_bytes) {
        ck(cudaStreamSynchronize(c->copy_stream), "cudaStreamSynchronize");
        for (int i = 0; i < 2; ++i) {
            if (c->h_stage[i]) cudaFreeHost(c->h_stage[i]);
            c->h_stage[i] = nullptr;
        }
        for (int i = 0; i < 2; ++i)
            ck(cudaMallocHost(&c->h_stage[i], bytes_per_slot), "cudaMallocHost(stage)");
        c->h_stage_bytes = bytes_per_slot;
    }
}

bool is_pinned(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

int begin_accumulate(gnm_ctx* c, const gnm_registry* reg) {
    if (c->accumulating && (c->acc_reg != reg || c->acc_version != reg->r.version()))
        return fail(GNM_ERR_INVALID_ARGUMENT,
                    "registry changed during an accumulation; finalize or reset first");
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    ensure_table(c, reg);
    ensure_partials(c, static_cast<uint32_t>(reg->r.sites().size()));
    if (!c->accumulating) {
        c->accumulating = true;
        c->acc_reg = reg;
        c->acc_version = reg->r.version();
        c->records = 0;
    }
    return GNM_OK;
}

gnm::DevLog slice_view(const gnm_ctx* c, const gnm_ctx::LogSlice& sl) {
    gnm::DevLog lg;
    lg.entries = c->d_log + sl.entry_off;
    lg.buckets = c->log_wide ? c->d_logb + sl.entry_off : nullptr;
    lg.counts = c->d_counts + sl.count_off;
    lg.warp_cap = sl.warp_cap;
    lg.regions = sl.regions;
    lg.hosts = c->hosts ? c->d_lhost + sl.entry_off : nullptr;
    lg.octs = c->hosts ? c->d_loct + sl.entry_off : nullptr;
    lg.durs = c->hosts ? c->d_ldur + sl.entry_off : nullptr;
    return lg;
}

// Grow a device buffer preserving its first `used` elements (stream-ordered).
template <typename T>
void grow_buf(gnm_ctx* c, T** buf, size_t* cap, size_t used, size_t need, const char* what) {
    if (need <= *cap) return;
    if (c->capturing) throw CudaError(std::string(what) + ": no allocation during graph capture");
    const size_t ncap = std::max(need, *cap + *cap / 2);
    T* nb = nullptr;
    ck(cudaMallocAsync(reinterpret_cast<void**>(&nb), ncap * sizeof(T), c->stream), what);
    if (*buf) {
        if (used) ck(cudaMemcpyAsync(nb, *buf, used * sizeof(T), cudaMemcpyDeviceToDevice, c->stream), what);
        ck(cudaFreeAsync(*buf, c->stream), what);
    }
    *buf = nb;
    *cap = ncap;
    c->alloc_gen += 1;
}

void grow_u32(gnm_ctx* c, unsigned int** buf, size_t* cap, size_t used, size_t need, const char* what) {
    grow_buf(c, buf, cap, used, need, what);
}

// This launch's slice of the per-flow log: one region of warp_cap entries per
// warp of the grid, the per-warp counts after the previous slices'.
gnm::DevLog reserve_log(gnm_ctx* c, const gnm::LaunchCfg& cfg, const gnm::DevBatch& b) {
    gnm_ctx::LogSlice sl;
    sl.warp_cap = gnm::k2_warp_cap(cfg, b);
    sl.regions = gnm::k2_regions(cfg);
    sl.entry_off = c->log_used;
    sl.count_off = c->counts_used;
    const size_t need = static_cast<size_t>(sl.warp_cap) * sl.regions;
    const bool wide = c->P.n_sites >= gnm::kLogPackedSites;
    if (c->slices.empty()) c->log_wide = wide;
    grow_u32(c, &c->d_log, &c->log_cap, c->log_used, c->log_used + need, "log");
    if (wide) grow_u32(c, &c->d_logb, &c->logb_cap, c->log_used, c->log_cap, "log buckets");
    grow_u32(c, &c->d_counts, &c->counts_cap, c->counts_used, c->counts_used + sl.regions, "log counts");
    if (c->hosts && c->lhost_cap < c->log_cap) {
        const size_t used = c->log_used, want = c->log_cap;
        size_t k = c->lhost_cap;
        grow_buf(c, &c->d_lhost, &k, used, want, "log hosts");
        k = c->lhost_cap;
        grow_buf(c, &c->d_loct, &k, used, want, "log octets");
        k = c->lhost_cap;
        grow_buf(c, &c->d_ldur, &k, used, want, "log durations");
        c->lhost_cap = k;
    }
    c->log_used += need;
    c->counts_used += sl.regions;
    c->slices.push_back(sl);
    return slice_view(c, sl);
}

void launch_k2_timed(gnm_ctx* c, const gnm::DevBatch& b, const gnm::DevParams& p) {
    if (b.n == 0) return;
    EventPair pe, ev;
    if (c->timing) {
        pe = take_pair(c);
        ck(cudaEventRecord(pe.a, c->stream), "cudaEventRecord");
    }
    // K1: hot-site plan for this batch (skipped when no site can be hot).
    const gnm::LaunchCfg cold = gnm::k2_config(c->device, b, c->table.n_words, false, c->occ, c->hosts);
    bool hot = false;
    if (c->hot_mode != GNM_HOT_OFF) {
        cudaError_t e;
        hot = gnm::plan_hot(c->device, b, c->table, p, c->P.n_sites, c->d_scratch, c->P.mn, c->P.mx, cold.grid,
                            c->hot_mode == GNM_HOT_FORCE, cold.table_in_smem, c->stream, &c->kernel_launches, &e);
        ck(e, "hot-site plan");
    }
    const gnm::LaunchCfg cfg =
        hot ? gnm::k2_config(c->device, b, c->table.n_words, true, c->occ, c->hosts) : cold;
    gnm::DevHot h{c->d_scratch + gnm::plan_hot_site_offset(c->P.n_sites), hot ? gnm::kHotSlots : 0u,
                  cold.table_in_smem ? c->d_scratch + gnm::plan_slot_offset(c->P.n_sites) : nullptr,
                  c->table.node_begin, c->table.leaf_begin};
    if (c->timing) {
        ck(cudaEventRecord(pe.b, c->stream), "cudaEventRecord");
        c->plan_pairs.push_back(pe);
        ev = take_pair(c);
        ck(cudaEventRecord(ev.a, c->stream), "cudaEventRecord");
    }
    const gnm::DevLog lg = reserve_log(c, cfg, b);
    ck(gnm::launch_k2(cfg, b, c->table, p, c->P, h, lg, c->stream), "K2 launch");
    if (c->timing) {
        ck(cudaEventRecord(ev.b, c->stream), "cudaEventRecord");
        c->k2_pairs.push_back(ev);
    }
    c->k2_launches += 1;
    c->kernel_launches += 1;
    c->records += b.n;
}

constexpr uint64_t kMaxLaunchRecords = 1ull << 31;

gnm::DevBatch soa_batch(const void* const* cols, uint64_t n) {
    gnm::DevBatch b{};
    b.aos = false;
    b.soa = gnm::DevSoA{static_cast<const uint32_t*>(cols[0]), static_cast<const uint32_t*>(cols[1]),
                        static_cast<const uint32_t*>(cols[2]), static_cast<const uint32_t*>(cols[3]),
                        static_cast<const uint64_t*>(cols[4]), static_cast<const uint64_t*>(cols[5]), n};
    b.n = n;
    return b;
}

gnm::DevBatch aos_batch(const void* rec, uint64_t n) {
    gnm::DevBatch b{};
    b.aos = true;
    b.rec = rec;
    b.n = n;
    return b;
}

// Host batches: pinned, double-buffered H2D on the copy stream overlapped
// with K2 on the compute stream, chunk by chunk (SURVEY.md §8 loader L1).
// Columns already in pinned memory DMA straight from the caller's buffers;
// pageable columns go through the context's pinned staging slots.
// Host threads for the loader's staging work: the cores of this process's
// share of the node -- hardware threads / the ranks torchrun put on it
// (LOCAL_WORLD_SIZE) / the contexts of a group loading at once -- at most 16.
// GNM_STAGE_THREADS overrides.
unsigned stage_threads(const gnm_ctx* c) {
    static const unsigned kNode = [] {
        unsigned t = std::thread::hardware_concurrency();
        if (const char* l = std::getenv("LOCAL_WORLD_SIZE")) t /= std::max(1, std::atoi(l));
        return std::max(1u, t);
    }();
    if (const char* e = std::getenv("GNM_STAGE_THREADS")) return std::max(1, std::min(std::atoi(e), 16));
    return std::max(1u, std::min(kNode / std::max(1u, c->stage_share), 16u));
}

// Pageable host input: the copy into the pinned staging slot is the
// bottleneck of the loader (one core copies ~10 GB/s, PCIe takes ~55), so
// a chunk's column pieces are copied by several host threads, each taking
// an equal share of the concatenated bytes.
struct CopySeg {
    unsigned char* dst;
    const unsigned char* src;
    size_t bytes;
};

// fn(t, nt) on nt host threads (the calling thread is t = 0), on the
// context's persistent worker pool: a loader chunk is a few milliseconds of
// work, so spawning threads per chunk would cost a visible share of it.
template <typename F>
void parallel_for(gnm_ctx* c, unsigned nt, F&& fn) {
    if (nt <= 1) {
        fn(0u, 1u);
        return;
    }
    if (!c->pool_workers || c->pool_workers->size() + 1 < nt) c->pool_workers.reset(new WorkerPool(nt - 1));
    c->pool_workers->run(nt, fn);
}

#ifndef GNM_RESULT_COPY_THREADS
#define GNM_RESULT_COPY_THREADS 4
#endif
void staged_copy(gnm_ctx* c, const std::vector<CopySeg>& segs, unsigned kThreads) {
    constexpr size_t kMinPerThread = 192u << 10;
    size_t total = 0;
    for (const CopySeg& g : segs) total += g.bytes;
    const unsigned nt = static_cast<unsigned>(std::min<size_t>(kThreads, std::max<size_t>(1, total / kMinPerThread)));
    const size_t per = nt <= 1 ? total : (total / nt + 4095) & ~size_t(4095);
    // bytes [a, b) of the concatenation
    parallel_for(c, nt, [&](unsigned t, unsigned) {
        const size_t a = std::min(total, per * t), b = std::min(total, per * (t + 1));
        size_t at = 0;
        for (const CopySeg& g : segs) {
            const size_t lo = std::max(a, at), hi = std::min(b, at + g.bytes);
            if (lo < hi) std::memcpy(g.dst + (lo - at), g.src + (lo - at), hi - lo);
            at += g.bytes;
        }
    });
}

// Device -> pageable host copies of a megabyte or more (the per-host rows,
// 64 B each; the per-host histogram entries, up to hundreds of MB): through
// the two pinned staging slots, each chunk's host copy (several threads,
// which also take the destination's first-touch page faults) overlapping the
// next chunk's DMA; below 64 MB in one chunk, whose host copy is spread over
// the threads. A direct pageable cudaMemcpy runs at ~22 GB/s. Small or
// pinned destinations go directly.
void d2h_large(gnm_ctx* c, void* dst, const void* src, size_t bytes) {
    const size_t kChunk = bytes < (64u << 20) ? bytes : 32u << 20;
    if (bytes < (1u << 20) || is_pinned(dst)) {
        if (bytes) ck(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c->stream), "cudaMemcpyAsync(D2H)");
        ck(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");
        return;
    }
    ensure_stage(c, std::max<size_t>(c->stage_bytes, kChunk), true);
    const size_t chunk = std::min({c->h_stage_bytes, c->stage_bytes, kChunk});
    cudaEvent_t done[2] = {c->ev_h2d[0], c->ev_h2d[1]}; // idle outside the loader
    auto* d = static_cast<unsigned char*>(dst);
    const auto* sp = static_cast<const unsigned char*>(src);
    size_t pending_off = 0, pending_len = 0;
    int pending_slot = -1;
    for (size_t off = 0, k = 0; off < bytes; off += chunk, ++k) {
        const int slot = static_cast<int>(k & 1);
        const size_t len = std::min(chunk, bytes - off);
        ck(cudaMemcpyAsync(c->h_stage[slot], sp + off, len, cudaMemcpyDeviceToHost, c->stream), "D2H chunk");
        ck(cudaEventRecord(done[slot], c->stream), "cudaEventRecord");
        if (pending_slot >= 0) { // drain the previous chunk while this one is in flight
            ck(cudaEventSynchronize(done[pending_slot]), "cudaEventSynchronize");
            staged_copy(c, {{d + pending_off, c->h_stage[pending_slot], pending_len}}, stage_threads(c));
        }
        pending_slot = slot;
        pending_off = off;
        pending_len = len;
    }
    ck(cudaEventSynchronize(done[pending_slot]), "cudaEventSynchronize");
    staged_copy(c, {{d + pending_off, c->h_stage[pending_slot], pending_len}}, stage_threads(c));
}


// Host SoA batches analysed without a snapshot window need only
// dur = end - start of the two u64 columns (reduce_slice, rate_engine.cpp:
// 211-236 uses nothing else of them): the loader sends it as u32 (20 bytes
// per record over PCIe instead of 32) and K2 reads it in place (layout 5).
// Computed on host threads while the previous chunk's DMA runs; a chunk with
// any duration >= 2^32 (e.g. end < start, which wraps) goes uncompacted.
// Pageable input: the four u32 columns are staged in the same pass.
void load_and_run(gnm_ctx* c, bool aos, const void* const* cols, const size_t* widths, int ncols,
                  uint64_t n, const gnm::DevParams& p, bool archive);

void load_and_run_compact(gnm_ctx* c, const gnm_batch_soa* b, const gnm::DevParams& p) {
    const uint64_t n = b->n;
    bool pinned = true;
    const void* cols[6] = {b->src_addr, b->dst_addr, b->d_pkts, b->d_octets, b->start_ms, b->end_ms};
    for (const void* q : cols) pinned = pinned && is_pinned(q);
    if (pinned && stage_threads(c) < 8) { // too few cores to out-run the plain DMA of pinned columns
        const size_t widths[6] = {4, 4, 4, 4, 8, 8};
        load_and_run(c, false, cols, widths, 6, n, p, false);
        return;
    }
    const uint64_t chunk = (std::max<uint64_t>(1024, std::min<uint64_t>(c->chunk, n)) + 3) & ~uint64_t(3);
    const size_t col = chunk * 4; // one u32 column of a slot, 16-byte multiple
    // device slot: src | dst | pkts | octets | dur32, or the 32-byte fallback
    // layout src | dst | pkts | octets | start | end; host slot: the staged columns
    ensure_stage(c, chunk * 32, true);
    const unsigned nt = stage_threads(c);
    for (uint64_t base = 0, k = 0; base < n; base += chunk, ++k) {
        const int slot = static_cast<int>(k & 1);
        const uint64_t m = std::min<uint64_t>(chunk, n - base);
        ck(cudaStreamWaitEvent(c->copy_stream, c->ev_k2[slot], 0), "cudaStreamWaitEvent");
        ck(cudaEventSynchronize(c->ev_h2d[slot]), "cudaEventSynchronize"); // the host slot is free
        EventPair ev;
        if (c->timing) {
            ev = take_pair(c);
            ck(cudaEventRecord(ev.a, c->copy_stream), "cudaEventRecord");
        }
        unsigned char* hs = c->h_stage[slot];
        unsigned char* ds = c->d_stage[slot];
        uint32_t* hdur = reinterpret_cast<uint32_t*>(hs + (pinned ? 0 : 4 * col));
        const auto* st = b->start_ms + base;
        const auto* en = b->end_ms + base;
        std::atomic<bool> wide{false};
        parallel_for(c, nt, [&](unsigned t, unsigned ntt) {
            const uint64_t lo = m * t / ntt, hi = m * (t + 1) / ntt;
            if (!pinned) // the four u32 columns into the pinned slot
                for (int q = 0; q < 4; ++q)
                    std::memcpy(hs + q * col + lo * 4, static_cast<const uint32_t*>(cols[q]) + base + lo,
                                (hi - lo) * 4);
            uint64_t over = 0;
            for (uint64_t i = lo; i < hi; ++i) {
                const uint64_t d = en[i] - st[i];
                over |= d >> 32;
                hdur[i] = static_cast<uint32_t>(d);
            }
            if (over) wide.store(true, std::memory_order_relaxed);
        });
        const void* dcols[6];
        for (int q = 0; q < 4; ++q) {
            dcols[q] = ds + q * col;
            const void* from = pinned ? static_cast<const void*>(static_cast<const uint32_t*>(cols[q]) + base)
                                      : static_cast<const void*>(hs + q * col);
            ck(cudaMemcpyAsync(ds + q * col, from, m * 4, cudaMemcpyHostToDevice, c->copy_stream), "H2D");
        }
        c->h2d_bytes += m * (wide.load() ? 32 : 20);
        gnm::DevBatch db;
        if (!wide.load()) {
            ck(cudaMemcpyAsync(ds + 4 * col, hdur, m * 4, cudaMemcpyHostToDevice, c->copy_stream), "H2D dur");
            db = soa_batch(dcols, m);
            db.soa.start = db.soa.end = nullptr;
            db.soa.dur32 = reinterpret_cast<const uint32_t*>(ds + 4 * col);
        } else { // a duration needs 64 bits: send start/end (8-byte columns after the u32 ones)
            dcols[4] = ds + 4 * col;
            dcols[5] = ds + 4 * col + chunk * 8;
            ck(cudaMemcpyAsync(ds + 4 * col, st, m * 8, cudaMemcpyHostToDevice, c->copy_stream), "H2D start");
            ck(cudaMemcpyAsync(ds + 4 * col + chunk * 8, en, m * 8, cudaMemcpyHostToDevice, c->copy_stream),
               "H2D end");
            db = soa_batch(dcols, m);
        }
        if (c->timing) {
            ck(cudaEventRecord(ev.b, c->copy_stream), "cudaEventRecord");
            c->h2d_pairs.push_back(ev);
        }
        ck(cudaEventRecord(c->ev_h2d[slot], c->copy_stream), "cudaEventRecord");
        ck(cudaStreamWaitEvent(c->stream, c->ev_h2d[slot], 0), "cudaStreamWaitEvent");
        launch_k2_timed(c, db, p);
        ck(cudaEventRecord(c->ev_k2[slot], c->stream), "cudaEventRecord");
    }
    ck(cudaStreamSynchronize(c->copy_stream), "cudaStreamSynchronize");
}

// The same compaction for host FlowRecord rows (the C++ drop-in's
// std::vector): host threads gather src, dst, d_pkts, d_octets and the u32
// duration of each 64-byte row (netflow.hpp:59-67) into the staging slot, so
// 20 of the 64 bytes per record cross PCIe. Chunks with a duration >= 2^32
// send their rows whole (layout 2).
void load_and_run_compact_aos(gnm_ctx* c, const gnm_batch_aos* b, const gnm::DevParams& p) {
    const uint64_t n = b->n;
    const bool pinned = is_pinned(b->records);
    const uint64_t chunk = (std::max<uint64_t>(1024, std::min<uint64_t>(c->chunk, n)) + 3) & ~uint64_t(3);
    const size_t col = chunk * 4;
    ensure_stage(c, chunk * GNM_FLOW_RECORD_BYTES, true);
    const unsigned nt = stage_threads(c);
    const auto* rows = static_cast<const unsigned char*>(b->records);
    for (uint64_t base = 0, k = 0; base < n; base += chunk, ++k) {
        const int slot = static_cast<int>(k & 1);
        const uint64_t m = std::min<uint64_t>(chunk, n - base);
        ck(cudaStreamWaitEvent(c->copy_stream, c->ev_k2[slot], 0), "cudaStreamWaitEvent");
        ck(cudaEventSynchronize(c->ev_h2d[slot]), "cudaEventSynchronize");
        EventPair ev;
        if (c->timing) {
            ev = take_pair(c);
            ck(cudaEventRecord(ev.a, c->copy_stream), "cudaEventRecord");
        }
        unsigned char* hs = c->h_stage[slot];
        unsigned char* ds = c->d_stage[slot];
        auto* hsrc = reinterpret_cast<uint32_t*>(hs);
        auto* hdst = reinterpret_cast<uint32_t*>(hs + col);
        auto* hpk = reinterpret_cast<uint32_t*>(hs + 2 * col);
        auto* hoc = reinterpret_cast<uint32_t*>(hs + 3 * col);
        auto* hdu = reinterpret_cast<uint32_t*>(hs + 4 * col);
        std::atomic<bool> wide{false};
        parallel_for(c, nt, [&](unsigned t, unsigned ntt) {
            const uint64_t lo = m * t / ntt, hi = m * (t + 1) / ntt;
            uint64_t over = 0;
            for (uint64_t i = lo; i < hi; ++i) {
                const unsigned char* r = rows + (base + i) * GNM_FLOW_RECORD_BYTES;
                uint32_t w[6];
                uint64_t st, en;
                std::memcpy(w, r, 24);
                std::memcpy(&st, r + 48, 8);
                std::memcpy(&en, r + 56, 8);
                const uint64_t d = en - st;
                over |= d >> 32;
                hsrc[i] = w[0];
                hdst[i] = w[1];
                hpk[i] = w[4];
                hoc[i] = w[5];
                hdu[i] = static_cast<uint32_t>(d);
            }
            if (over) wide.store(true, std::memory_order_relaxed);
        });
        gnm::DevBatch db;
        if (!wide.load()) {
            for (int q = 0; q < 5; ++q)
                ck(cudaMemcpyAsync(ds + q * col, hs + q * col, m * 4, cudaMemcpyHostToDevice, c->copy_stream),
                   "H2D");
            c->h2d_bytes += m * 20;
            const void* dcols[6] = {ds, ds + col, ds + 2 * col, ds + 3 * col, nullptr, nullptr};
            db = soa_batch(dcols, m);
            db.soa.dur32 = reinterpret_cast<const uint32_t*>(ds + 4 * col);
        } else { // a duration needs 64 bits: the rows go whole
            ck(cudaMemcpyAsync(ds, rows + base * GNM_FLOW_RECORD_BYTES, m * GNM_FLOW_RECORD_BYTES,
                               cudaMemcpyHostToDevice, c->copy_stream),
               "H2D rows");
            c->h2d_bytes += m * GNM_FLOW_RECORD_BYTES;
            db = aos_batch(ds, m);
        }
        if (c->timing) {
            ck(cudaEventRecord(ev.b, c->copy_stream), "cudaEventRecord");
            c->h2d_pairs.push_back(ev);
        }
        ck(cudaEventRecord(c->ev_h2d[slot], c->copy_stream), "cudaEventRecord");
        ck(cudaStreamWaitEvent(c->stream, c->ev_h2d[slot], 0), "cudaStreamWaitEvent");
        launch_k2_timed(c, db, p);
        ck(cudaEventRecord(c->ev_k2[slot], c->stream), "cudaEventRecord");
    }
    ck(cudaStreamSynchronize(c->copy_stream), "cudaStreamSynchronize");
    (void)pinned;
}

void load_and_run(gnm_ctx* c, bool aos, const void* const* cols, const size_t* widths, int ncols,
                  uint64_t n, const gnm::DevParams& p, bool archive) {
    size_t rec_bytes = 0;
    bool pinned = true;
    for (int i = 0; i < ncols; ++i) {
        rec_bytes += widths[i];
        pinned = pinned && is_pinned(cols[i]);
    }
    const uint64_t chunk = std::max<uint64_t>(1024, std::min<uint64_t>(c->chunk, n));
    ensure_stage(c, chunk * rec_bytes, !pinned);
    for (uint64_t base = 0, k = 0; base < n; base += chunk, ++k) {
        const int slot = static_cast<int>(k & 1);
        const uint64_t m = std::min<uint64_t>(chunk, n - base);
        // The device slot is free once the K2 that last read it finished.
        ck(cudaStreamWaitEvent(c->copy_stream, c->ev_k2[slot], 0), "cudaStreamWaitEvent");
        EventPair ev;
        if (c->timing) {
            ev = take_pair(c);
            ck(cudaEventRecord(ev.a, c->copy_stream), "cudaEventRecord");
        }
        unsigned char* dslot = c->d_stage[slot];
        size_t off = 0;
        const void* dcols[6];
        if (!pinned) {
            // The pinned slot is free once its previous H2D completed.
            ck(cudaEventSynchronize(c->ev_h2d[slot]), "cudaEventSynchronize");
            size_t hoff = 0;
            std::vector<CopySeg> segs;
            for (int i = 0; i < ncols; ++i) {
                segs.push_back({c->h_stage[slot] + hoff, static_cast<const unsigned char*>(cols[i]) + base * widths[i],
                                m * widths[i]});
                hoff += m * widths[i];
            }
            staged_copy(c, segs, stage_threads(c));
            ck(cudaMemcpyAsync(dslot, c->h_stage[slot], hoff, cudaMemcpyHostToDevice, c->copy_stream),
               "cudaMemcpyAsync(H2D)");
            c->h2d_bytes += hoff;
            for (int i = 0; i < ncols; ++i) {
                dcols[i] = dslot + off;
                off += m * widths[i];
            }
        } else {
            for (int i = 0; i < ncols; ++i) {
                ck(cudaMemcpyAsync(dslot + off, static_cast<const unsigned char*>(cols[i]) + base * widths[i],
                                   m * widths[i], cudaMemcpyHostToDevice, c->copy_stream),
                   "cudaMemcpyAsync(H2D)");
                c->h2d_bytes += m * widths[i];
                dcols[i] = dslot + off;
                off += m * widths[i];
            }
        }
        if (c->timing) {
            ck(cudaEventRecord(ev.b, c->copy_stream), "cudaEventRecord");
            c->h2d_pairs.push_back(ev);
        }
        ck(cudaEventRecord(c->ev_h2d[slot], c->copy_stream), "cudaEventRecord");
        ck(cudaStreamWaitEvent(c->stream, c->ev_h2d[slot], 0), "cudaStreamWaitEvent");
        gnm::DevBatch db = aos ? aos_batch(dcols[0], m) : soa_batch(dcols, m);
        db.archive = archive;
        launch_k2_timed(c, db, p);
        ck(cudaEventRecord(c->ev_k2[slot], c->stream), "cudaEventRecord");
    }
    // The caller's host buffers may be reused once their copies are done.
    ck(cudaStreamSynchronize(c->copy_stream), "cudaStreamSynchronize");
}

int check_soa(const gnm_batch_soa* b) {
    if (!b) return fail(GNM_ERR_INVALID_ARGUMENT, "null batch");
    if (b->n && (!b->src_addr || !b->dst_addr || !b->d_pkts || !b->d_octets || !b->start_ms || !b->end_ms))
        return fail(GNM_ERR_INVALID_ARGUMENT, "null column in a non-empty batch");
    if (b->mem != GNM_MEM_HOST && b->mem != GNM_MEM_DEVICE)
        return fail(GNM_ERR_INVALID_ARGUMENT, "batch.mem must be GNM_MEM_HOST or GNM_MEM_DEVICE");
    return GNM_OK;
}

struct Window {
    uint64_t lo, hi;
};

void apply_window(gnm::DevParams& p, const Window* w) {
    if (!w) return;
    p.windowed = 1;
    p.win_lo = w->lo;
    p.win_hi = w->hi;
}

int accumulate_soa(gnm_ctx* c, const gnm_registry* reg, const gnm_filter_params* params,
                   const gnm_batch_soa* b, const Window* win = nullptr) {
    if (int e = check_soa(b)) return e;
    if (c->prepared) return fail(GNM_ERR_INVALID_ARGUMENT, "gnm_prepare_median already ran; finalize first");
    if (int e = begin_accumulate(c, reg)) return e;
    gnm::DevParams p = dev_params(c, params);
    apply_window(p, win);
    if (b->n == 0) return GNM_OK;
    if (b->mem == GNM_MEM_DEVICE) {
        // K2 indexes 64-record tiles in 32 bits: launches of < 2^31 records
        for (uint64_t o = 0; o < b->n; o += kMaxLaunchRecords) {
            const void* cols[6] = {b->src_addr + o, b->dst_addr + o, b->d_pkts + o, b->d_octets + o,
                                   b->start_ms + o, b->end_ms + o};
            launch_k2_timed(c, soa_batch(cols, std::min<uint64_t>(kMaxLaunchRecords, b->n - o)), p);
        }
    } else {
        if (!p.windowed && !std::getenv("GNM_NO_COMPACT")) {
            load_and_run_compact(c, b, p);
        } else {
            const void* cols[6] = {b->src_addr, b->dst_addr, b->d_pkts, b->d_octets, b->start_ms, b->end_ms};
            const size_t widths[6] = {4, 4, 4, 4, 8, 8};
            load_and_run(c, false, cols, widths, 6, b->n, p, false);
        }
    }
    return GNM_OK;
}

int accumulate_aos(gnm_ctx* c, const gnm_registry* reg, const gnm_filter_params* params,
                   const gnm_batch_aos* b, const Window* win = nullptr) {
    if (!b) return fail(GNM_ERR_INVALID_ARGUMENT, "null batch");
    if (b->n && !b->records) return fail(GNM_ERR_INVALID_ARGUMENT, "null records");
    // the AoS layouts read u32/u64 fields in place (FlowRecord is 8-byte aligned)
    if (b->mem == GNM_MEM_DEVICE && reinterpret_cast<uintptr_t>(b->records) % 8)
        return fail(GNM_ERR_INVALID_ARGUMENT, "device FlowRecord rows must be 8-byte aligned");
    if (c->prepared) return fail(GNM_ERR_INVALID_ARGUMENT, "gnm_prepare_median already ran; finalize first");
    if (int e = begin_accumulate(c, reg)) return e;
    gnm::DevParams p = dev_params(c, params);
    apply_window(p, win);
    if (b->n == 0) return GNM_OK;
    if (b->mem == GNM_MEM_DEVICE) {
        for (uint64_t o = 0; o < b->n; o += kMaxLaunchRecords)
            launch_k2_timed(c, aos_batch(static_cast<const unsigned char*>(b->records) + o * GNM_FLOW_RECORD_BYTES,
                                         std::min<uint64_t>(kMaxLaunchRecords, b->n - o)),
                            p);
    } else {
        // compaction pays when enough cores can gather the rows faster than
        // PCIe moves them whole (pageable rows are copied by the CPU anyway)
        if (!p.windowed && !std::getenv("GNM_NO_COMPACT") && (stage_threads(c) >= 8 || !is_pinned(b->records))) {
            load_and_run_compact_aos(c, b, p);
        } else {
            const void* cols[1] = {b->records};
            const size_t widths[1] = {GNM_FLOW_RECORD_BYTES};
            load_and_run(c, true, cols, widths, 1, b->n, p, false);
        }
    }
    return GNM_OK;
}

// Hosts local phase (H0..H2) on this context's log.
cudaError_t build_hosts_local(gnm_ctx* c, const gnm_registry* reg) {
    std::vector<gnm::HostSlice> hs;
    for (const auto& sl : c->slices) hs.push_back({slice_view(c, sl), sl.entry_off, sl.count_off});
    const uint64_t max_keys = 256ull * reg->r.entries().size(); // hosts lie in registered /24s
    c->kernel_launches += 3 + hs.size(); // own kernels; cub scan/sorts not counted
    const uint32_t n16 = c->table.leaf_begin - c->table.node_begin; // one node per non-empty /16
    return gnm::build_hosts_local(c->device, hs.data(), static_cast<int>(hs.size()), c->d_counts, c->counts_used,
                                  max_keys, static_cast<uint32_t>(reg->r.sites().size()), c->table.words, n16,
                                  c->table.packed, c->hrows, c->hlocal, c->stream);
}

// Round 1 -> round 2 of the median: K3a finds every site's median
// super-bucket from the (possibly all-reduced) coarse counts, K2b rebuilds
// that super-bucket's fine counts from this context's log.
void prepare_median(gnm_ctx* c) {
    if (c->prepared) return;
    ck(gnm::launch_k3a(c->device, c->P, c->stream), "K3a launch");
    c->kernel_launches += 1;
    for (const auto& sl : c->slices) {
        ck(gnm::launch_k2b(c->device, c->P, slice_view(c, sl), c->stream), "K2b launch");
        c->kernel_launches += 1;
    }
    c->prepared = true;
}

void clear_log(gnm_ctx* c) {
    c->log_used = 0;
    c->counts_used = 0;
    c->slices.clear();
    c->prepared = false;
}

// The multi-GPU combine of the site partials, stream-ordered
// on the context's stream between K2 and K3b: round 1 (one grouped call:
// sums and coarse counts SUM, min MIN, max MAX), K3a + K2b on this rank's
// log against the global coarse counts, round 2 (fine counts SUM). Every
// rank ends with the same global partials, so K3b's rows are identical.
void combine_sites(gnm_ctx* c) {
    gnm::Comm& m = *c->comm;
    const size_t n = c->P.n_sites;
    m.group_start();
    m.all_reduce(c->P.sums, n * 4 + 4, gnm::DType::U64, gnm::RedOp::Sum, c->stream);
    m.all_reduce(c->P.coarse, n * gnm::kCoarse, gnm::DType::U32, gnm::RedOp::Sum, c->stream);
    m.all_reduce(c->P.mn, n, gnm::DType::F64, gnm::RedOp::Min, c->stream);
    m.all_reduce(c->P.mx, n, gnm::DType::F64, gnm::RedOp::Max, c->stream);
    m.group_end();
    prepare_median(c);
    m.all_reduce(c->P.fine, n * gnm::kFineW, gnm::DType::U32, gnm::RedOp::Sum, c->stream);
}

// Per-host rows across the ranks: every rank's sorted distinct (site, host)
// keys are all-gathered (counts first, then the key lists padded to the
// longest), their sorted union becomes the global rows, and the same two
// rounds as the sites run over them. Synchronises the stream (the union's
// size sizes the partials), so it is never captured in a graph.
void combine_hosts(gnm_ctx* c, const gnm_registry* reg) {
    gnm::Comm& m = *c->comm;
    const int N = m.nranks();
    if (!c->hlocal.ready) ck(build_hosts_local(c, reg), "per-host local phase");
    const uint64_t nl = c->hrows.n_rows;
    unsigned long long* d_cnt = nullptr;
    ck(cudaMallocAsync(reinterpret_cast<void**>(&d_cnt), 8 * (N + 1), c->stream), "cudaMallocAsync(key counts)");
    ck(cudaMemcpyAsync(d_cnt + N, &nl, 8, cudaMemcpyHostToDevice, c->stream), "cudaMemcpyAsync(key count)");
    m.all_gather(d_cnt + N, d_cnt, 8, c->stream);
    std::vector<uint64_t> counts(N);
    ck(cudaMemcpyAsync(counts.data(), d_cnt, 8 * N, cudaMemcpyDeviceToHost, c->stream), "D2H key counts");
    ck(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");
    ck(cudaFreeAsync(d_cnt, c->stream), "cudaFreeAsync");
    const uint64_t maxn = std::max<uint64_t>(1, *std::max_element(counts.begin(), counts.end()));
    // stream-ordered temporaries, released on every path
    struct Temps {
        cudaStream_t s;
        unsigned long long *send = nullptr, *all = nullptr, *uni = nullptr;
        ~Temps() {
            for (void* p : {static_cast<void*>(send), static_cast<void*>(all), static_cast<void*>(uni)})
                if (p) cudaFreeAsync(p, s);
        }
    } tmp{c->stream};
    unsigned long long*& send = tmp.send;
    unsigned long long*& all = tmp.all;
    unsigned long long*& uni = tmp.uni;
    ck(cudaMallocAsync(reinterpret_cast<void**>(&send), 8 * maxn, c->stream), "cudaMallocAsync(keys)");
    ck(cudaMallocAsync(reinterpret_cast<void**>(&all), 8 * maxn * N, c->stream), "cudaMallocAsync(keys)");
    ck(cudaMallocAsync(reinterpret_cast<void**>(&uni), 8 * maxn * N, c->stream), "cudaMallocAsync(keys)");
    ck(cudaMemsetAsync(send, 0xFF, 8 * maxn, c->stream), "cudaMemsetAsync(keys)"); // padding sorts last
    if (nl) ck(cudaMemcpyAsync(send, c->hlocal.hk_sorted, 8 * nl, cudaMemcpyDeviceToDevice, c->stream), "keys");
    m.all_gather(send, all, 8 * maxn, c->stream);
    uint64_t nu = 0;
    ck(gnm::hosts_key_union(c->device, all, maxn * N, uni, &nu, c->stream), "per-host key union");
    if (nu >= (1ull << 24)) throw std::runtime_error("the per-host key union holds at most 2^24 - 1 rows");
    ck(gnm::hosts_global_begin(c->device, c->hrows, c->hlocal, uni, nu, c->hglobal, c->stream),
       "per-host union partials");
    c->kernel_launches += 4;
    gnm::HostGlobal& g = c->hglobal;
    m.group_start();
    m.all_reduce(g.sums, nu * 3, gnm::DType::U64, gnm::RedOp::Sum, c->stream);
    m.all_reduce(g.min, nu, gnm::DType::F64, gnm::RedOp::Min, c->stream);
    m.all_reduce(g.max, nu, gnm::DType::F64, gnm::RedOp::Max, c->stream);
    m.all_reduce(g.coarse, nu * 157, gnm::DType::U32, gnm::RedOp::Sum, c->stream);
    m.group_end();
    ck(gnm::hosts_global_prepare(c->device, c->hrows, g, c->stream), "per-host round 2");
    c->kernel_launches += 2;
    m.all_reduce(g.fine, nu * 64, gnm::DType::U32, gnm::RedOp::Sum, c->stream);
}

// phase: 1 = the device work (stream-ordered, capturable), 2 = the host
// part (wait, copy the rows out, reset the accumulation), 3 = both.
int finalize(gnm_ctx* c, const gnm_registry* reg, gnm_result* r, int phase = 3) {
    if (!r) return fail(GNM_ERR_INVALID_ARGUMENT, "null result");
    const uint32_t n_sites = static_cast<uint32_t>(reg->r.sites().size());
    if (r->sites_capacity < n_sites || (n_sites && !r->sites))
        return fail(GNM_ERR_CAPACITY, "result.sites holds " + std::to_string(r->sites_capacity) +
                                          " rows, registry has " + std::to_string(n_sites) + " sites");
    if (phase & 1) {
        if (int e = begin_accumulate(c, reg)) return e; // no-op when already accumulating
        ensure_out(c, n_sites);
        EventPair ev;
        if (c->timing) {
            ev = take_pair(c);
            ck(cudaEventRecord(ev.a, c->stream), "cudaEventRecord");
        }
        const double thr = r->threshold_bps;
        const bool export_hist = r->histograms != nullptr;
        if (!c->hlocal.ready) gnm::free_hosts(c->hrows, c->stream); // else: gnm_hosts_local_keys built them
        if (c->hosts && c->log_used >= (1ull << 32))
            return fail(GNM_ERR_CAPACITY, "per-host mode holds < 2^32 log entries per finalize");
        if (c->comm) combine_sites(c);
        else prepare_median(c);
        ck(gnm::launch_k3b(c->device, c->P, thr, c->d_out, 1, c->stream), "K3b launch");
        c->kernel_launches += 1;
        if (c->timing) {
            ck(cudaEventRecord(ev.b, c->stream), "cudaEventRecord");
            c->k3_pairs.push_back(ev);
        }
        ck(cudaMemcpyAsync(c->h_out, c->d_out, (static_cast<size_t>(n_sites) + 1) * sizeof(gnm_site_stats),
                           cudaMemcpyDeviceToHost, c->stream),
           "cudaMemcpyAsync(D2H)");
        if (export_hist) {
            // RateHistogram::buckets_ per site, rebuilt exactly from the log.
            const size_t bytes = static_cast<size_t>(n_sites) * gnm::kBuckets * 4;
            uint32_t* dense = nullptr;
            ck(cudaMallocAsync(reinterpret_cast<void**>(&dense), std::max<size_t>(bytes, 4), c->stream),
               "cudaMallocAsync(hist export)");
            ck(cudaMemsetAsync(dense, 0, bytes, c->stream), "cudaMemsetAsync(hist export)");
            for (const auto& sl : c->slices) {
                ck(gnm::launch_hist_from_log(c->device, slice_view(c, sl), n_sites, dense, c->stream), "hist export");
                c->kernel_launches += 1;
            }
            // every rank rebuilt its own flows' buckets: sum them over the ranks
            if (c->comm)
                c->comm->all_reduce(dense, static_cast<size_t>(n_sites) * gnm::kBuckets, gnm::DType::U32,
                                    gnm::RedOp::Sum, c->stream);
            if (!c->discard_hist_out)
                ck(cudaMemcpyAsync(r->histograms, dense, bytes, cudaMemcpyDeviceToHost, c->stream),
                   "cudaMemcpyAsync(D2H hist)");
            ck(cudaFreeAsync(dense, c->stream), "cudaFreeAsync(hist export)");
        }
        if (c->hosts) {
            // SiteResult::hosts: the per-host post-pass over the same log.
            if (c->comm && !c->hglobal.prepared) combine_hosts(c, reg);
            if (c->hglobal.prepared) { // rows of the cross-context union
                ck(gnm::hosts_global_finish(c->device, c->hrows, c->hglobal, c->stream), "per-host rows (union)");
                c->kernel_launches += 1;
            } else {
                if (!c->hlocal.ready) ck(build_hosts_local(c, reg), "per-host post-pass");
                ck(gnm::finish_hosts(c->device, c->hrows, c->hlocal, c->stream), "per-host post-pass");
                c->kernel_launches += 4;
            }
            gnm::free_local(c->hlocal, c->stream);
            gnm::free_global(c->hglobal, c->stream);
        }
    } // device phase
    if (!(phase & 2)) return GNM_OK;
    clear_log(c);
    ck(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");
    // K3b computed every field, avg included (rounded like the host's libgcc).
    if (n_sites) {
        // ~80 B per site: a 10k-site registry is 0.8 MB on every step's
        // critical path, spread over a few pool threads
        const size_t bytes = static_cast<size_t>(n_sites) * sizeof(gnm_site_stats);
        staged_copy(c, {{reinterpret_cast<unsigned char*>(r->sites), reinterpret_cast<const unsigned char*>(c->h_out),
                         bytes}},
                    std::min<unsigned>(GNM_RESULT_COPY_THREADS, stage_threads(c)));
    }
    const auto* t = reinterpret_cast<const uint64_t*>(c->h_out + n_sites);
    r->tallies.forward = t[0];
    r->tallies.pure_ack = t[1];
    r->tallies.administrative = t[2];
    r->tallies.unmatched = t[3];
    r->n_sites = n_sites;
    c->accumulating = false;
    // coarse counts are u32 per (super-bucket, site): with fewer than 2^32
    // Forward flows per accumulation (all ranks) none of them can wrap
    if (r->tallies.forward >> 32)
        return fail(GNM_ERR_CAPACITY, "more than 2^32-1 Forward flows in one accumulation: "
                                      "finalize at least every 4G Forward flows");
    if (c->timing) {
        c->tot_k2 += c->k2_pairs.size();
        c->acc_ms = drain_pairs(c, c->k2_pairs);
        c->plan_ms = drain_pairs(c, c->plan_pairs);
        c->fin_ms = drain_pairs(c, c->k3_pairs);
        c->h2d_ms = drain_pairs(c, c->h2d_pairs);
        c->tot_acc_ms += c->acc_ms;
        c->tot_plan_ms += c->plan_ms;
        c->tot_fin_ms += c->fin_ms;
        c->tot_finalizes += 1;
    }
    c->accumulating = false;
    return GNM_OK;
}

} // namespace

extern "C" {

const char* gnm_last_error(void) { return g_last_error.c_str(); }
int gnm_abi_version(void) { return GNM_ABI_VERSION; }

void gnm_filter_params_default(gnm_filter_params* out) {
    if (!out) return;
    out->ack_avg_size_max = 96;
    out->min_packets = 20;
    out->min_duration_ms = 100;
    out->workers = 1;
}

// ---- registry ----------------------------------------------------------------
int gnm_cidr_parse(const char* text, gnm_cidr* out) {
    if (!text || !out) return fail(GNM_ERR_INVALID_ARGUMENT, "null argument");
    gnm::Cidr c;
    std::string err;
    if (!gnm::parse_cidr(text, &c, &err)) return fail(GNM_ERR_INVALID_CIDR, err);
    out->addr = c.addr;
    out->prefix_len = c.prefix_len;
    return GNM_OK;
}

int gnm_ipv4_parse(const char* text, uint32_t* out) {
    if (!text || !out) return fail(GNM_ERR_INVALID_ARGUMENT, "null argument");
    std::string err;
    if (!gnm::parse_ipv4(text, out, &err)) return fail(GNM_ERR_INVALID_CIDR, err);
    return GNM_OK;
}

int gnm_registry_create(gnm_registry** out) {
    if (!out) return fail(GNM_ERR_INVALID_ARGUMENT, "null out");
    return guarded([&] {
        *out = new gnm_registry();
        return GNM_OK;
    });
}

void gnm_registry_destroy(gnm_registry* reg) { delete reg; }

int gnm_registry_register_site(gnm_registry* reg, const char* name, const gnm_cidr* cidrs,
                               size_t n_cidrs, uint32_t* out_site_id) {
    if (!reg || !name || (n_cidrs && !cidrs)) return fail(GNM_ERR_INVALID_ARGUMENT, "null argument");
    return guarded([&] {
        std::vector<gnm::Cidr> list(n_cidrs);
        for (size_t i = 0; i < n_cidrs; ++i) list[i] = gnm::Cidr{cidrs[i].addr, cidrs[i].prefix_len};
        std::string err;
        uint32_t id = 0;
        const int rc = reg->r.register_site(name, list, &id, &err);
        if (rc == 2) return fail(GNM_ERR_OVERLAP, err);
        if (rc == 3) return fail(GNM_ERR_INVALID_CIDR, err);
        if (rc) return fail(GNM_ERR_CAPACITY, err);
        if (out_site_id) *out_site_id = id;
        return static_cast<int>(GNM_OK);
    });
}

uint32_t gnm_registry_lookup(const gnm_registry* reg, uint32_t ip) {
    return reg ? reg->r.lookup(ip) : GNM_NO_SITE;
}
uint32_t gnm_registry_sequential_lookup(const gnm_registry* reg, uint32_t ip) {
    return reg ? reg->r.sequential_lookup(ip) : GNM_NO_SITE;
}
size_t gnm_registry_site_count(const gnm_registry* reg) { return reg ? reg->r.sites().size() : 0; }
size_t gnm_registry_entry_count(const gnm_registry* reg) { return reg ? reg->r.entries().size() : 0; }
size_t gnm_registry_entries(const gnm_registry* reg, uint32_t* prefix24, uint32_t* site, size_t cap) {
    if (!reg) return 0;
    const auto& e = reg->r.entries();
    const size_t n = std::min(cap, e.size());
    for (size_t i = 0; i < n; ++i) {
        if (prefix24) prefix24[i] = e[i].first;
        if (site) site[i] = e[i].second;
    }
    return e.size();
}
const char* gnm_registry_site_name(const gnm_registry* reg, uint32_t site) {
    if (!reg || site >= reg->r.sites().size()) return nullptr;
    return reg->r.sites()[site].name.c_str();
}
uint64_t gnm_registry_version(const gnm_registry* reg) { return reg ? reg->r.version() : 0; }

// ---- context -------------------------------------------------------------------
int gnm_ctx_create(int device, gnm_ctx** out) {
    if (!out) return fail(GNM_ERR_INVALID_ARGUMENT, "null out");
    *out = nullptr;
    int count = 0;
    const cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0) {
        cudaGetLastError();
        return fail(GNM_ERR_NO_DEVICE, std::string("no CUDA device (") + cudaGetErrorString(e) +
                                           "): gnetmon has no CPU fallback");
    }
    if (device < 0 || device >= count)
        return fail(GNM_ERR_INVALID_ARGUMENT, "device ordinal out of range");
    return guarded([&] {
        auto* c = new gnm_ctx();
        try {
            c->device = device;
            ck(cudaSetDevice(device), "cudaSetDevice");
            ck(gnm::init_kernel_attributes(), "kernel attributes");
            // Keep stream-ordered allocations (log growth, the per-host
            // post-pass scratch) in the device pool between calls instead of
            // returning them to the driver at every synchronisation.
            cudaMemPool_t pool;
            ck(cudaDeviceGetDefaultMemPool(&pool, device), "cudaDeviceGetDefaultMemPool");
            uint64_t keep = UINT64_MAX;
            ck(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep), "cudaMemPoolSetAttribute");
            ck(cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking), "cudaStreamCreate");
            ck(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking), "cudaStreamCreate");
            c->stream = c->own_stream;
            for (int i = 0; i < 2; ++i) {
                ck(cudaEventCreateWithFlags(&c->ev_h2d[i], cudaEventDisableTiming), "cudaEventCreate");
                ck(cudaEventCreateWithFlags(&c->ev_k2[i], cudaEventDisableTiming), "cudaEventCreate");
            }
        } catch (...) {
            gnm_ctx_destroy(c);
            throw;
        }
        *out = c;
        return static_cast<int>(GNM_OK);
    });
}

void gnm_ctx_destroy(gnm_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    if (c->copy_stream) cudaStreamSynchronize(c->copy_stream);
    cudaFree(c->d_table);
    cudaFree(c->P.sums);
    cudaFree(c->P.mn);
    cudaFree(c->P.mx);
    cudaFree(c->P.coarse);
    cudaFree(c->P.fine);
    cudaFree(c->P.msb);
    cudaFree(c->P.mrank);
    cudaFree(c->P.cnt);
    cudaFree(c->P.heavy_next);
    cudaFree(c->P.map16);
    cudaFree(c->d_log);
    cudaFree(c->d_logb);
    cudaFree(c->d_counts);
    cudaFree(c->d_lhost);
    cudaFree(c->d_loct);
    cudaFree(c->d_ldur);
    gnm::free_hosts(c->hrows, c->stream);
    gnm::free_local(c->hlocal, c->stream);
    gnm::free_global(c->hglobal, c->stream);
    if (c->stream) cudaStreamSynchronize(c->stream);
    cudaFree(c->d_scratch);
    cudaFree(c->d_out);
    if (c->h_out) cudaFreeHost(c->h_out);
    for (int i = 0; i < 2; ++i) {
        cudaFree(c->d_stage[i]);
        if (c->h_stage[i]) cudaFreeHost(c->h_stage[i]);
        if (c->ev_h2d[i]) cudaEventDestroy(c->ev_h2d[i]);
        if (c->ev_k2[i]) cudaEventDestroy(c->ev_k2[i]);
    }
    for (auto* v : {&c->pool, &c->k2_pairs, &c->k3_pairs, &c->h2d_pairs, &c->plan_pairs})
        for (EventPair& p : *v) {
            cudaEventDestroy(p.a);
            cudaEventDestroy(p.b);
        }
    for (auto& ge : c->graph_cache)
        if (ge.exec) cudaGraphExecDestroy(ge.exec);
    if (c->own_stream) cudaStreamDestroy(c->own_stream);
    if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
    delete c;
}

int gnm_ctx_set_stream(gnm_ctx* c, void* s) {
    if (!c) return fail(GNM_ERR_INVALID_ARGUMENT, "null ctx");
    return guarded([&] {
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        ck(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");
        c->stream = s ? static_cast<cudaStream_t>(s) : c->own_stream;
        return static_cast<int>(GNM_OK);
    });
}

void* gnm_ctx_stream(gnm_ctx* c) { return c ? c->stream : nullptr; }

int gnm_ctx_set_chunk_records(gnm_ctx* c, uint64_t records) {
    if (!c || records == 0) return fail(GNM_ERR_INVALID_ARGUMENT, "bad chunk");
    c->chunk = records;
    return GNM_OK;
}

int gnm_ctx_set_hot_mode(gnm_ctx* c, int mode) {
    if (!c || mode < GNM_HOT_OFF || mode > GNM_HOT_FORCE) return fail(GNM_ERR_INVALID_ARGUMENT, "bad hot mode");
    c->hot_mode = mode;
    return GNM_OK;
}

int gnm_ctx_set_hosts(gnm_ctx* c, int enable) {
    if (!c) return fail(GNM_ERR_INVALID_ARGUMENT, "null ctx");
    if (c->accumulating) return fail(GNM_ERR_INVALID_ARGUMENT, "per-host mode changes only between accumulations");
    c->hosts = enable != 0;
    return GNM_OK;
}

uint64_t gnm_host_count(gnm_ctx* c) { return c ? c->hrows.n_rows : 0; }

int gnm_host_results(gnm_ctx* c, gnm_host_stats* out, uint64_t capacity, uint32_t* histograms) {
    if (!c) return fail(GNM_ERR_INVALID_ARGUMENT, "null ctx");
    const uint64_t n = c->hrows.n_rows;
    if (capacity < n || (n && !out))
        return fail(GNM_ERR_CAPACITY, "host rows: capacity " + std::to_string(capacity) + " < " + std::to_string(n));
    return guarded([&] {
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        d2h_large(c, out, c->hrows.rows, n * sizeof(gnm_host_stats));
        if (n && histograms) {
            const size_t bytes = n * gnm::kBuckets * 4;
            uint32_t* dense = nullptr;
            ck(cudaMallocAsync(reinterpret_cast<void**>(&dense), bytes, c->stream), "cudaMallocAsync(host hist)");
            ck(cudaMemsetAsync(dense, 0, bytes, c->stream), "cudaMemsetAsync(host hist)");
            ck(gnm::hosts_histograms(c->device, c->hrows, dense, c->stream), "host histograms");
            c->kernel_launches += 1;
            d2h_large(c, histograms, dense, bytes);
            ck(cudaFreeAsync(dense, c->stream), "cudaFreeAsync(host hist)");
        }
        ck(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");
        return static_cast<int>(GNM_OK);
    });
}

int gnm_host_histogram_entries(gnm_ctx* c, uint32_t* rows, uint32_t* buckets, uint32_t* counts,
                               uint64_t capacity, uint64_t* n_entries) {
    if (!c || !n_entries) return fail(GNM_ERR_INVALID_ARGUMENT, "null argument");
    return guarded([&] {
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        uint64_t n = 0;
        ck(gnm::hosts_sparse(c->device, c->hrows, &n, c->stream), "host histogram entries");
        *n_entries = n;
        if (!rows || n == 0) return static_cast<int>(GNM_OK);
        if (capacity < n || !buckets || !counts)
            return fail(GNM_ERR_CAPACITY, "host histogram entries: capacity " + std::to_string(capacity) + " < " +
                                              std::to_string(n));
        uint32_t* d = nullptr;
        ck(cudaMallocAsync(reinterpret_cast<void**>(&d), n * 12, c->stream), "cudaMallocAsync(host entries)");
        ck(gnm::hosts_sparse_export(c->device, c->hrows, d, d + n, d + 2 * n, c->stream), "host entries export");
        c->kernel_launches += 1;
        d2h_large(c, rows, d, n * 4);
        d2h_large(c, buckets, d + n, n * 4);
        d2h_large(c, counts, d + 2 * n, n * 4);
        ck(cudaFreeAsync(d, c->stream), "cudaFreeAsync(host entries)");
        ck(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");
        return static_cast<int>(GNM_OK);
    });
}

int gnm_hosts_local_keys(gnm_ctx* c, const gnm_registry* reg, const uint64_t** keys, uint64_t* n) {
    if (!c || !reg || !keys || !n) return fail(GNM_ERR_INVALID_ARGUMENT, "null argument");
    if (!c->hosts) return fail(GNM_ERR_INVALID_ARGUMENT, "per-host mode is off (gnm_ctx_set_hosts)");
    return guarded([&] {
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        if (int e = begin_accumulate(c, reg)) return e;
        if (c->log_used >= (1ull << 32))
            return fail(GNM_ERR_CAPACITY, "per-host mode holds < 2^32 log entries per finalize");
        if (!c->hlocal.ready) ck(build_hosts_local(c, reg), "per-host local phase");
        *keys = reinterpret_cast<const uint64_t*>(c->hlocal.hk_sorted);
        *n = c->hrows.n_rows;
        return static_cast<int>(GNM_OK);
    });
}

int gnm_hosts_set_keys(gnm_ctx* c, const uint64_t* keys, uint64_t n, gnm_host_partials* out) {
    if (!c || !out || (n && !keys)) return fail(GNM_ERR_INVALID_ARGUMENT, "null argument");
    if (!c->hlocal.ready) return fail(GNM_ERR_INVALID_ARGUMENT, "gnm_hosts_local_keys first");
    if (n >= (1ull << 24)) return fail(GNM_ERR_CAPACITY, "the key union holds at most 2^24 - 1 rows");
    return guarded([&] {
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        ck(gnm::hosts_global_begin(c->device, c->hrows, c->hlocal, reinterpret_cast<const unsigned long long*>(keys),
                                   n, c->hglobal, c->stream),
           "per-host union partials");
        c->kernel_launches += 4;
        out->sums = reinterpret_cast<uint64_t*>(c->hglobal.sums);
        out->min = reinterpret_cast<double*>(c->hglobal.min);
        out->max = reinterpret_cast<double*>(c->hglobal.max);
        out->coarse = c->hglobal.coarse;
        out->fine = c->hglobal.fine;
        out->n = n;
        ck(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize"); // the caller's collectives read them
        return static_cast<int>(GNM_OK);
    });
}

int gnm_hosts_prepare_median(gnm_ctx* c) {
    if (!c) return fail(GNM_ERR_INVALID_ARGUMENT, "null ctx");
    if (!c->hglobal.keys) return fail(GNM_ERR_INVALID_ARGUMENT, "gnm_hosts_set_keys first");
    return guarded([&] {
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        ck(gnm::hosts_global_prepare(c->device, c->hrows, c->hglobal, c->stream), "per-host round 2");
        c->kernel_launches += 2;
        ck(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");
        return static_cast<int>(GNM_OK);
    });
}

int gnm_ctx_enable_timing(gnm_ctx* c, int enable) {
    if (!c) return fail(GNM_ERR_INVALID_ARGUMENT, "null ctx");
    c->timing = enable != 0;
    if (c->timing) {
        c->tot_plan_ms = c->tot_acc_ms = c->tot_fin_ms = 0;
        c->tot_finalizes = c->tot_k2 = 0;
    }
    return GNM_OK;
}

int gnm_ctx_timing(gnm_ctx* c, gnm_timing* out) {
    if (!c || !out) return fail(GNM_ERR_INVALID_ARGUMENT, "null argument");
    out->accumulate_ms = c->acc_ms;
    out->plan_ms = c->plan_ms;
    out->finalize_ms = c->fin_ms;
    out->h2d_ms = c->h2d_ms;
    out->k2_launches = c->k2_launches;
    out->kernel_launches = c->kernel_launches;
    out->records = c->records;
    out->total_plan_ms = c->tot_plan_ms;
    out->total_accumulate_ms = c->tot_acc_ms;
    out->total_finalize_ms = c->tot_fin_ms;
    out->total_finalizes = c->tot_finalizes;
    out->total_k2_launches = c->tot_k2;
    out->h2d_bytes = c->h2d_bytes;
    return GNM_OK;
}

// ---- analysis ----------------------------------------------------------------
int gnm_accumulate(gnm_ctx* c, const gnm_registry* reg, const gnm_filter_params* params,
                   const gnm_batch_soa* batch) {
    if (!c || !reg) return fail(GNM_ERR_INVALID_ARGUMENT, "null ctx/registry");
    return guarded([&] { return accumulate_soa(c, reg, params, batch); });
}

int gnm_accumulate_aos(gnm_ctx* c, const gnm_registry* reg, const gnm_filter_params* params,
                       const gnm_batch_aos* batch) {
    if (!c || !reg) return fail(GNM_ERR_INVALID_ARGUMENT, "null ctx/registry");
    return guarded([&] { return accumulate_aos(c, reg, params, batch); });
}

int gnm_finalize(gnm_ctx* c, const gnm_registry* reg, gnm_result* result) {
    if (!c || !reg) return fail(GNM_ERR_INVALID_ARGUMENT, "null ctx/registry");
    return guarded([&] { return finalize(c, reg, result); });
}

int gnm_prepare_median(gnm_ctx* c, const gnm_registry* reg) {
    if (!c || !reg) return fail(GNM_ERR_INVALID_ARGUMENT, "null ctx/registry");
    if (c->comm) return fail(GNM_ERR_INVALID_ARGUMENT, "the context's communicator combines inside gnm_finalize");
    return guarded([&] {
        if (int e = begin_accumulate(c, reg)) return e;
        EventPair ev;
        if (c->timing) {
            ev = take_pair(c);
            ck(cudaEventRecord(ev.a, c->stream), "cudaEventRecord");
        }
        prepare_median(c);
        if (c->timing) {
            ck(cudaEventRecord(ev.b, c->stream), "cudaEventRecord");
            c->k3_pairs.push_back(ev);
        }
        return static_cast<int>(GNM_OK);
    });
}

int gnm_reset(gnm_ctx* c) {
    if (!c) return fail(GNM_ERR_INVALID_ARGUMENT, "null ctx");
    return guarded([&] {
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        if (c->P.sums) {
            ck(gnm::launch_reset(c->device, c->P, c->stream), "reset launch");
            c->kernel_launches += 1;
            ck(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");
        }
        clear_log(c);
        gnm::free_hosts(c->hrows, c->stream);
        gnm::free_local(c->hlocal, c->stream);
        gnm::free_global(c->hglobal, c->stream);
        drain_pairs(c, c->k2_pairs);
        drain_pairs(c, c->plan_pairs);
        drain_pairs(c, c->k3_pairs);
        drain_pairs(c, c->h2d_pairs);
        c->accumulating = false;
        return static_cast<int>(GNM_OK);
    });
}

int gnm_decode_netflow(gnm_ctx* c, const uint8_t* datagrams, uint64_t bytes, const uint64_t* offsets,
                       uint64_t n, int32_t in_mem, void* out_records, uint64_t capacity, int32_t out_mem,
                       uint8_t* status, gnm_netflow_stats* stats) {
    if (!c || (n && (!datagrams || !offsets)) || (capacity && !out_records))
        return fail(GNM_ERR_INVALID_ARGUMENT, "null argument");
    if ((in_mem != GNM_MEM_HOST && in_mem != GNM_MEM_DEVICE) || (out_mem != GNM_MEM_HOST && out_mem != GNM_MEM_DEVICE))
        return fail(GNM_ERR_INVALID_ARGUMENT, "mem must be GNM_MEM_HOST or GNM_MEM_DEVICE");
    return guarded([&] {
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        cudaStream_t s = c->stream;
        if (in_mem == GNM_MEM_HOST && n) {
            if (offsets[n] > bytes) return fail(GNM_ERR_INVALID_ARGUMENT, "offsets[n] exceeds bytes");
            for (uint64_t i = 0; i < n; ++i)
                if (offsets[i + 1] < offsets[i]) return fail(GNM_ERR_INVALID_ARGUMENT, "offsets must be non-decreasing");
        }
        // Device scratch: datagrams + offsets (host input), per-datagram counts,
        // offsets, status, stats, and the output rows when they cannot go
        // straight to device memory of sufficient capacity.
        const uint64_t max_rows = n * 30;
        const bool direct = out_mem == GNM_MEM_DEVICE && capacity >= max_rows;
        const size_t in_bytes = in_mem == GNM_MEM_HOST ? bytes : 0;
        const size_t off_bytes = in_mem == GNM_MEM_HOST ? (n + 1) * 8 : 0;
        auto up = [](size_t x) { return (x + 255) / 256 * 256; };
        const size_t scratch_bytes = gnm::netflow_scratch_words(n) * 8;
        const size_t total = up(in_bytes) + up(off_bytes) + up(scratch_bytes) + up(n) + up(5 * 8) +
                             (direct ? 0 : up(max_rows * 64));
        unsigned char* scratch = nullptr;
        ck(cudaMallocAsync(reinterpret_cast<void**>(&scratch), std::max<size_t>(total, 256), s), "cudaMallocAsync(netflow)");
        unsigned char* q = scratch;
        const uint8_t* d = datagrams;
        const uint64_t* off = offsets;
        if (in_mem == GNM_MEM_HOST) {
            ck(cudaMemcpyAsync(q, datagrams, bytes, cudaMemcpyHostToDevice, s), "H2D datagrams");
            d = q;
            q += up(in_bytes);
            ck(cudaMemcpyAsync(q, offsets, (n + 1) * 8, cudaMemcpyHostToDevice, s), "H2D offsets");
            off = reinterpret_cast<const uint64_t*>(q);
            q += up(off_bytes);
        }
        auto* tiles = reinterpret_cast<unsigned long long*>(q);
        q += up(scratch_bytes);
        auto* st = reinterpret_cast<uint8_t*>(q);
        q += up(n);
        auto* dstats = reinterpret_cast<unsigned long long*>(q);
        q += up(5 * 8);
        uint8_t* out = direct ? static_cast<uint8_t*>(out_records) : q;
        ck(cudaMemsetAsync(dstats, 0, 5 * 8, s), "cudaMemsetAsync");
        ck(gnm::launch_netflow_decode(d, off, n, tiles, st, dstats, out, c->device, s), "netflow decode");
        c->kernel_launches += n ? 1 : 0;
        unsigned long long hs[5] = {0, 0, 0, 0, 0};
        ck(cudaMemcpyAsync(hs, dstats, sizeof hs, cudaMemcpyDeviceToHost, s), "D2H stats");
        if (status && n) ck(cudaMemcpyAsync(status, st, n, cudaMemcpyDeviceToHost, s), "D2H status");
        ck(cudaStreamSynchronize(s), "cudaStreamSynchronize");
        int rc = GNM_OK;
        if (hs[3] > capacity) {
            rc = fail(GNM_ERR_CAPACITY, std::to_string(hs[3]) + " accepted records exceed capacity " +
                                            std::to_string(capacity));
        } else if (!direct && hs[3]) {
            ck(cudaMemcpyAsync(out_records, out, hs[3] * 64,
                               out_mem == GNM_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, s),
               "copy records");
        }
        ck(cudaFreeAsync(scratch, s), "cudaFreeAsync(netflow)");
        ck(cudaStreamSynchronize(s), "cudaStreamSynchronize");
        if (stats) {
            stats->datagrams = n;
            stats->decode_errors = hs[1];
            stats->records_rejected = hs[2];
            stats->records_accepted = hs[3];
        }
        return rc;
    });
}

// FlowStore::load's checks (flow_store.cpp:167-207) on an in-memory archive:
// returns the record count or fails with the ArchiveError kind's status.
int archive_header(gnm_ctx* c, const uint8_t* bytes, uint64_t len, int32_t mem, uint64_t* count) {
    if (mem != GNM_MEM_HOST && mem != GNM_MEM_DEVICE)
        return fail(GNM_ERR_INVALID_ARGUMENT, "mem must be GNM_MEM_HOST or GNM_MEM_DEVICE");
    if (len < 20) return fail(GNM_ERR_TRUNCATED, "archive header truncated");
    if (!bytes) return fail(GNM_ERR_INVALID_ARGUMENT, "null archive");
    uint8_t h[20];
    if (mem == GNM_MEM_DEVICE) {
        ck(cudaMemcpyAsync(h, bytes, 20, cudaMemcpyDeviceToHost, c->stream), "D2H archive header");
        ck(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");
    } else {
        std::memcpy(h, bytes, 20);
    }
    if (std::memcmp(h, "FLOWARC1", 8) != 0) return fail(GNM_ERR_BAD_MAGIC, "bad archive magic");
    const uint32_t version = uint32_t(h[8]) << 24 | uint32_t(h[9]) << 16 | uint32_t(h[10]) << 8 | h[11];
    if (version != 1) return fail(GNM_ERR_BAD_VERSION, "unsupported archive version " + std::to_string(version));
    uint64_t n = 0;
    for (int i = 0; i < 8; ++i) n = n << 8 | h[12 + i];
    if ((len - 20) / 64 < n) return fail(GNM_ERR_TRUNCATED, "archive body truncated");
    if (len - 20 != n * 64) return fail(GNM_ERR_TRUNCATED, "trailing bytes after " + std::to_string(n) + " records");
    if (mem == GNM_MEM_DEVICE && (reinterpret_cast<uintptr_t>(bytes) & 3u))
        return fail(GNM_ERR_INVALID_ARGUMENT, "device archive must be 4-byte aligned");
    *count = n;
    return GNM_OK;
}

int accumulate_archive(gnm_ctx* c, const gnm_registry* reg, const gnm_filter_params* params,
                       const uint8_t* bytes, uint64_t len, int32_t mem, const Window* win) {
    uint64_t n = 0;
    if (int e = archive_header(c, bytes, len, mem, &n)) return e;
    if (c->prepared) return fail(GNM_ERR_INVALID_ARGUMENT, "gnm_prepare_median already ran; finalize first");
    if (int e = begin_accumulate(c, reg)) return e;
    gnm::DevParams p = dev_params(c, params);
    apply_window(p, win);
    if (n == 0) return GNM_OK;
    if (mem == GNM_MEM_DEVICE) {
        gnm::DevBatch b = aos_batch(bytes + 20, n);
        b.archive = true;
        launch_k2_timed(c, b, p);
    } else {
        const void* cols[1] = {bytes + 20};
        const size_t widths[1] = {64};
        load_and_run(c, true, cols, widths, 1, n, p, true);
    }
    return GNM_OK;
}

int gnm_decode_archive(gnm_ctx* c, const uint8_t* bytes, uint64_t len, int32_t in_mem, void* out_records,
                       uint64_t capacity, int32_t out_mem, uint64_t* n_out) {
    if (!c || !n_out) return fail(GNM_ERR_INVALID_ARGUMENT, "null argument");
    if (out_mem != GNM_MEM_HOST && out_mem != GNM_MEM_DEVICE)
        return fail(GNM_ERR_INVALID_ARGUMENT, "out_mem must be GNM_MEM_HOST or GNM_MEM_DEVICE");
    return guarded([&] {
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        uint64_t n = 0;
        if (int e = archive_header(c, bytes, len, in_mem, &n)) return e;
        *n_out = n;
        if (n > capacity) return fail(GNM_ERR_CAPACITY, std::to_string(n) + " records exceed capacity");
        if (n == 0) return static_cast<int>(GNM_OK);
        cudaStream_t s = c->stream;
        const uint8_t* d = bytes + 20;
        uint8_t* din = nullptr;
        uint8_t* dout = static_cast<uint8_t*>(out_records);
        const bool dev_out = out_mem == GNM_MEM_DEVICE && (reinterpret_cast<uintptr_t>(out_records) & 15u) == 0;
        if (in_mem == GNM_MEM_HOST) {
            ck(cudaMallocAsync(reinterpret_cast<void**>(&din), n * 64, s), "cudaMallocAsync(archive)");
            ck(cudaMemcpyAsync(din, bytes + 20, n * 64, cudaMemcpyHostToDevice, s), "H2D archive");
            d = din;
        }
        uint8_t* staged = nullptr;
        if (!dev_out) {
            ck(cudaMallocAsync(reinterpret_cast<void**>(&staged), n * 64, s), "cudaMallocAsync(archive out)");
            dout = staged;
        }
        ck(gnm::launch_archive_decode(d, n, dout, s), "archive decode");
        c->kernel_launches += 1;
        if (!dev_out)
            ck(cudaMemcpyAsync(out_records, staged, n * 64,
                               out_mem == GNM_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, s),
               "copy records");
        if (din) ck(cudaFreeAsync(din, s), "cudaFreeAsync");
        if (staged) ck(cudaFreeAsync(staged, s), "cudaFreeAsync");
        ck(cudaStreamSynchronize(s), "cudaStreamSynchronize");
        return static_cast<int>(GNM_OK);
    });
}

int gnm_accumulate_archive(gnm_ctx* c, const gnm_registry* reg, const gnm_filter_params* params,
                           const uint8_t* bytes, uint64_t len, int32_t mem) {
    if (!c || !reg) return fail(GNM_ERR_INVALID_ARGUMENT, "null ctx/registry");
    return guarded([&] { return accumulate_archive(c, reg, params, bytes, len, mem, nullptr); });
}

int gnm_analyze_archive(gnm_ctx* c, const gnm_registry* reg, const gnm_filter_params* params,
                        const uint8_t* bytes, uint64_t len, int32_t mem, gnm_result* result) {
    if (!c || !reg) return fail(GNM_ERR_INVALID_ARGUMENT, "null ctx/registry");
    if (c->accumulating) return fail(GNM_ERR_INVALID_ARGUMENT, "an accumulation is in progress");
    return guarded([&] {
        if (int e = accumulate_archive(c, reg, params, bytes, len, mem, nullptr)) return e;
        return finalize(c, reg, result);
    });
}

int gnm_accumulate_window(gnm_ctx* c, const gnm_registry* reg, const gnm_filter_params* params,
                          const gnm_batch_soa* batch, uint64_t window_start_ms, uint64_t window_end_ms) {
    if (!c || !reg) return fail(GNM_ERR_INVALID_ARGUMENT, "null ctx/registry");
    const Window w{window_start_ms, window_end_ms};
    return guarded([&] { return accumulate_soa(c, reg, params, batch, &w); });
}

int gnm_accumulate_window_aos(gnm_ctx* c, const gnm_registry* reg, const gnm_filter_params* params,
                              const gnm_batch_aos* batch, uint64_t window_start_ms,
                              uint64_t window_end_ms) {
    if (!c || !reg) return fail(GNM_ERR_INVALID_ARGUMENT, "null ctx/registry");
    const Window w{window_start_ms, window_end_ms};
    return guarded([&] { return accumulate_aos(c, reg, params, batch, &w); });
}

namespace {
constexpr size_t kGraphCache = 32;

void drop_graphs(gnm_ctx* c) {
    for (auto& ge : c->graph_cache)
        if (ge.exec) cudaGraphExecDestroy(ge.exec);
    c->graph_cache.clear();
}

// A device-batch analysis repeated with the same inputs (column pointers,
// sizes, registry version, parameters, window) replays a CUDA graph of its
// whole device phase (K1, K2, K3a, K2b, K3b, the resets and the row
// copy-out): the second call with a given input set captures it, later ones
// launch it, for up to kGraphCache recent input sets (a ring of streaming
// batches replays too). Only the host part (wait, rows out) runs per call.
// Not for host batches, per-host mode, histogram export or timing (their
// host-side work differs per call), nor on the legacy default stream.
int analyze_graphed(gnm_ctx* c, const gnm_registry* reg, const gnm_filter_params* params,
                    const gnm_batch_soa* b, const gnm_batch_aos* ba, gnm_result* r, const Window* win) {
    gnm_ctx::GraphKey k;
    std::memset(&k, 0, sizeof k);
    if (b) {
        const void* cols[6] = {b->src_addr, b->dst_addr, b->d_pkts, b->d_octets, b->start_ms, b->end_ms};
        for (int i = 0; i < 6; ++i) k.cols[i] = cols[i];
        k.n = b->n;
    } else {
        k.cols[0] = ba->records;
        k.n = ba->n;
        k.aos = 1;
    }
    auto accumulate = [&]() {
        return b ? accumulate_soa(c, reg, params, b, win) : accumulate_aos(c, reg, params, ba, win);
    };
    k.reg = reg;
    k.version = reg->r.version();
    if (params) k.params = *params;
    else gnm_filter_params_default(&k.params);
    k.windowed = win != nullptr;
    k.win_lo = win ? win->lo : 0;
    k.win_hi = win ? win->hi : 0;
    k.threshold = r->threshold_bps;
    k.hot_mode = c->hot_mode;
    k.n_sites = static_cast<uint32_t>(reg->r.sites().size());
    // The registry's table and partials for this call (a no-op when nothing
    // changed; any reallocation or upload bumps alloc_gen and so the key).
    if (int e = begin_accumulate(c, reg)) return e;
    c->accumulating = false;
    k.alloc_gen = c->alloc_gen;
    // Entries of an older allocation generation can never match again.
    for (size_t i = 0; i < c->graph_cache.size();) {
        if (c->graph_cache[i].key.alloc_gen != k.alloc_gen) {
            if (c->graph_cache[i].exec) cudaGraphExecDestroy(c->graph_cache[i].exec);
            c->graph_cache.erase(c->graph_cache.begin() + static_cast<long>(i));
        } else {
            ++i;
        }
    }
    gnm_ctx::GraphEntry* hit = nullptr;
    for (auto& ge : c->graph_cache)
        if (ge.key == k) hit = &ge;
    if (hit && hit->exec) {
        hit->last_use = ++c->graph_clock;
        ck(cudaGraphLaunch(hit->exec, c->stream), "cudaGraphLaunch");
        c->kernel_launches += hit->kernels;
        c->k2_launches += 1;
        c->records = k.n;
        return finalize(c, reg, r, 2);
    }
    if (!hit) { // first sighting: remember the input set, run the call plainly
        if (c->graph_cache.size() >= kGraphCache) {
            auto lru = std::min_element(c->graph_cache.begin(), c->graph_cache.end(),
                                        [](const auto& x, const auto& y) { return x.last_use < y.last_use; });
            if (lru->exec) cudaGraphExecDestroy(lru->exec);
            c->graph_cache.erase(lru);
        }
        gnm_ctx::GraphEntry ge;
        ge.key = k;
        ge.last_use = ++c->graph_clock;
        c->graph_cache.push_back(ge);
        if (int e = accumulate()) return e;
        return finalize(c, reg, r);
    }
    // Second sighting: capture the device phase, then launch it.
    const uint64_t k0 = c->kernel_launches;
    ck(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal), "cudaStreamBeginCapture");
    int e = GNM_OK;
    c->capturing = true;
    try {
        e = accumulate();
        if (e == GNM_OK) e = finalize(c, reg, r, 1);
    } catch (...) {
        e = GNM_ERR_CUDA;
    }
    c->capturing = false;
    cudaGraph_t g = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(c->stream, &g);
    cudaGraphExec_t exec = nullptr;
    cudaError_t ie = cudaErrorUnknown;
    if (e == GNM_OK && ce == cudaSuccess && g && c->alloc_gen == k.alloc_gen)
        ie = cudaGraphInstantiate(&exec, g, 0);
    if (g) cudaGraphDestroy(g);
    clear_log(c); // the captured work has not run: start the accumulation over
    c->accumulating = false;
    if (ie != cudaSuccess) { // not capturable here: plain calls from now on
        cudaGetLastError();
        c->graphs = false;
        drop_graphs(c);
        c->kernel_launches = k0;
        if (int e2 = accumulate()) return e2;
        return finalize(c, reg, r);
    }
    hit->exec = exec;
    hit->kernels = c->kernel_launches - k0;
    hit->last_use = ++c->graph_clock;
    ck(cudaGraphLaunch(exec, c->stream), "cudaGraphLaunch");
    return finalize(c, reg, r, 2);
}

bool graph_eligible(const gnm_ctx* c, int mem, uint64_t n, const gnm_result* r) {
    return c->graphs && !c->timing && !c->hosts && mem == GNM_MEM_DEVICE && n > 0 && r && !r->histograms &&
           c->stream != nullptr && (!c->comm || c->comm->capturable());
}
} // namespace

int gnm_ctx_set_graphs(gnm_ctx* c, int enable) {
    if (!c) return fail(GNM_ERR_INVALID_ARGUMENT, "null ctx");
    c->graphs = enable != 0;
    drop_graphs(c);
    return GNM_OK;
}

int gnm_analyze_window(gnm_ctx* c, const gnm_registry* reg, const gnm_filter_params* params,
                       const gnm_batch_soa* batch, gnm_result* result) {
    if (!c || !reg || !result) return fail(GNM_ERR_INVALID_ARGUMENT, "null ctx/registry/result");
    if (c->accumulating) return fail(GNM_ERR_INVALID_ARGUMENT, "an accumulation is in progress");
    const Window w{result->window_start_ms, result->window_end_ms};
    return guarded([&] {
        if (batch && graph_eligible(c, batch->mem, batch->n, result))
            return analyze_graphed(c, reg, params, batch, nullptr, result, &w);
        if (int e = accumulate_soa(c, reg, params, batch, &w)) return e;
        return finalize(c, reg, result);
    });
}

int gnm_analyze(gnm_ctx* c, const gnm_registry* reg, const gnm_filter_params* params,
                const gnm_batch_soa* batch, gnm_result* result) {
    if (!c || !reg) return fail(GNM_ERR_INVALID_ARGUMENT, "null ctx/registry");
    if (c->accumulating) return fail(GNM_ERR_INVALID_ARGUMENT, "an accumulation is in progress");
    return guarded([&] {
        if (batch && graph_eligible(c, batch->mem, batch->n, result))
            return analyze_graphed(c, reg, params, batch, nullptr, result, nullptr);
        if (int e = accumulate_soa(c, reg, params, batch)) return e;
        return finalize(c, reg, result);
    });
}

int gnm_analyze_aos(gnm_ctx* c, const gnm_registry* reg, const gnm_filter_params* params,
                    const gnm_batch_aos* batch, gnm_result* result) {
    if (!c || !reg) return fail(GNM_ERR_INVALID_ARGUMENT, "null ctx/registry");
    if (c->accumulating) return fail(GNM_ERR_INVALID_ARGUMENT, "an accumulation is in progress");
    return guarded([&] {
        if (batch && batch->records && graph_eligible(c, batch->mem, batch->n, result))
            return analyze_graphed(c, reg, params, nullptr, batch, result, nullptr);
        if (int e = accumulate_aos(c, reg, params, batch)) return e;
        return finalize(c, reg, result);
    });
}

int gnm_get_partials(gnm_ctx* c, const gnm_registry* reg, gnm_partials* out) {
    if (!c || !reg || !out) return fail(GNM_ERR_INVALID_ARGUMENT, "null argument");
    return guarded([&] {
        if (int e = begin_accumulate(c, reg)) return e;
        out->sums = reinterpret_cast<uint64_t*>(c->P.sums);
        out->min_bps = reinterpret_cast<double*>(c->P.mn);
        out->max_bps = reinterpret_cast<double*>(c->P.mx);
        out->coarse = c->P.coarse;
        out->fine = c->P.fine;
        out->n_sites = c->P.n_sites;
        out->sums_count = static_cast<uint64_t>(c->P.n_sites) * 4 + 4;
        out->coarse_count = static_cast<uint64_t>(c->P.n_sites) * gnm::kCoarse;
        out->fine_count = static_cast<uint64_t>(c->P.n_sites) * gnm::kFineW;
        return static_cast<int>(GNM_OK);
    });
}

int gnm_classify(gnm_ctx* c, const gnm_registry* reg, const gnm_filter_params* params,
                 const gnm_batch_soa* b, uint32_t* out, int32_t out_mem) {
    if (!c || !reg || !out) return fail(GNM_ERR_INVALID_ARGUMENT, "null argument");
    if (int e = check_soa(b)) return e;
    return guarded([&] {
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        ensure_table(c, reg);
        if (b->n == 0) return static_cast<int>(GNM_OK);
        const gnm::DevParams p = dev_params(c, params);
        std::vector<void*> temps;
        auto dev_copy = [&](const void* h, size_t bytes) -> const void* {
            void* d = nullptr;
            ck(cudaMalloc(&d, bytes), "cudaMalloc");
            temps.push_back(d);
            ck(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, c->stream), "cudaMemcpyAsync");
            return d;
        };
        int rc = GNM_OK;
        try {
            gnm::DevSoA d{b->src_addr, b->dst_addr, b->d_pkts, b->d_octets, b->start_ms, b->end_ms, b->n};
            if (b->mem == GNM_MEM_HOST) {
                d.src = static_cast<const uint32_t*>(dev_copy(b->src_addr, b->n * 4));
                d.dst = static_cast<const uint32_t*>(dev_copy(b->dst_addr, b->n * 4));
                d.pkts = static_cast<const uint32_t*>(dev_copy(b->d_pkts, b->n * 4));
                d.octets = static_cast<const uint32_t*>(dev_copy(b->d_octets, b->n * 4));
                d.start = static_cast<const uint64_t*>(dev_copy(b->start_ms, b->n * 8));
                d.end = static_cast<const uint64_t*>(dev_copy(b->end_ms, b->n * 8));
            }
            uint32_t* dout = out;
            if (out_mem == GNM_MEM_HOST) {
                void* t = nullptr;
                ck(cudaMalloc(&t, b->n * 4), "cudaMalloc");
                temps.push_back(t);
                dout = static_cast<uint32_t*>(t);
            }
            gnm::DevBatch cb{};
            cb.n = b->n;
            cb.aos = true; // the classify kernel uses the plain launch shape
            const gnm::LaunchCfg cfg = gnm::k2_config(c->device, cb, c->table.n_words, false, c->occ);
            ck(gnm::launch_classify(cfg, d, c->table, p, dout, c->stream), "classify launch");
            c->kernel_launches += 1;
            if (out_mem == GNM_MEM_HOST)
                ck(cudaMemcpyAsync(out, dout, b->n * 4, cudaMemcpyDeviceToHost, c->stream), "cudaMemcpyAsync");
            ck(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");
        } catch (...) {
            for (void* t : temps) cudaFree(t);
            throw;
        }
        for (void* t : temps) cudaFree(t);
        return rc;
    });
}

// ---- warnings -------------------------------------------------------------------
int gnm_warning_state_create(gnm_warning_state** out) {
    if (!out) return fail(GNM_ERR_INVALID_ARGUMENT, "null out");
    return guarded([&] {
        *out = new gnm_warning_state();
        return static_cast<int>(GNM_OK);
    });
}
void gnm_warning_state_destroy(gnm_warning_state* st) { delete st; }
uint32_t gnm_warning_state_streak(const gnm_warning_state* st, uint32_t site) {
    if (!st) return 0;
    auto it = st->streaks.find(site);
    return it == st->streaks.end() ? 0 : it->second;
}

// evaluate_warnings, monitor.cpp:13-34.
int gnm_evaluate_warnings(const gnm_result* r, gnm_warning_state* st, double threshold,
                          gnm_warning* out, size_t cap, size_t* n_out) {
    if (!r || !st) return fail(GNM_ERR_INVALID_ARGUMENT, "null argument");
    if (r->n_sites && !r->sites) return fail(GNM_ERR_INVALID_ARGUMENT, "null sites");
    return guarded([&] {
        size_t n = 0;
        for (uint32_t s = 0; s < r->n_sites; ++s) {
            const gnm_site_stats& ss = r->sites[s];
            if (ss.flow_count == 0) continue; // frozen (monitor.cpp:18-20)
            uint32_t& streak = st->streaks[s];
            if (ss.median_bps < threshold) ++streak;
            else streak = 0;
            if (streak >= 2) {
                if (n < cap && out) out[n] = gnm_warning{s, streak, ss.median_bps};
                ++n;
            }
        }
        if (n_out) *n_out = n;
        return static_cast<int>(GNM_OK);
    });
}

// ---- multi-GPU inside the library ---------------------------------------------

int gnm_comm_unique_id(unsigned char out[GNM_COMM_ID_BYTES]) {
    if (!out) return fail(GNM_ERR_INVALID_ARGUMENT, "null out");
    return guarded([&] {
        gnm::nccl_unique_id(out);
        return static_cast<int>(GNM_OK);
    });
}

int gnm_ctx_comm_init(gnm_ctx* c, int nranks, int rank, const unsigned char id[GNM_COMM_ID_BYTES]) {
    if (!c || !id) return fail(GNM_ERR_INVALID_ARGUMENT, "null argument");
    if (nranks < 1 || rank < 0 || rank >= nranks) return fail(GNM_ERR_INVALID_ARGUMENT, "bad rank / nranks");
    if (c->accumulating) return fail(GNM_ERR_INVALID_ARGUMENT, "attach a communicator between accumulations");
    return guarded([&] {
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        ck(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");
        drop_graphs(c); // graphs captured without the collectives must not replay
        c->comm = gnm::nccl_comm(nranks, rank, id);
        return static_cast<int>(GNM_OK);
    });
}

int gnm_ctx_comm_destroy(gnm_ctx* c) {
    if (!c) return fail(GNM_ERR_INVALID_ARGUMENT, "null ctx");
    if (c->accumulating) return fail(GNM_ERR_INVALID_ARGUMENT, "detach a communicator between accumulations");
    return guarded([&] {
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        ck(cudaStreamSynchronize(c->stream), "cudaStreamSynchronize");
        drop_graphs(c); // their captured collectives refer to this communicator
        c->comm.reset();
        return static_cast<int>(GNM_OK);
    });
}

int gnm_ctx_comm_size(gnm_ctx* c) { return c && c->comm ? c->comm->nranks() : 1; }

} // extern "C"

struct gnm_group {
    std::vector<gnm_ctx*> ctx;
    int kind = GNM_GROUP_NCCL;
    bool broken = false; // a rank failed and the communicators were aborted
};

namespace {

// One host thread per rank (each drives its own device and communicator,
// as NCCL requires when one process owns several ranks): rank i runs `work`
// on its context; the first failing rank's status and message are returned.
template <typename F>
int on_every_rank(gnm_group* g, F&& work) {
    const int n = static_cast<int>(g->ctx.size());
    std::vector<int> st(n, GNM_OK);
    std::vector<std::string> msg(n);
    std::atomic<int> first_fail{-1}; // the root cause, not the ranks it aborted
    auto body = [&](int i) {
        st[i] = guarded([&] {
            ck(cudaSetDevice(g->ctx[i]->device), "cudaSetDevice");
            return work(i, g->ctx[i]);
        });
        if (st[i] != GNM_OK) {
            msg[i] = g_last_error;
            int none = -1;
            first_fail.compare_exchange_strong(none, i);
            // the other ranks may be blocked in (or about to enter) a
            // collective this rank will never join: abort the clique
            for (gnm_ctx* c : g->ctx)
                if (c->comm) c->comm->abort();
            g->broken = true;
        }
    };
    if (g->broken) return fail(GNM_ERR_COMM, "the group's communicators were aborted by an earlier failure");
    if (n == 1) {
        body(0);
    } else {
        std::vector<std::thread> th;
        for (int i = 0; i < n; ++i) th.emplace_back(body, i);
        for (auto& t : th) t.join();
    }
    if (const int i = first_fail.load(); i >= 0) return fail(st[i], "rank " + std::to_string(i) + ": " + msg[i]);
    return GNM_OK;
}

// Shard i of n records over N ranks: the reference's worker boundaries.
std::pair<uint64_t, uint64_t> shard(uint64_t n, int i, int N) {
    const unsigned __int128 a = static_cast<unsigned __int128>(n) * i / N;
    const unsigned __int128 b = static_cast<unsigned __int128>(n) * (i + 1) / N;
    return {static_cast<uint64_t>(a), static_cast<uint64_t>(b)};
}

int group_analyze(gnm_group* g, const gnm_registry* reg, const gnm_filter_params* params, const gnm_batch_soa* b,
                  const gnm_batch_aos* ba, gnm_result* r) {
    if (!g || !reg || !r) return fail(GNM_ERR_INVALID_ARGUMENT, "null argument");
    if (b) {
        if (int e = check_soa(b)) return e;
    } else {
        if (!ba) return fail(GNM_ERR_INVALID_ARGUMENT, "null batch");
        if (ba->n && !ba->records) return fail(GNM_ERR_INVALID_ARGUMENT, "null records");
        if (ba->mem == GNM_MEM_DEVICE && reinterpret_cast<uintptr_t>(ba->records) % 8)
            return fail(GNM_ERR_INVALID_ARGUMENT, "device FlowRecord rows must be 8-byte aligned");
    }
    const uint32_t n_sites = static_cast<uint32_t>(reg->r.sites().size());
    if (r->sites_capacity < n_sites || (n_sites && !r->sites))
        return fail(GNM_ERR_CAPACITY, "result.sites holds fewer rows than the registry has sites");
    const int N = static_cast<int>(g->ctx.size());
    for (gnm_ctx* c : g->ctx)
        if (c->hosts != g->ctx[0]->hosts)
            return fail(GNM_ERR_INVALID_ARGUMENT, "per-host mode must be alike on every rank");
    std::vector<std::vector<gnm_site_stats>> rows(N);
    std::vector<gnm_result> res(N, *r);
    return on_every_rank(g, [&](int i, gnm_ctx* c) -> int {
        const uint64_t n = b ? b->n : ba->n;
        const auto [lo, hi] = shard(n, i, N);
        if (i) { // the other ranks' rows stay internal; histograms: all-reduced, not copied out
            rows[i].resize(n_sites);
            res[i].sites = rows[i].data();
        }
        int e;
        if (b) {
            gnm_batch_soa s = *b;
            s.src_addr += lo;
            s.dst_addr += lo;
            s.d_pkts += lo;
            s.d_octets += lo;
            s.start_ms += lo;
            s.end_ms += lo;
            s.n = hi - lo;
            e = accumulate_soa(c, reg, params, &s);
        } else {
            gnm_batch_aos a = *ba;
            a.records = static_cast<const unsigned char*>(ba->records) + lo * GNM_FLOW_RECORD_BYTES;
            a.n = hi - lo;
            e = accumulate_aos(c, reg, params, &a);
        }
        if (e) {
            gnm_reset(c);
            return e;
        }
        // test hook: one rank fails between its accumulation and the combine
        // (the others must not hang in a collective it never joins)
        static const int fail_rank = [] {
            const char* v = std::getenv("GNM_TEST_FAIL_RANK");
            return v ? std::atoi(v) : -1;
        }();
        if (i == fail_rank) {
            gnm_reset(c);
            return fail(GNM_ERR_INVALID_ARGUMENT, "injected failure (GNM_TEST_FAIL_RANK)");
        }
        c->discard_hist_out = i != 0;
        try {
            e = finalize(c, reg, &res[i]);
        } catch (...) {
            c->discard_hist_out = false;
            throw;
        }
        c->discard_hist_out = false;
        if (!e && i == 0) *r = res[0];
        return e;
    });
}

} // namespace

extern "C" {

int gnm_group_create(const int* devices, int n, int kind, gnm_group** out) {
    if (!devices || n < 1 || !out) return fail(GNM_ERR_INVALID_ARGUMENT, "bad group arguments");
    if (kind != GNM_GROUP_NCCL && kind != GNM_GROUP_LOOPBACK) return fail(GNM_ERR_INVALID_ARGUMENT, "bad group kind");
    *out = nullptr;
    auto* g = new gnm_group();
    g->kind = kind;
    for (int i = 0; i < n; ++i) {
        gnm_ctx* c = nullptr;
        if (int e = gnm_ctx_create(devices[i], &c)) {
            gnm_group_destroy(g);
            return e;
        }
        g->ctx.push_back(c);
    }
    const int e = guarded([&] {
        auto comms = kind == GNM_GROUP_NCCL ? gnm::nccl_clique(devices, n) : gnm::loopback_clique(n);
        for (int i = 0; i < n; ++i) {
            g->ctx[i]->comm = std::move(comms[i]);
            g->ctx[i]->stage_share = static_cast<unsigned>(n); // the ranks load at once
        }
        return static_cast<int>(GNM_OK);
    });
    if (e) {
        gnm_group_destroy(g);
        return e;
    }
    *out = g;
    return GNM_OK;
}

void gnm_group_destroy(gnm_group* g) {
    if (!g) return;
    for (gnm_ctx* c : g->ctx) gnm_ctx_destroy(c);
    delete g;
}

int gnm_group_size(const gnm_group* g) { return g ? static_cast<int>(g->ctx.size()) : 0; }

gnm_ctx* gnm_group_ctx(gnm_group* g, int rank) {
    return g && rank >= 0 && rank < static_cast<int>(g->ctx.size()) ? g->ctx[rank] : nullptr;
}

int gnm_group_analyze(gnm_group* g, const gnm_registry* reg, const gnm_filter_params* params,
                      const gnm_batch_soa* batch, gnm_result* result) {
    if (!batch) return fail(GNM_ERR_INVALID_ARGUMENT, "null batch");
    return group_analyze(g, reg, params, batch, nullptr, result);
}

int gnm_group_analyze_aos(gnm_group* g, const gnm_registry* reg, const gnm_filter_params* params,
                          const gnm_batch_aos* batch, gnm_result* result) {
    if (!batch) return fail(GNM_ERR_INVALID_ARGUMENT, "null batch");
    return group_analyze(g, reg, params, nullptr, batch, result);
}

uint64_t gnm_group_host_count(gnm_group* g) { return g && !g->ctx.empty() ? gnm_host_count(g->ctx[0]) : 0; }

int gnm_group_host_results(gnm_group* g, gnm_host_stats* out, uint64_t capacity) {
    if (!g || g->ctx.empty()) return fail(GNM_ERR_INVALID_ARGUMENT, "null group");
    return gnm_host_results(g->ctx[0], out, capacity, nullptr); // every rank holds the same global rows
}

int gnm_group_host_histogram_entries(gnm_group* g, uint32_t* rows, uint32_t* buckets, uint32_t* counts,
                                     uint64_t capacity, uint64_t* n_entries) {
    if (!g || g->ctx.empty() || !n_entries) return fail(GNM_ERR_INVALID_ARGUMENT, "null argument");
    // Each rank's entries count its own flows over the global rows; the
    // group's histograms are their sum, merged here in (row, bucket) order.
    std::vector<uint64_t> keys;
    std::vector<uint32_t> cnts;
    for (gnm_ctx* c : g->ctx) {
        uint64_t n = 0;
        if (int e = gnm_host_histogram_entries(c, nullptr, nullptr, nullptr, 0, &n)) return e;
        std::vector<uint32_t> r(n), b(n), k(n);
        if (n)
            if (int e = gnm_host_histogram_entries(c, r.data(), b.data(), k.data(), n, &n)) return e;
        for (uint64_t i = 0; i < n; ++i) {
            keys.push_back(static_cast<uint64_t>(r[i]) << 32 | b[i]);
            cnts.push_back(k[i]);
        }
    }
    std::vector<uint64_t> order(keys.size());
    for (uint64_t i = 0; i < order.size(); ++i) order[i] = i;
    std::sort(order.begin(), order.end(), [&](uint64_t x, uint64_t y) { return keys[x] < keys[y]; });
    uint64_t m = 0;
    for (uint64_t i = 0; i < order.size(); ++i) {
        const uint64_t k = keys[order[i]];
        const bool fresh = i == 0 || k != keys[order[i - 1]];
        if (fresh) ++m;
        if (!rows) continue;
        if (m > capacity || !buckets || !counts) return fail(GNM_ERR_CAPACITY, "host histogram entries: capacity");
        if (fresh) {
            rows[m - 1] = static_cast<uint32_t>(k >> 32);
            buckets[m - 1] = static_cast<uint32_t>(k);
            counts[m - 1] = 0;
        }
        counts[m - 1] += cnts[order[i]];
    }
    *n_entries = m;
    return GNM_OK;
}

} // extern "C"

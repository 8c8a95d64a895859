// The drop-in C++ adapter: flowmon::aggregate and flowmon::aggregate_partitioned
// with the reference's exact signatures (rate_engine.hpp:143-154), computed on
// the B200 through the C-ABI (include/gnetmon.h, libgnetmon.so).
//
// Link-time substitution (the reference has no plugin mechanism, SURVEY.md
// §8b): the reference's rate_engine.cpp is compiled with
//   -Daggregate=cpu_aggregate -Daggregate_partitioned=cpu_aggregate_partitioned
// so its CPU path stays callable under those names, and this file provides
// the two symbols every caller binds -- monitor.cpp:118 (run_cycle),
// toolkit.cpp:297 (run_bench), acceptance.cpp:220/351, engine_test.cpp. The
// rest of rate_engine.cpp (RateHistogram, classify, flow_rate, bucket_index,
// attribute) is the reference's own code.
//
// The whole AnalysisResult is produced, not just the site level: every
// SiteResult with its RateStats and RateHistogram, and SiteResult::hosts with
// each host's RateStats and RateHistogram (rate_engine.cpp:255-292), so the
// reference's AnalysisResult::operator== (rate_engine.hpp:112-119) can judge
// it against cpu_aggregate.
//
// RateHistogram keeps its state private (rate_engine.hpp:68-73); it is rebuilt
// through its public add(): one add at the exact min rate carrying the whole
// u128 micro-bps sum, one at the exact max, and the remaining count of every
// bucket at a rate inside that bucket and inside [min, max]. count_,
// sum_ubps_, min_bps_, max_bps_ and buckets_ then equal the GPU's exact
// integers and doubles field for field.
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <memory>
#include <mutex>
#include <thread>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "flowmon/rate_engine.hpp"
#include "flowmon/site_catalog.hpp"
#include "gnetmon.h"

namespace flowmon {

namespace {

using u128 = unsigned __int128;

[[noreturn]] void gpu_fail(const char* what) {
    throw std::runtime_error(std::string("flowmon GPU adapter: ") + what + ": " + gnm_last_error());
}

void check(int status, const char* what) {
    if (status != GNM_OK) gpu_fail(what);
}

// One context per host thread (gnetmon.h: calls on a context are serialized;
// the reference's callers are single-threaded per monitor).
// GNM_ADAPTER_DEVICES="0,1,2,3" shards every call across those GPUs
// (gnm_group: the reference's worker boundaries, the combine over NCCL);
// "loopback:0,0" runs the same multi-rank orchestration through host memory
// (a test hook for one-GPU boxes). Default: one context on GNM_DEVICE or 0.
struct Engine {
    gnm_group* group = nullptr;
    gnm_ctx* ctx = nullptr; // the only context, or rank 0 of the group
    gnm_registry* reg = nullptr;
    // the catalog the registry was compiled from: its (prefix24, site) entries
    // and sites, compared on every call (a rebuild only on change)
    std::vector<std::pair<std::uint32_t, SiteId>> entries;
    std::size_t n_sites = 0;
    std::vector<std::uint32_t> ent_r, ent_b, ent_c; // host histogram entries (reused)

    Engine() {
        if (const char* spec = std::getenv("GNM_ADAPTER_DEVICES")) {
            std::string s = spec;
            int kind = GNM_GROUP_NCCL;
            if (s.rfind("loopback:", 0) == 0) {
                kind = GNM_GROUP_LOOPBACK;
                s = s.substr(9);
            }
            std::vector<int> devs;
            for (std::size_t a = 0; a < s.size();) {
                const std::size_t b = std::min(s.find(',', a), s.size());
                devs.push_back(std::stoi(s.substr(a, b - a)));
                a = b + 1;
            }
            check(gnm_group_create(devs.data(), static_cast<int>(devs.size()), kind, &group), "gnm_group_create");
            for (int i = 0; i < gnm_group_size(group); ++i)
                check(gnm_ctx_set_hosts(gnm_group_ctx(group, i), 1), "gnm_ctx_set_hosts");
            ctx = gnm_group_ctx(group, 0);
        } else {
            const char* dev = std::getenv("GNM_DEVICE");
            check(gnm_ctx_create(dev ? std::atoi(dev) : 0, &ctx), "gnm_ctx_create");
            check(gnm_ctx_set_hosts(ctx, 1), "gnm_ctx_set_hosts"); // SiteResult::hosts
        }
    }
    ~Engine() {
        gnm_registry_destroy(reg);
        if (group) gnm_group_destroy(group);
        else gnm_ctx_destroy(ctx);
    }
    int host_entries(std::uint32_t* rows, std::uint32_t* buckets, std::uint32_t* counts, std::uint64_t cap,
                     std::uint64_t* n) {
        return group ? gnm_group_host_histogram_entries(group, rows, buckets, counts, cap, n)
                     : gnm_host_histogram_entries(ctx, rows, buckets, counts, cap, n);
    }
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;

    // SiteCatalog -> gnm_registry, sites in registration order so SiteIds
    // (dense registration indices, site_catalog.cpp:91) are identical.
    void sync(const SiteCatalog& catalog) {
        if (reg && n_sites == catalog.site_count() && entries == catalog.entries()) return;
        gnm_registry* r = nullptr;
        check(gnm_registry_create(&r), "gnm_registry_create");
        std::vector<gnm_cidr> cidrs;
        for (const SiteCatalog::Site& s : catalog.sites()) {
            cidrs.clear();
            for (const Cidr& c : s.cidrs) cidrs.push_back({c.addr, static_cast<std::int32_t>(c.prefix_len)});
            std::uint32_t id = 0;
            if (gnm_registry_register_site(r, s.name.c_str(), cidrs.data(), cidrs.size(), &id) != GNM_OK ||
                id != s.id) {
                gnm_registry_destroy(r);
                gpu_fail("registry rebuild");
            }
        }
        gnm_registry_destroy(reg);
        reg = r;
        entries = catalog.entries();
        n_sites = catalog.site_count();
    }
};

Engine& engine() {
    thread_local Engine e;
    return e;
}

// GNM_ADAPTER_PROFILE=1: per-call phase times on stderr (diagnosis only).
struct PhaseClock {
    bool on = std::getenv("GNM_ADAPTER_PROFILE") != nullptr;
    std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
    void mark(const char* what) {
        if (!on) return;
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[adapter] %-22s %8.2f ms\n", what,
                     std::chrono::duration<double, std::milli>(now - t).count());
        t = now;
    }
};

struct BucketCount {
    std::uint32_t bucket;
    std::uint32_t count;
};

// RateHistogram with exactly these buckets (ascending, non-zero), count, u128
// sum and bounds, through its public add() (see the file comment).
RateHistogram rebuild_histogram(const std::vector<BucketCount>& buckets, std::uint64_t count, u128 sum,
                                double min_bps, double max_bps) {
    RateHistogram h;
    if (count == 0) {
        if (!buckets.empty()) throw std::runtime_error("flowmon GPU adapter: buckets without flows");
        return h;
    }
    std::uint64_t total = 0;
    for (const BucketCount& b : buckets) total += b.count;
    const std::size_t bmin = bucket_index(min_bps), bmax = bucket_index(max_bps);
    std::vector<BucketCount> rem = buckets;
    auto take = [&](std::size_t k) {
        for (BucketCount& b : rem)
            if (b.bucket == k && b.count) {
                --b.count;
                return;
            }
        throw std::runtime_error("flowmon GPU adapter: min/max outside the histogram's buckets");
    };
    if (total != count || min_bps > max_bps)
        throw std::runtime_error("flowmon GPU adapter: histogram inconsistent with its stats");
    h.add(min_bps, sum);
    take(bmin);
    if (count > 1) {
        h.add(max_bps, 0);
        take(bmax);
    }
    for (const BucketCount& b : rem) {
        double rate;
        if (b.bucket == bmin) rate = min_bps;
        else if (b.bucket == bmax) rate = max_bps;
        else if (b.bucket + 1 < kBucketCount) rate = static_cast<double>(b.bucket) * kBucketWidthBps + kBucketWidthBps / 2;
        else throw std::runtime_error("flowmon GPU adapter: overflow bucket above max");
        // strictly between bmin and bmax: the midpoint lies inside (min, max)
        for (std::uint32_t i = 0; i < b.count; ++i) h.add(rate, 0);
    }
    return h;
}

RateStats stats_of(std::uint64_t count, double min_bps, double max_bps, double avg_bps, double median_bps) {
    RateStats s;
    s.flow_count = count;
    s.min_bps = min_bps;
    s.max_bps = max_bps;
    s.avg_bps = avg_bps;
    s.median_bps = median_bps;
    return s;
}

u128 join(std::uint64_t lo, std::uint64_t hi) { return static_cast<u128>(hi) << 64 | lo; }

// The GPU's finalize (site rows, tallies, per-host rows and their sparse
// histograms) -> AnalysisResult, in the reference's map order.
AnalysisResult collect(Engine& e, const gnm_result& r, const std::vector<gnm_site_stats>& rows, PhaseClock& clk) {
    AnalysisResult out;
    out.window_start_ms = r.window_start_ms;
    out.window_end_ms = r.window_end_ms;
    out.tallies.forward = r.tallies.forward;
    out.tallies.pure_ack = r.tallies.pure_ack;
    out.tallies.administrative = r.tallies.administrative;
    out.tallies.unmatched = r.tallies.unmatched;

    const std::uint64_t nh = gnm_host_count(e.ctx);
    std::vector<gnm_host_stats> hosts(nh);
    if (nh) check(gnm_host_results(e.ctx, hosts.data(), nh, nullptr), "gnm_host_results");
    std::uint64_t ne = 0;
    clk.mark("host rows");
    check(e.host_entries(nullptr, nullptr, nullptr, 0, &ne), "host histogram entries");
    clk.mark("entries: sort + count");
    // The engine's entry buffers persist across calls (grown, never shrunk):
    // a fresh 100+ MB allocation per call would page-fault on first touch.
    if (e.ent_r.size() < ne) {
        e.ent_r.resize(ne);
        e.ent_b.resize(ne);
        e.ent_c.resize(ne);
    }
    std::uint32_t *er = e.ent_r.data(), *eb = e.ent_b.data(), *ec = e.ent_c.data();
    if (ne) check(e.host_entries(er, eb, ec, ne, &ne), "host histogram entries");
    clk.mark("entries: export");

    // Host rows arrive in (site, host) order: one group of rows per present
    // site. Groups (and their histogram entries) are independent, so they
    // are rebuilt on several host threads -- RateHistogram::add runs once
    // per flow -- and moved into the ordered maps afterwards.
    struct Group {
        std::uint32_t site;
        std::uint64_t row0, row1, e0, e1;
    };
    std::vector<Group> groups;
    for (std::uint64_t i = 0, ei = 0; i < nh;) {
        Group g{hosts[i].site, i, i, ei, ei};
        if (g.site >= rows.size() || rows[g.site].flow_count == 0)
            throw std::runtime_error("flowmon GPU adapter: host row of an empty or unknown site");
        for (; i < nh && hosts[i].site == g.site; ++i)
            for (; ei < ne && er[ei] == i; ++ei) {
            }
        g.row1 = i;
        g.e1 = ei;
        groups.push_back(g);
    }
    if (!groups.empty() && groups.back().e1 != ne)
        throw std::runtime_error("flowmon GPU adapter: histogram entries past the last host row");
    std::vector<SiteResult> built(groups.size());
    auto build = [&](std::size_t gi) {
        const Group& gr = groups[gi];
        const gnm_site_stats& g = rows[gr.site];
        SiteResult& sr = built[gi];
        std::vector<std::uint64_t> site_dense(kBucketCount, 0);
        std::vector<BucketCount> hb, sb;
        std::uint64_t host_flows = 0, ei = gr.e0;
        for (std::uint64_t i = gr.row0; i < gr.row1; ++i) {
            const gnm_host_stats& h = hosts[i];
            hb.clear();
            for (; ei < gr.e1 && er[ei] == i; ++ei) {
                hb.push_back({eb[ei], ec[ei]});
                site_dense[eb[ei]] += ec[ei];
            }
            HostResult& hr = sr.hosts.emplace_hint(sr.hosts.end(), h.host, HostResult{})->second;
            hr.stats = stats_of(h.flow_count, h.min_bps, h.max_bps, h.avg_bps, h.median_bps);
            hr.histogram = rebuild_histogram(hb, h.flow_count, join(h.rate_ubps_lo, h.rate_ubps_hi), h.min_bps,
                                             h.max_bps);
            host_flows += h.flow_count;
        }
        if (host_flows != g.flow_count)
            throw std::runtime_error("flowmon GPU adapter: host rows do not sum to the site's flows");
        for (std::size_t k = 0; k < kBucketCount; ++k)
            if (site_dense[k]) {
                if (site_dense[k] > UINT32_MAX) throw std::runtime_error("flowmon GPU adapter: bucket overflow");
                sb.push_back({static_cast<std::uint32_t>(k), static_cast<std::uint32_t>(site_dense[k])});
            }
        sr.stats = stats_of(g.flow_count, g.min_bps, g.max_bps, g.avg_bps, g.median_bps);
        sr.histogram = rebuild_histogram(sb, g.flow_count, join(g.rate_ubps_lo, g.rate_ubps_hi), g.min_bps,
                                         g.max_bps);
    };
    const unsigned nt = std::max(1u, std::min<unsigned>(std::thread::hardware_concurrency(), 16u));
    if (nt == 1 || groups.size() < 2 || r.tallies.forward < (1u << 16)) {
        for (std::size_t gi = 0; gi < groups.size(); ++gi) build(gi);
    } else {
        std::atomic<std::size_t> next{0};
        std::vector<std::exception_ptr> errs(nt);
        std::vector<std::thread> th;
        for (unsigned t = 0; t < nt; ++t)
            th.emplace_back([&, t] {
                try {
                    for (std::size_t gi; (gi = next.fetch_add(1)) < groups.size();) build(gi);
                } catch (...) {
                    errs[t] = std::current_exception();
                }
            });
        for (auto& x : th) x.join();
        for (auto& ep : errs)
            if (ep) std::rethrow_exception(ep);
    }
    clk.mark("rebuild histograms");
    for (std::size_t gi = 0; gi < groups.size(); ++gi)
        out.sites.emplace_hint(out.sites.end(), groups[gi].site, std::move(built[gi]));
    clk.mark("maps");
    std::uint64_t present = 0;
    for (const gnm_site_stats& g : rows) present += g.flow_count != 0;
    if (present != groups.size()) throw std::runtime_error("flowmon GPU adapter: site without host rows");
    return out;
}

// Slices (the reference's run_partitioned, rate_engine.cpp:294-331) become
// successive gnm_accumulate_aos calls into one accumulation; the GPU result
// is identical for any split (exact integer reductions), as the reference's
// is by its monoid contract.
AnalysisResult run_gpu(std::span<const FlowRecord> view, const SiteCatalog& catalog, const FilterParams& params,
                       const std::vector<std::size_t>& boundaries, std::uint64_t window_start_ms,
                       std::uint64_t window_end_ms) {
    static_assert(sizeof(FlowRecord) == GNM_FLOW_RECORD_BYTES, "FlowRecord is the 64-byte gnm_batch_aos row");
    PhaseClock clk;
    Engine& e = engine();
    e.sync(catalog);
    clk.mark("registry");
    const gnm_filter_params p{params.ack_avg_size_max, params.min_packets, params.min_duration_ms,
                              params.workers};
    std::vector<gnm_site_stats> rows(e.n_sites);
    gnm_result r{};
    r.window_start_ms = window_start_ms; // copied through, never a filter (rate_engine.cpp:257-258)
    r.window_end_ms = window_end_ms;
    r.threshold_bps = GNM_DEFAULT_WARN_THRESHOLD_BPS;
    r.sites_capacity = static_cast<std::uint32_t>(rows.size());
    r.sites = rows.data();
    r.histograms = nullptr; // site histograms are the sums of the host histograms
    if (e.group) {
        // shards across the group's GPUs by the reference's worker boundaries;
        // caller slices need no separate pass (the result is partition-independent)
        for (std::size_t b : boundaries)
            if (b > view.size()) throw std::out_of_range("aggregate_partitioned: boundary past the view");
        const gnm_batch_aos b{view.data(), view.size(), GNM_MEM_HOST};
        check(gnm_group_analyze_aos(e.group, e.reg, &p, &b, &r), "gnm_group_analyze_aos");
        clk.mark("gpu (group)");
        return collect(e, r, rows, clk);
    }
    std::size_t prev = 0;
    auto slice = [&](std::size_t end) {
        if (end < prev || end > view.size()) {
            gnm_reset(e.ctx);
            throw std::out_of_range("aggregate_partitioned: boundaries must be sorted and within the view");
        }
        const gnm_batch_aos b{view.data() + prev, end - prev, GNM_MEM_HOST};
        if (int st = gnm_accumulate_aos(e.ctx, e.reg, &p, &b)) {
            gnm_reset(e.ctx);
            check(st, "gnm_accumulate_aos");
        }
        prev = end;
    };
    for (std::size_t b : boundaries) slice(b);
    slice(view.size());
    clk.mark("accumulate (H2D+K2)");
    check(gnm_finalize(e.ctx, e.reg, &r), "gnm_finalize");
    clk.mark("finalize (K3+hosts)");
    return collect(e, r, rows, clk);
}

} // namespace

// rate_engine.cpp:335-347. `workers` and `mode` select nothing on the GPU:
// the result is identical for every worker count and lookup mode, by the
// reference's own contract (engine_test.cpp:344-360).
AnalysisResult aggregate(std::span<const FlowRecord> view, const SiteCatalog& catalog, const FilterParams& params,
                         unsigned /*workers*/, LookupMode /*mode*/, std::uint64_t window_start_ms,
                         std::uint64_t window_end_ms) {
    return run_gpu(view, catalog, params, {}, window_start_ms, window_end_ms);
}

// rate_engine.cpp:349-355 (the test hook over caller-chosen slices).
AnalysisResult aggregate_partitioned(std::span<const FlowRecord> view, const SiteCatalog& catalog,
                                     const FilterParams& params, const std::vector<std::size_t>& boundaries,
                                     LookupMode /*mode*/, std::uint64_t window_start_ms,
                                     std::uint64_t window_end_ms) {
    return run_gpu(view, catalog, params, boundaries, window_start_ms, window_end_ms);
}

} // namespace flowmon

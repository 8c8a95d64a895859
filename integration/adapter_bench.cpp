// adapter_bench -- end-to-end throughput of the drop-in: the reference's own
// call, flowmon::aggregate(std::span<const FlowRecord>, SiteCatalog, ...),
// served by the GPU adapter (integration/flowmon_gpu.cpp) from a PAGEABLE
// std::vector<FlowRecord>, returning the full AnalysisResult (sites, hosts
// and every RateHistogram) -- what monitor.cpp:118 (run_cycle) gets.
//
//   adapter_bench [--workload D3] [--records N] [--steps K] [--warmup W]
//
// The records are the bench's synthetic workload (workloads/synth.c, the
// same generator and seeds as bench.py), the catalog is the workload's
// sites registered in order. Prints one JSON line.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "flowmon/rate_engine.hpp"
#include "flowmon/site_catalog.hpp"

extern "C" {
struct gnm_synth_spec {
    std::uint64_t seed, n, index_offset;
    std::uint32_t n_sites;
    const std::uint32_t* site_base;
    const std::uint32_t* site_size;
    double zipf_s;
    std::uint32_t hosts_per_site;
    double frac_ack, frac_admin, frac_fwd;
    double mu, sigma;
    std::uint64_t window_start_ms, window_ms;
};
int gnm_synth_generate(const gnm_synth_spec* sp, std::uint32_t* src, std::uint32_t* dst, std::uint32_t* pkts,
                       std::uint32_t* octets, std::uint64_t* start, std::uint64_t* end);
void gnm_synth_to_aos(std::uint64_t n, const std::uint32_t* src, const std::uint32_t* dst, const std::uint32_t* pkts,
                      const std::uint32_t* octets, const std::uint64_t* start, const std::uint64_t* end, void* out);
}

using namespace flowmon;
using Clock = std::chrono::steady_clock;

int main(int argc, char** argv) {
    std::string workload = "D3";
    std::uint64_t n = 0;
    int steps = 5, warmup = 2;
    for (int i = 1; i + 1 < argc; i += 2) {
        const std::string k = argv[i], v = argv[i + 1];
        if (k == "--workload") workload = v;
        else if (k == "--records") n = std::stoull(v);
        else if (k == "--steps") steps = std::stoi(v);
        else if (k == "--warmup") warmup = std::stoi(v);
    }
    // workloads/__init__.py: D1 (seed 1, 256 /24 sites, uniform), D3 (seed 3,
    // 10k /24 sites, Zipf 1, one-hour window).
    std::uint32_t n_sites;
    gnm_synth_spec sp{};
    if (workload == "D1") {
        n_sites = 256, sp.seed = 1, sp.zipf_s = 0.0, sp.window_ms = 60'000;
        if (!n) n = 100'000;
    } else if (workload == "D3") {
        n_sites = 10'000, sp.seed = 3, sp.zipf_s = 1.0, sp.window_ms = 3'600'000;
        if (!n) n = 100'000'000;
    } else {
        std::fprintf(stderr, "workload D1 or D3\n");
        return 2;
    }
    std::vector<std::uint32_t> base(n_sites), size(n_sites, 256);
    SiteCatalog catalog;
    for (std::uint32_t i = 0; i < n_sites; ++i) {
        base[i] = (10u << 24) + (i << 8);
        const std::string cidr = std::to_string(base[i] >> 24) + "." + std::to_string(base[i] >> 16 & 255) + "." +
                                 std::to_string(base[i] >> 8 & 255) + ".0/24";
        catalog.register_site("site" + std::to_string(i), std::vector<std::string>{cidr});
    }
    sp.n = n;
    sp.n_sites = n_sites;
    sp.site_base = base.data();
    sp.site_size = size.data();
    sp.hosts_per_site = 8;
    sp.frac_ack = 0.30, sp.frac_admin = 0.20, sp.frac_fwd = 0.40;
    sp.mu = 14.5, sp.sigma = 1.5;
    sp.window_start_ms = 1'600'000'000'000ull;
    std::vector<FlowRecord> records(n);
    {
        std::vector<std::uint32_t> src(n), dst(n), pkts(n), oct(n);
        std::vector<std::uint64_t> start(n), end(n);
        if (gnm_synth_generate(&sp, src.data(), dst.data(), pkts.data(), oct.data(), start.data(), end.data())) {
            std::fprintf(stderr, "generator failed\n");
            return 1;
        }
        gnm_synth_to_aos(n, src.data(), dst.data(), pkts.data(), oct.data(), start.data(), end.data(),
                         records.data());
    }
    const std::span<const FlowRecord> view(records);
    AnalysisResult res;
    for (int i = 0; i < warmup; ++i) res = aggregate(view, catalog, FilterParams{}, 1);
    std::vector<double> ms;
    for (int i = 0; i < steps; ++i) {
        const auto t0 = Clock::now();
        res = aggregate(view, catalog, FilterParams{}, 1);
        ms.push_back(std::chrono::duration<double, std::milli>(Clock::now() - t0).count());
    }
    std::sort(ms.begin(), ms.end());
    double sum = 0;
    for (double x : ms) sum += x;
    std::uint64_t hosts = 0;
    for (const auto& [id, sr] : res.sites) hosts += sr.hosts.size();
    std::printf("{\"workload\": \"%s\", \"records\": %lu, \"steps\": %d, \"ms_per_step\": %.3f, \"ms_min\": %.3f, "
                "\"records_per_s\": %.1f, \"sites\": %zu, \"host_rows\": %lu, \"forward\": %lu, "
                "\"source\": \"flowmon::aggregate (GPU adapter) from a pageable std::vector<FlowRecord>, full "
                "AnalysisResult incl. hosts and histograms\"}\n",
                workload.c_str(), n, steps, sum / ms.size(), ms.front(), n / (sum / ms.size() / 1e3),
                res.sites.size(), hosts, res.tallies.forward);
    return 0;
}

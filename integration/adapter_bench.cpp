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

#include "workload_gen.hpp"

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
    std::vector<FlowRecord> records;
    SiteCatalog catalog;
    if (!gnm_workload::make(workload, n, records, catalog)) {
        std::fprintf(stderr, "workload D1 or D3\n");
        return 2;
    }
    n = records.size();
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

// adapter_parity -- TEST INFRASTRUCTURE: judges the drop-in adapter
// (flowmon::aggregate on the GPU, integration/flowmon_gpu.cpp) against the
// unmodified reference CPU path (flowmon::cpu_aggregate: rate_engine.cpp
// compiled with the aggregate -> cpu_aggregate rename) with the reference's
// own AnalysisResult::operator== (rate_engine.hpp:112-119): tallies, every
// site's RateStats and RateHistogram, every host's RateStats and
// RateHistogram, bit for bit.
//
//   adapter_parity RECORDS CATALOG [--workers W] [--cpu-workers W] [--partitions K]
//                  [--params ACK,PKTS,DUR] [--window S,E] [--repeat R] [--seed S]
//   adapter_parity --workload D1|D3 [--records N] [options]
//
// RECORDS: raw 64-byte FlowRecord rows; CATALOG: SiteCatalog::load text; or
// a bench workload generated in process (workload_gen.hpp).
// Prints one JSON line; exit status 0 iff every comparison held.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "flowmon/rate_engine.hpp"
#include "flowmon/site_catalog.hpp"
#include "workload_gen.hpp"

namespace flowmon {
// the reference's own aggregate, renamed at compile time (integration/Makefile)
AnalysisResult cpu_aggregate(std::span<const FlowRecord> view, const SiteCatalog& catalog,
                             const FilterParams& params, unsigned workers, LookupMode mode,
                             std::uint64_t window_start_ms, std::uint64_t window_end_ms);
AnalysisResult cpu_aggregate_partitioned(std::span<const FlowRecord> view, const SiteCatalog& catalog,
                                         const FilterParams& params,
                                         const std::vector<std::size_t>& boundaries, LookupMode mode,
                                         std::uint64_t window_start_ms, std::uint64_t window_end_ms);
} // namespace flowmon

using namespace flowmon;
using Clock = std::chrono::steady_clock;

namespace {

double ms_since(Clock::time_point t0) {
    return std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
}

// First difference between two results, for the failure message.
std::string first_diff(const AnalysisResult& a, const AnalysisResult& b) {
    std::ostringstream o;
    if (!(a.tallies == b.tallies)) return "tallies differ";
    if (a.window_start_ms != b.window_start_ms || a.window_end_ms != b.window_end_ms) return "window differs";
    if (a.sites.size() != b.sites.size())
        return "site count " + std::to_string(a.sites.size()) + " vs " + std::to_string(b.sites.size());
    for (auto ia = a.sites.begin(), ib = b.sites.begin(); ia != a.sites.end(); ++ia, ++ib) {
        if (ia->first != ib->first) return "site ids differ at " + std::to_string(ia->first);
        const SiteResult &x = ia->second, &y = ib->second;
        o << "site " << ia->first << ": ";
        if (!(x.stats == y.stats)) {
            o.precision(17);
            o << "stats (count " << x.stats.flow_count << "/" << y.stats.flow_count << ", min " << x.stats.min_bps
              << "/" << y.stats.min_bps << ", max " << x.stats.max_bps << "/" << y.stats.max_bps << ", avg "
              << x.stats.avg_bps << "/" << y.stats.avg_bps << ", median " << x.stats.median_bps << "/"
              << y.stats.median_bps << ")";
            return o.str();
        }
        if (!(x.histogram == y.histogram)) {
            o << "histogram (sum " << x.histogram.sum_bps() << "/" << y.histogram.sum_bps() << ")";
            return o.str();
        }
        if (x.hosts.size() != y.hosts.size()) {
            o << "host count " << x.hosts.size() << "/" << y.hosts.size();
            return o.str();
        }
        for (auto ha = x.hosts.begin(), hb = y.hosts.begin(); ha != x.hosts.end(); ++ha, ++hb) {
            if (ha->first != hb->first || !(ha->second == hb->second)) {
                o << "host " << format_ipv4(ha->first) << " / " << format_ipv4(hb->first);
                return o.str();
            }
        }
        o.str("");
    }
    return "";
}

} // namespace

int main(int argc, char** argv) {
    if (argc < 3) {
        std::fprintf(stderr, "usage: %s RECORDS CATALOG [options]\n", argv[0]);
        return 2;
    }
    unsigned workers = 1, cpu_workers = 1;
    std::uint64_t gen_records = 0;
    int partitions = 0, repeat = 1;
    std::uint64_t ws = 0, we = 0, seed = 1;
    FilterParams params;
    for (int i = 3; i + 1 < argc; i += 2) {
        const std::string k = argv[i], v = argv[i + 1];
        if (k == "--workers") workers = std::stoul(v);
        else if (k == "--cpu-workers") cpu_workers = std::stoul(v);
        else if (k == "--partitions") partitions = std::stoi(v);
        else if (k == "--repeat") repeat = std::max(1, std::stoi(v));
        else if (k == "--seed") seed = std::stoull(v);
        else if (k == "--records") gen_records = std::stoull(v);
        else if (k == "--window") std::sscanf(v.c_str(), "%lu,%lu", &ws, &we);
        else if (k == "--params")
            std::sscanf(v.c_str(), "%u,%u,%u", &params.ack_avg_size_max, &params.min_packets,
                        &params.min_duration_ms);
        else {
            std::fprintf(stderr, "unknown option %s\n", k.c_str());
            return 2;
        }
    }

    std::vector<FlowRecord> records;
    SiteCatalog catalog;
    if (std::string(argv[1]) == "--workload") {
        if (!gnm_workload::make(argv[2], gen_records, records, catalog)) {
            std::fprintf(stderr, "unknown workload %s\n", argv[2]);
            return 2;
        }
    } else {
        std::ifstream f(argv[1], std::ios::binary | std::ios::ate);
        if (!f) {
            std::fprintf(stderr, "cannot open %s\n", argv[1]);
            return 2;
        }
        const std::size_t bytes = static_cast<std::size_t>(f.tellg());
        records.resize(bytes / sizeof(FlowRecord));
        f.seekg(0);
        f.read(reinterpret_cast<char*>(records.data()),
               static_cast<std::streamsize>(records.size() * sizeof(FlowRecord)));
        catalog = SiteCatalog::load_file(argv[2]);
    }
    const std::span<const FlowRecord> view(records);

    // GPU through the adapter: the first call builds and uploads the registry;
    // the timed ones are the steady state a monitor loop sees.
    std::vector<double> gpu_ms;
    AnalysisResult gpu;
    for (int r = 0; r < repeat; ++r) {
        const auto t0 = Clock::now();
        gpu = aggregate(view, catalog, params, workers, LookupMode::Hash, ws, we);
        gpu_ms.push_back(ms_since(t0));
    }
    auto t0 = Clock::now();
    const AnalysisResult cpu = cpu_aggregate(view, catalog, params, cpu_workers, LookupMode::Hash, ws, we);
    const double cpu_ms = ms_since(t0);

    bool ok = gpu == cpu;
    std::string diff = ok ? "" : first_diff(gpu, cpu);

    // aggregate_partitioned over random sorted boundaries (engine_test.cpp:282-305)
    int part_ok = 0;
    std::mt19937_64 rng(seed);
    for (int t = 0; t < partitions; ++t) {
        std::vector<std::size_t> b;
        const std::size_t cuts = rng() % 7 + 1;
        for (std::size_t i = 0; i < cuts; ++i) b.push_back(rng() % (records.size() + 1));
        std::sort(b.begin(), b.end());
        const AnalysisResult g = aggregate_partitioned(view, catalog, params, b, LookupMode::Hash, ws, we);
        if (g == cpu) ++part_ok;
        else if (diff.empty()) diff = "partitioned: " + first_diff(g, cpu);
    }
    ok = ok && part_ok == partitions;

    std::uint64_t hosts = 0;
    for (const auto& [id, sr] : cpu.sites) hosts += sr.hosts.size();
    std::sort(gpu_ms.begin(), gpu_ms.end());
    std::printf("{\"equal\": %s, \"records\": %zu, \"sites\": %zu, \"host_rows\": %lu, \"forward\": %lu, "
                "\"pure_ack\": %lu, \"administrative\": %lu, \"unmatched\": %lu, \"partitions_equal\": %d, "
                "\"partitions\": %d, \"gpu_ms_min\": %.3f, \"gpu_ms_median\": %.3f, \"cpu_ms\": %.3f, "
                "\"cpu_workers\": %u, \"diff\": \"%s\"}\n",
                ok ? "true" : "false", records.size(), cpu.sites.size(), hosts, cpu.tallies.forward,
                cpu.tallies.pure_ack, cpu.tallies.administrative, cpu.tallies.unmatched, part_ok, partitions,
                gpu_ms.front(), gpu_ms[gpu_ms.size() / 2], cpu_ms, cpu_workers, diff.c_str());
    return ok ? 0 : 1;
}

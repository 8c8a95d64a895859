// workload_gen.hpp -- TEST/BENCH INFRASTRUCTURE: the bench's synthetic
// workloads (workloads/synth.c, the same generator and seeds as bench.py and
// the Python tests) as a std::vector<FlowRecord> plus the matching
// SiteCatalog, for the C++ drivers (adapter_bench, adapter_parity).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "flowmon/netflow.hpp"
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

namespace gnm_workload {

// workloads/__init__.py: D1 (seed 1, 256 /24 sites, uniform), D3 (seed 3,
// 10k /24 sites, Zipf 1, one-hour window). n = 0: the workload's own size.
// Returns false for an unknown workload.
inline bool make(const std::string& name, std::uint64_t n, std::vector<flowmon::FlowRecord>& records,
                 flowmon::SiteCatalog& catalog) {
    std::uint32_t n_sites;
    gnm_synth_spec sp{};
    if (name == "D1") {
        n_sites = 256, sp.seed = 1, sp.zipf_s = 0.0, sp.window_ms = 60'000;
        if (!n) n = 100'000;
    } else if (name == "D3") {
        n_sites = 10'000, sp.seed = 3, sp.zipf_s = 1.0, sp.window_ms = 3'600'000;
        if (!n) n = 100'000'000;
    } else {
        return false;
    }
    std::vector<std::uint32_t> base(n_sites), size(n_sites, 256);
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
    records.resize(n);
    std::vector<std::uint32_t> src(n), dst(n), pkts(n), oct(n);
    std::vector<std::uint64_t> start(n), end(n);
    if (gnm_synth_generate(&sp, src.data(), dst.data(), pkts.data(), oct.data(), start.data(), end.data()))
        return false;
    gnm_synth_to_aos(n, src.data(), dst.data(), pkts.data(), oct.data(), start.data(), end.data(), records.data());
    return true;
}

} // namespace gnm_workload

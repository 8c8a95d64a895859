// ref_driver.cpp — extern "C" shim around the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY (see oracle/gnm_oracle.c header). Built by
// oracle/Makefile together with the reference's own sources, compiled in
// place from /root/reference/proj/core/src (never copied), into
// oracle/_ref/libflowmon_ref.so. Used to (1) validate the C restatement,
// (2) generate the golden vectors under tests/golden/, and (3) time the
// reference CPU path for bench.py's cpu_baseline and --impl reference arm.
//
// Nothing here re-implements the hot path: every computation is a call into
// flowmon:: (rate_engine.cpp, site_catalog.cpp, monitor.cpp, toolkit.cpp).
#include <chrono>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "flowmon/flow_store.hpp"
#include "flowmon/monitor.hpp"
#include "flowmon/netflow.hpp"
#include "flowmon/rate_engine.hpp"
#include "flowmon/site_catalog.hpp"
#include "flowmon/toolkit.hpp"

using namespace flowmon;

namespace {
thread_local std::string g_err;

void set_err(const std::exception& e) { g_err = e.what(); }

FilterParams make_params(uint32_t ack, uint32_t minp, uint32_t mind, uint32_t workers) {
    FilterParams p;
    p.ack_avg_size_max = ack;
    p.min_packets = minp;
    p.min_duration_ms = mind;
    p.workers = workers;
    return p;
}

FlowRecord make_record(uint32_t src, uint32_t dst, uint32_t pkts, uint32_t octets, uint64_t start,
                       uint64_t end) {
    FlowRecord r;
    r.raw.src_addr = src;
    r.raw.dst_addr = dst;
    r.raw.d_pkts = pkts;
    r.raw.d_octets = octets;
    r.raw.first = static_cast<uint32_t>(start);
    r.raw.last = static_cast<uint32_t>(end);
    r.start_ms = start;
    r.end_ms = end;
    return r;
}
} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
size_t ref_flow_record_size() { return sizeof(FlowRecord); }

// ---- SiteCatalog --------------------------------------------------------
void* ref_catalog_create() { return new SiteCatalog(); }
void ref_catalog_destroy(void* c) { delete static_cast<SiteCatalog*>(c); }

// cidrs: comma-separated CIDR text. Returns the SiteId, -1 on Overlap,
// -2 on InvalidCidr.
long long ref_catalog_register(void* c, const char* name, const char* cidrs) {
    auto* cat = static_cast<SiteCatalog*>(c);
    std::vector<std::string> list;
    std::string s(cidrs), item;
    size_t pos = 0;
    while (pos <= s.size()) {
        size_t comma = s.find(',', pos);
        if (comma == std::string::npos) comma = s.size();
        item = s.substr(pos, comma - pos);
        if (!item.empty()) list.push_back(item);
        pos = comma + 1;
    }
    try {
        return cat->register_site(name, list);
    } catch (const CatalogError& e) {
        set_err(e);
        return e.kind() == CatalogError::Kind::Overlap ? -1 : -2;
    }
}

// Register one site from a (addr, prefix_len) pair list (Cidr{base,len}
// as catalog_test.cpp:93-105 does).
long long ref_catalog_register_raw(void* c, const char* name, const uint32_t* addr,
                                   const int32_t* len, size_t n) {
    auto* cat = static_cast<SiteCatalog*>(c);
    std::vector<Cidr> list;
    for (size_t i = 0; i < n; ++i) list.push_back(Cidr{addr[i], len[i]});
    try {
        return cat->register_site(name, list);
    } catch (const CatalogError& e) {
        set_err(e);
        return e.kind() == CatalogError::Kind::Overlap ? -1 : -2;
    }
}

int ref_cidr_parse(const char* text, uint32_t* addr, int32_t* len) {
    try {
        Cidr c = Cidr::parse(text);
        *addr = c.addr;
        *len = c.prefix_len;
        return 0;
    } catch (const CatalogError& e) {
        set_err(e);
        return -2;
    }
}

uint32_t ref_catalog_lookup(const void* c, uint32_t ip) {
    auto s = static_cast<const SiteCatalog*>(c)->lookup(ip);
    return s ? *s : 0xFFFFFFFFu;
}
uint32_t ref_catalog_sequential_lookup(const void* c, uint32_t ip) {
    auto s = static_cast<const SiteCatalog*>(c)->sequential_lookup(ip);
    return s ? *s : 0xFFFFFFFFu;
}
size_t ref_catalog_entry_count(const void* c) {
    return static_cast<const SiteCatalog*>(c)->entry_count();
}
size_t ref_catalog_site_count(const void* c) {
    return static_cast<const SiteCatalog*>(c)->site_count();
}
size_t ref_catalog_entries(const void* c, uint32_t* prefix, uint32_t* site, size_t cap) {
    const auto& e = static_cast<const SiteCatalog*>(c)->entries();
    size_t n = e.size() < cap ? e.size() : cap;
    for (size_t i = 0; i < n; ++i) {
        prefix[i] = e[i].first;
        site[i] = e[i].second;
    }
    return e.size();
}

// ---- records --------------------------------------------------------------
void* ref_records_create(const uint32_t* src, const uint32_t* dst, const uint32_t* pkts,
                         const uint32_t* octets, const uint64_t* start, const uint64_t* end,
                         size_t n) {
    auto* v = new std::vector<FlowRecord>(n);
    for (size_t i = 0; i < n; ++i) (*v)[i] = make_record(src[i], dst[i], pkts[i], octets[i], start[i], end[i]);
    return v;
}
void ref_records_destroy(void* r) { delete static_cast<std::vector<FlowRecord>*>(r); }
size_t ref_records_size(const void* r) { return static_cast<const std::vector<FlowRecord>*>(r)->size(); }
// Raw 64-byte AoS bytes of the records (the FlowRecord layout).
const void* ref_records_data(const void* r) {
    return static_cast<const std::vector<FlowRecord>*>(r)->data();
}

// toolkit::generate for a scenario described by (cidr, hosts, fixed rate or
// lognormal, flows/hour, ack, admin) per site; acceptance.cpp:367-392 and
// cmd_bench (flowmon.cpp:297-332) build exactly such specs.
void* ref_generate(uint32_t duration_hours, uint64_t base_wall_ms, uint64_t seed, size_t n_sites,
                   const char* const* cidrs, const uint32_t* hosts, const int32_t* lognormal,
                   const double* fixed_bps, const double* mu, const double* sigma,
                   const uint32_t* flows_per_hour, const double* ack, const double* admin) {
    ScenarioSpec spec;
    spec.duration_hours = duration_hours;
    spec.base_wall_ms = base_wall_ms;
    spec.seed = seed;
    for (size_t i = 0; i < n_sites; ++i) {
        SiteSpec s;
        s.name = "site" + std::to_string(i);
        s.cidr = cidrs[i];
        s.host_count = hosts[i];
        if (lognormal[i]) {
            s.rate.kind = RateDistribution::Kind::Lognormal;
            s.rate.lognormal_mu = mu[i];
            s.rate.lognormal_sigma = sigma[i];
        } else {
            s.rate.kind = RateDistribution::Kind::Fixed;
            s.rate.fixed_bps = fixed_bps[i];
        }
        s.flows_per_hour = flows_per_hour[i];
        s.ack_fraction = ack[i];
        s.admin_fraction = admin[i];
        spec.sites.push_back(s);
    }
    try {
        return new std::vector<FlowRecord>(generate(spec));
    } catch (const std::exception& e) {
        set_err(e);
        return nullptr;
    }
}
// Column export of a record vector.
void ref_records_columns(const void* r, uint32_t* src, uint32_t* dst, uint32_t* pkts,
                         uint32_t* octets, uint64_t* start, uint64_t* end) {
    const auto& v = *static_cast<const std::vector<FlowRecord>*>(r);
    for (size_t i = 0; i < v.size(); ++i) {
        src[i] = v[i].raw.src_addr;
        dst[i] = v[i].raw.dst_addr;
        pkts[i] = v[i].raw.d_pkts;
        octets[i] = v[i].raw.d_octets;
        start[i] = v[i].start_ms;
        end[i] = v[i].end_ms;
    }
}

// ---- scalar functions (rate_engine.hpp:121-138) ----------------------------
int ref_classify(uint32_t src, uint32_t dst, uint32_t pkts, uint32_t octets, uint64_t start,
                 uint64_t end, uint32_t ack, uint32_t minp, uint32_t mind, const void* c, int seq) {
    return static_cast<int>(classify(make_record(src, dst, pkts, octets, start, end),
                                     make_params(ack, minp, mind, 1),
                                     *static_cast<const SiteCatalog*>(c),
                                     seq ? LookupMode::Sequential : LookupMode::Hash));
}
// Returns 0 on success, -1 on RateError (ZeroDuration).
int ref_flow_rate(uint32_t octets, uint64_t start, uint64_t end, double* rate, uint64_t* ubps_lo,
                  uint64_t* ubps_hi) {
    try {
        const FlowRecord r = make_record(0, 0, 1, octets, start, end);
        *rate = flow_rate(r);
        const unsigned __int128 u = flow_rate_ubps(r);
        *ubps_lo = static_cast<uint64_t>(u);
        *ubps_hi = static_cast<uint64_t>(u >> 64);
        return 0;
    } catch (const RateError& e) {
        set_err(e);
        return -1;
    }
}
size_t ref_bucket_index(double rate) { return bucket_index(rate); }
// attribute: returns site or ~0, host via *host.
uint32_t ref_attribute(uint32_t src, uint32_t dst, const void* c, int seq, uint32_t* host) {
    auto a = attribute(make_record(src, dst, 1, 1, 0, 1), *static_cast<const SiteCatalog*>(c),
                       seq ? LookupMode::Sequential : LookupMode::Hash);
    if (!a) return 0xFFFFFFFFu;
    *host = a->second;
    return a->first;
}

// ---- RateHistogram --------------------------------------------------------
void* ref_hist_create() { return new RateHistogram(); }
void ref_hist_destroy(void* h) { delete static_cast<RateHistogram*>(h); }
void ref_hist_add(void* h, double rate, uint64_t ubps_lo, uint64_t ubps_hi) {
    static_cast<RateHistogram*>(h)->add(
        rate, static_cast<unsigned __int128>(ubps_hi) << 64 | ubps_lo);
}
// 0 ok, -1 when EmptyHistogram was thrown.
int ref_hist_median(const void* h, double* out) {
    try {
        *out = static_cast<const RateHistogram*>(h)->median_bps();
        return 0;
    } catch (const RateError& e) {
        set_err(e);
        return -1;
    }
}

// ---- aggregate ------------------------------------------------------------
void* ref_aggregate(const void* records, const void* c, uint32_t ack, uint32_t minp, uint32_t mind,
                    uint32_t workers, int seq, uint64_t ws, uint64_t we, double* elapsed_ms) {
    const auto& v = *static_cast<const std::vector<FlowRecord>*>(records);
    const auto t0 = std::chrono::steady_clock::now();
    auto* res = new AnalysisResult(aggregate(v, *static_cast<const SiteCatalog*>(c),
                                             make_params(ack, minp, mind, workers), workers,
                                             seq ? LookupMode::Sequential : LookupMode::Hash, ws, we));
    if (elapsed_ms)
        *elapsed_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    return res;
}
// Same over a [begin, end) record sub-range (for chunked timing samples).
double ref_aggregate_time_range(const void* records, size_t begin, size_t end, const void* c,
                                uint32_t workers) {
    const auto& v = *static_cast<const std::vector<FlowRecord>*>(records);
    std::span<const FlowRecord> view(v.data() + begin, end - begin);
    const auto t0 = std::chrono::steady_clock::now();
    AnalysisResult res = aggregate(view, *static_cast<const SiteCatalog*>(c), FilterParams{}, workers,
                                   LookupMode::Hash);
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    volatile size_t sink = res.sites.size();
    (void)sink;
    return ms;
}
void* ref_aggregate_partitioned(const void* records, const void* c, uint32_t ack, uint32_t minp,
                                uint32_t mind, const size_t* boundaries, size_t nb) {
    const auto& v = *static_cast<const std::vector<FlowRecord>*>(records);
    std::vector<size_t> b(boundaries, boundaries + nb);
    return new AnalysisResult(aggregate_partitioned(v, *static_cast<const SiteCatalog*>(c),
                                                    make_params(ack, minp, mind, 1), b));
}
void ref_result_destroy(void* r) { delete static_cast<AnalysisResult*>(r); }
int ref_result_equal(const void* a, const void* b) {
    return *static_cast<const AnalysisResult*>(a) == *static_cast<const AnalysisResult*>(b);
}
void ref_result_tallies(const void* r, uint64_t* t) {
    const auto& tl = static_cast<const AnalysisResult*>(r)->tallies;
    t[0] = tl.forward;
    t[1] = tl.pure_ack;
    t[2] = tl.administrative;
    t[3] = tl.unmatched;
}
size_t ref_result_site_ids(const void* r, uint32_t* ids, size_t cap) {
    const auto& s = static_cast<const AnalysisResult*>(r)->sites;
    size_t i = 0;
    for (const auto& [id, sr] : s) {
        if (i < cap) ids[i] = id;
        ++i;
    }
    return s.size();
}

namespace {
// The exact u128 micro-bps accumulator is private to RateHistogram; its
// public view is sum_bps() = double(sum)/1e6 (rate_engine.hpp:62). The exact
// integer sum is rebuilt by ref_site_sums below.
void export_hist(const RateHistogram& h, const RateStats& st, uint64_t* count, double* stats4,
                 double* sum_bps, uint32_t* buckets) {
    *count = st.flow_count;
    stats4[0] = st.min_bps;
    stats4[1] = st.max_bps;
    stats4[2] = st.avg_bps;
    stats4[3] = st.median_bps;
    *sum_bps = h.sum_bps();
    if (buckets) {
        for (size_t k = 0; k < kBucketCount; ++k) buckets[k] = static_cast<uint32_t>(h.bucket(k));
    }
}
} // namespace

// Per-site stats: count, {min,max,avg,median}, sum_bps, histogram (10001
// u32, optional). Returns 0 when present.
int ref_result_site(const void* r, uint32_t site, uint64_t* count, double* stats4, double* sum_bps,
                    uint32_t* buckets, uint64_t* n_hosts) {
    const auto& s = static_cast<const AnalysisResult*>(r)->sites;
    auto it = s.find(site);
    if (it == s.end()) return -1;
    export_hist(it->second.histogram, it->second.stats, count, stats4, sum_bps, buckets);
    *n_hosts = it->second.hosts.size();
    return 0;
}
size_t ref_result_hosts(const void* r, uint32_t site, uint32_t* ips, size_t cap) {
    const auto& s = static_cast<const AnalysisResult*>(r)->sites;
    auto it = s.find(site);
    if (it == s.end()) return 0;
    size_t i = 0;
    for (const auto& [ip, hr] : it->second.hosts) {
        if (i < cap) ips[i] = ip;
        ++i;
    }
    return it->second.hosts.size();
}
int ref_result_host(const void* r, uint32_t site, uint32_t ip, uint64_t* count, double* stats4,
                    double* sum_bps, uint32_t* buckets) {
    const auto& s = static_cast<const AnalysisResult*>(r)->sites;
    auto it = s.find(site);
    if (it == s.end()) return -1;
    auto h = it->second.hosts.find(ip);
    if (h == it->second.hosts.end()) return -1;
    export_hist(h->second.histogram, h->second.stats, count, stats4, sum_bps, buckets);
    return 0;
}

// Exact u128 micro-bps sum of a site: rebuilt from the reference's own
// per-flow function flow_rate_ubps (rate_engine.cpp:111-117) over the
// Forward flows attributed to the site (the reference's accumulator is
// private). Also the per-site byte sum (north-star extension, unpinned by
// reference tests): d_octets over Forward flows (classify + attribute).
void ref_site_sums(const void* records, const void* c, uint32_t ack, uint32_t minp, uint32_t mind,
                   uint32_t n_sites, uint64_t* ubps_lo, uint64_t* ubps_hi, uint64_t* octets) {
    const auto& v = *static_cast<const std::vector<FlowRecord>*>(records);
    const auto& cat = *static_cast<const SiteCatalog*>(c);
    const FilterParams p = make_params(ack, minp, mind, 1);
    std::vector<unsigned __int128> sums(n_sites, 0);
    for (uint32_t s = 0; s < n_sites; ++s) octets[s] = 0;
    for (const FlowRecord& r : v) {
        if (classify(r, p, cat) != FlowClass::Forward) continue;
        const auto a = attribute(r, cat);
        if (a->first >= n_sites) continue;
        sums[a->first] += flow_rate_ubps(r);
        octets[a->first] += r.raw.d_octets;
    }
    for (uint32_t s = 0; s < n_sites; ++s) {
        ubps_lo[s] = static_cast<uint64_t>(sums[s]);
        ubps_hi[s] = static_cast<uint64_t>(sums[s] >> 64);
    }
}

// ---- monitor --------------------------------------------------------------
void* ref_wstate_create() { return new WarningState(); }
void ref_wstate_destroy(void* w) { delete static_cast<WarningState*>(w); }
uint32_t ref_wstate_streak(const void* w, uint32_t site) {
    return static_cast<const WarningState*>(w)->streak(site);
}
size_t ref_evaluate_warnings(const void* r, const void* c, void* w, double threshold,
                             uint32_t* sites, uint32_t* hours, double* medians, size_t cap) {
    auto warns = evaluate_warnings(*static_cast<const AnalysisResult*>(r),
                                   *static_cast<const SiteCatalog*>(c),
                                   *static_cast<WarningState*>(w), threshold);
    for (size_t i = 0; i < warns.size() && i < cap; ++i) {
        sites[i] = warns[i].site;
        hours[i] = warns[i].consecutive_bad_hours;
        medians[i] = warns[i].median_bps;
    }
    return warns.size();
}


// ---- NetFlow v5 ingest (collector.cpp:101-129, netflow.cpp:78-161) ------------
// Collector::ingest_datagram without the store and the sequence tracker:
// decode_packet, the collector's reject rule (d_pkts == 0 || d_octets <
// d_pkts), resolve_times. Returns 0, or 1 + CodecError::Kind (BadVersion,
// Truncated, BadCount) when the datagram is dropped; `out` receives up to 30
// FlowRecords (64 bytes each) in order.
int ref_ingest_datagram(const uint8_t* d, size_t len, void* out, size_t* n_out, uint32_t* rejected) {
    *n_out = 0;
    *rejected = 0;
    DecodedPacket packet;
    try {
        packet = decode_packet(std::span<const std::uint8_t>(d, len));
    } catch (const CodecError& e) {
        return 1 + static_cast<int>(e.kind());
    }
    auto* o = static_cast<FlowRecord*>(out);
    for (const RawFlowRecord& raw : packet.records) {
        if (raw.d_pkts == 0 || raw.d_octets < raw.d_pkts) {
            ++*rejected;
            continue;
        }
        o[(*n_out)++] = resolve_times(packet.header, raw);
    }
    return 0;
}

// The collector's decode loop over a batch of datagrams (Collector::
// ingest_datagram minus the socket and the store, collector.cpp:101-129),
// timed in C: datagram i is bytes [off[i], off[i+1]). Returns the accepted
// record count; *ms = wall time of the loop.
size_t ref_ingest_batch(const uint8_t* buf, const uint64_t* off, size_t n, void* out, double* ms) {
    auto* o = static_cast<FlowRecord*>(out);
    size_t k = 0;
    const auto t0 = std::chrono::steady_clock::now();
    for (size_t i = 0; i < n; ++i) {
        DecodedPacket packet;
        try {
            packet = decode_packet(std::span<const std::uint8_t>(buf + off[i], off[i + 1] - off[i]));
        } catch (const CodecError&) {
            continue;
        }
        for (const RawFlowRecord& raw : packet.records) {
            if (raw.d_pkts == 0 || raw.d_octets < raw.d_pkts) continue;
            o[k++] = resolve_times(packet.header, raw);
        }
    }
    *ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    return k;
}

// encode_packet (netflow.cpp:115-143): h = {version, count, sys_uptime,
// unix_secs, unix_nsecs, flow_sequence, engine_type, engine_id,
// sampling_interval}; `raw` holds `n` RawFlowRecords (48-byte struct).
// Returns the datagram length written to `out`, or 0 on CodecError.
size_t ref_encode_packet(const uint32_t* h, const void* raw, size_t n, uint8_t* out) {
    ExportHeader header;
    header.version = static_cast<std::uint16_t>(h[0]);
    header.count = static_cast<std::uint16_t>(h[1]);
    header.sys_uptime = h[2];
    header.unix_secs = h[3];
    header.unix_nsecs = h[4];
    header.flow_sequence = h[5];
    header.engine_type = static_cast<std::uint8_t>(h[6]);
    header.engine_id = static_cast<std::uint8_t>(h[7]);
    header.sampling_interval = static_cast<std::uint16_t>(h[8]);
    try {
        const auto buf = encode_packet(
            header, std::span<const RawFlowRecord>(static_cast<const RawFlowRecord*>(raw), n));
        std::memcpy(out, buf.data(), buf.size());
        return buf.size();
    } catch (const CodecError& e) {
        set_err(e);
        return 0;
    }
}
size_t ref_raw_record_size() { return sizeof(RawFlowRecord); }

// ---- FLOWARC1 archives (flow_store.cpp:144-207) ------------------------------
// FlowStore::write_archive of a records handle (ref_records_create /
// ref_generate); 0 or -1 (ref_last_error).
int ref_archive_write(const void* records, const char* path) {
    try {
        const auto* v = static_cast<const std::vector<FlowRecord>*>(records);
        FlowStore::write_archive(path, *v);
        return 0;
    } catch (const std::exception& e) {
        set_err(e);
        return -1;
    }
}
// FlowStore::load -> a records handle, or null with *kind = ArchiveError::Kind.
void* ref_archive_load(const char* path, int* kind) {
    *kind = -1;
    try {
        return new std::vector<FlowRecord>(FlowStore::load(path));
    } catch (const ArchiveError& e) {
        set_err(e);
        *kind = static_cast<int>(e.kind());
        return nullptr;
    }
}
} // extern "C"

#!/usr/bin/env python3
"""Generate the golden fixtures in tests/golden/ from the UNMODIFIED
reference (oracle/_ref/libflowmon_ref.so, compiled in place from
/root/reference/proj/core/src by `make -C oracle ref`).

    python tests/golden/make_golden.py

Each fixture is an .npz holding the inputs (SoA columns, the catalog as CIDR
text, FilterParams) and the reference's outputs:
  * tallies                      AnalysisResult::tallies
  * per site: count, min, max, avg, median (RateStats, rate_engine.cpp:242-253),
    histogram (sparse: site, bucket, count)
  * exact u128 micro-bps sums and byte sums (rebuilt from flow_rate_ubps /
    classify / attribute, ref_driver.cpp ref_site_sums)
  * per-record class/site (classify + attribute, gnm_classify encoding)
plus fixtures for the catalog (lookups), the scalar known answers and the
warning scenarios of acceptance.cpp criterion 7.

The fixtures are the parity anchor on the GPU box, where /root/reference
does not exist.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

from oracle import Reference  # noqa: E402
import parity  # noqa: E402
from paper_1108_1785_b200 import synth  # noqa: E402

R = Reference()
U32 = 2**32


def catalog_arrays(cidr_lists):
    return np.array(["|".join(c) for c in cidr_lists])


def analysis_fixture(name, sites, cols, params=(96, 20, 100)):
    cat = R.catalog(sites)
    rec = R.records(cols)
    res = R.aggregate(rec, cat, params)
    d = R.result(res, hist=True)
    n_sites = len(sites)
    lo, hi, octs = R.site_sums(rec, cat, n_sites, params)
    count = np.zeros(n_sites, np.uint64)
    stats = np.zeros((n_sites, 4))
    hs, hb, hc = [], [], []
    for s, x in d["sites"].items():
        count[s] = x["count"]
        stats[s] = [x["min"], x["max"], x["avg"], x["median"]]
        nz = np.nonzero(x["hist"])[0]
        hs += [s] * len(nz)
        hb += nz.tolist()
        hc += x["hist"][nz].tolist()
    # per-record class/site via the reference's classify + attribute
    src, dst, pkts, octets, start, end = cols
    assign = np.zeros(len(src), np.uint32)
    for i in range(len(src)):
        c = R.classify(int(src[i]), int(dst[i]), int(pkts[i]), int(octets[i]), int(start[i]),
                       int(end[i]), cat, params)
        site = 0x3FFFFFFF
        if c == 0:
            site = R.attribute(int(src[i]), int(dst[i]), cat)[0]
        assign[i] = (c << 30) | site
    np.savez_compressed(
        os.path.join(HERE, f"{name}.npz"),
        sites=catalog_arrays(sites), params=np.array(params, np.uint32),
        src=src, dst=dst, pkts=pkts, octets=octets, start=start, end=end,
        tallies=d["tallies"], count=count, stats=stats, ubps_lo=lo, ubps_hi=hi, octet_sum=octs,
        hist_site=np.array(hs, np.uint32), hist_bucket=np.array(hb, np.uint32),
        hist_count=np.array(hc, np.uint32), assign=assign)
    print(f"{name}: {len(src)} records, {len(d['sites'])} sites present, tallies {d['tallies'].tolist()}")


def catalog_fixture():
    """catalog_test.cpp:93-121 / acceptance criterion 2 shapes: random /20../26
    registrations (overlaps rejected), boundary addresses and random IPs."""
    rng = np.random.default_rng(2)
    cat = R.catalog()
    regs, outcomes = [], []
    for i in range(60):
        ln = int(rng.integers(16, 27))
        base = int(rng.integers(0, U32)) & 0xFFFFFF00
        text = f"{base >> 24}.{base >> 16 & 255}.{base >> 8 & 255}.{base & 255}/{ln}"
        rid = R.register(cat, f"s{i}", [text])
        regs.append(text)
        outcomes.append(rid)
    # overlap and invalid cases
    for text in ["10.0.0.0/23", "10.0.1.0/24", "10.0.0.0", "10.0.0/24", "10.0.0.256/24",
                 "10.0.0.0/33", "10.0.0.0/0", "banana", "10.0.0.0/2x", "192.168.4.0/22",
                 "192.168.5.0/24", "10.1.2.128/26", "10.1.2.0/25"]:
        regs.append(text)
        outcomes.append(R.register(cat, f"x{len(regs)}", [text]))
    p, s = R.entries(cat)
    ips = [int(x) for x in rng.integers(0, U32, 200_000)]
    for pr in p.tolist():
        ips += [pr, pr + 255, (pr - 1) & 0xFFFFFFFF, (pr + 256) & 0xFFFFFFFF]
    ips = np.array(ips, np.uint32)
    look = np.array([R.lookup(cat, int(ip)) if R.lookup(cat, int(ip)) is not None else 0xFFFFFFFF
                     for ip in ips], np.uint32)
    seq = np.array([R.sequential_lookup(cat, int(ip)) if R.sequential_lookup(cat, int(ip)) is not None
                    else 0xFFFFFFFF for ip in ips[::50]], np.uint32)
    assert np.array_equal(look[::50], seq)
    np.savez_compressed(os.path.join(HERE, "catalog.npz"), regs=np.array(regs),
                        outcomes=np.array(outcomes, np.int64), entry_prefix=p, entry_site=s,
                        ips=ips, lookup=look)
    print(f"catalog: {len(regs)} registrations, {len(p)} entries, {len(ips)} probes")


def scalar_fixture():
    """flow_rate / flow_rate_ubps / bucket_index / median_bps known answers
    (engine_test.cpp:121-230) evaluated by the reference."""
    rng = np.random.default_rng(23)
    octs = np.concatenate([rng.integers(0, U32, 20000), [1_000_000, 125_000_000, 2305843009,
                                                         2305843010, U32 - 1, 0, 1]]).astype(np.uint64)
    durs = np.concatenate([rng.integers(1, 1_000_001, 20000), [8000, 1000, 1, 1, 1, 5, 7]]).astype(np.uint64)
    rate = np.zeros(len(octs))
    lo = np.zeros(len(octs), np.uint64)
    hi = np.zeros(len(octs), np.uint64)
    bucket = np.zeros(len(octs), np.uint32)
    for i in range(len(octs)):
        r, u = R.flow_rate(int(octs[i]), 2_000_000_000 - int(durs[i]), 2_000_000_000)
        rate[i] = r
        lo[i], hi[i] = u & (2**64 - 1), u >> 64
        bucket[i] = R.bucket_index(r)
    probe_rates = np.array([0, 9999, 10000, 99_995_000, 1e8, 5e9] +
                           [n * 1e4 for n in (0, 1, 17, 9999)] +
                           [(n + 1) * 1e4 - 0.001 for n in (0, 1, 17, 9999)] +
                           rng.uniform(0, 1.2e8, 2000).tolist())
    probe_bucket = np.array([R.bucket_index(float(r)) for r in probe_rates], np.uint32)
    # medians of random histograms (criterion 5 shape)
    med_sets, med_vals = [], []
    for _ in range(200):
        n = int(rng.integers(1, 500))
        rates = rng.uniform(0, 1.2e8, n)
        h = R.hist()
        for r in rates:
            R.hist_add(h, float(r), int(r * 1e6))
        med_sets.append(rates)
        med_vals.append(R.hist_median(h))
    lens = np.array([len(x) for x in med_sets])
    np.savez_compressed(os.path.join(HERE, "scalars.npz"), octets=octs, durations=durs, rate=rate,
                        ubps_lo=lo, ubps_hi=hi, bucket=bucket, probe_rates=probe_rates,
                        probe_bucket=probe_bucket, median_rates=np.concatenate(med_sets),
                        median_lens=lens, median=np.array(med_vals))
    print(f"scalars: {len(octs)} rate cases, {len(probe_rates)} bucket probes, 200 medians")


def warning_fixture():
    """acceptance.cpp:367-418 criterion 7: fixed-rate SiteA hours through the
    reference's generate() and hourly windows; the reference warning hours."""
    K_HOUR = 3_600_000
    K_BASE = 1_700_000_000_000
    scen = {"two": [10e6, 10e6, 10e6, 0.5e6, 0.5e6, 10e6], "one": [10e6, 0.5e6, 10e6, 10e6, 10e6, 10e6],
            "four": [10e6, 0.5e6, 0.5e6, 0.5e6, 0.5e6, 10e6]}
    out = {}
    for name, rates in scen.items():
        cols_all = [[] for _ in range(6)]
        for hour, rate in enumerate(rates):
            rec = R.generate([{"cidr": "10.1.1.0/24", "hosts": 8, "fixed_bps": rate,
                               "flows_per_hour": 200}], base_wall_ms=K_BASE + hour * K_HOUR, seed=7 + hour)
            for i, c in enumerate(R.record_columns(rec)):
                cols_all[i].append(c)
        cols = [np.concatenate(c) for c in cols_all]
        cat = R.catalog([["10.1.1.0/24"]])
        ws = R.wstate()
        warn_hours, medians = [], []
        for hour in range(len(rates)):
            s0, s1 = K_BASE + hour * K_HOUR, K_BASE + (hour + 1) * K_HOUR
            m = (cols[5] >= s0) & (cols[5] < s1)  # FlowStore::snapshot window (flow_store.cpp:75)
            win = [c[m] for c in cols]
            res = R.aggregate(R.records(win), cat, ws=s0, we=s1)
            d = R.result(res, hist=False)
            medians.append(d["sites"][0]["median"] if 0 in d["sites"] else -1.0)
            if R.evaluate_warnings(res, cat, ws):
                warn_hours.append(hour)
        out[f"{name}_cols"] = np.stack([c.astype(np.uint64) for c in cols])
        out[f"{name}_rates"] = np.array(rates)
        out[f"{name}_warn_hours"] = np.array(warn_hours, np.int64)
        out[f"{name}_medians"] = np.array(medians)
        print(f"warnings {name}: warning hours {warn_hours}")
    np.savez_compressed(os.path.join(HERE, "warnings.npz"), base=K_BASE, hour=K_HOUR, **out)


def netflow_fixture():
    """NetFlow v5 datagrams (valid and every CodecError kind) and the rows
    the unmodified reference's ingest path (decode_packet, the collector's
    reject rule, resolve_times) produces from them."""
    import netflow_gen as NG
    rng = np.random.default_rng(19)
    ds = NG.make_stream(rng, 400)
    buf, offs = NG.pack(ds)
    rows, status = [], []
    for d in ds:
        st, r, _ = R.ingest_datagram(d)
        rows.append(r)
        status.append(st)
    np.savez_compressed(os.path.join(HERE, "netflow.npz"), datagrams=buf, offsets=offs,
                        status=np.array(status, np.uint8),
                        records=np.frombuffer(b"".join(rows), np.uint8))


def hosts_fixture():
    """SiteResult::hosts of the unmodified reference (rate_engine.cpp:272-289)
    on the inputs of every analysis fixture: per (site, host) row, in the
    std::map's (site, host) order, count, min, max, avg, median, sum_bps and
    the host's histogram (sparse: row, bucket, count)."""
    import golden_io as G
    out = {}
    for name in G.ANALYSIS_SETS:
        z = G.load(name)
        params = G.params(z)
        cat = R.catalog(G.sites(z))
        res = R.aggregate(R.records(G.cols(z)), cat, params)
        d = R.result(res, hist=True, hosts=True)
        rows, stats, hr, hb, hc = [], [], [], [], []
        for s in sorted(d["sites"]):
            for ip in sorted(d["sites"][s]["hosts"]):
                h = d["sites"][s]["hosts"][ip]
                nz = np.nonzero(h["hist"])[0]
                hr += [len(rows)] * len(nz)
                hb += nz.tolist()
                hc += h["hist"][nz].tolist()
                rows.append((s, ip, h["count"]))
                stats.append((h["min"], h["max"], h["avg"], h["median"], h["sum_bps"]))
        r = np.array(rows, np.uint64).reshape(-1, 3)
        out[f"{name}_site"] = r[:, 0].astype(np.uint32)
        out[f"{name}_host"] = r[:, 1].astype(np.uint32)
        out[f"{name}_count"] = r[:, 2]
        out[f"{name}_stats"] = np.array(stats).reshape(-1, 5)
        out[f"{name}_hist_row"] = np.array(hr, np.uint32)
        out[f"{name}_hist_bucket"] = np.array(hb, np.uint32)
        out[f"{name}_hist_count"] = np.array(hc, np.uint32)
        print(f"hosts {name}: {len(rows)} (site, host) rows")
    np.savez_compressed(os.path.join(HERE, "hosts.npz"), **out)


if __name__ == "__main__":
    if len(sys.argv) > 1:  # regenerate only the named fixtures
        for name in sys.argv[1:]:
            globals()[f"{name}_fixture"]()
        sys.exit(0)
    sites, cols = parity.engine_stress_set(50_000, seed=37)
    analysis_fixture("engine_stress", sites, cols)
    sites, cols = parity.edge_set()
    analysis_fixture("edge", sites, cols)
    sites, cols = parity.tiny_duration_set()
    analysis_fixture("tiny_duration", sites, cols, params=(96, 1, 0))
    for wname, n in (("D1", 20_000), ("D2", 30_000), ("D3", 40_000)):
        w = synth.workload(wname)
        cols = synth.generate(w, n)
        analysis_fixture(f"{wname.lower()}_small", [[c] for c in w.sites.cidrs], cols)
    catalog_fixture()
    scalar_fixture()
    warning_fixture()
    netflow_fixture()
    hosts_fixture()

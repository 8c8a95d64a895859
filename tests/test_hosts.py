"""Per-host statistics (SiteResult::hosts, rate_engine.cpp:272-289; SURVEY.md
§8f next #1): the oracle restatement pinned to the unmodified reference's
rows (tests/golden/hosts.npz), and the GPU post-pass bit-exact against both
the reference fixtures and the oracle, through every input path, across
batch splits, hot-site modes, fused windows and wide registries."""
import numpy as np
import pytest

import golden_io as G
import parity
from paper_1108_1785_b200 import FilterParams, FlowBatch, FlowRecords, SiteCatalog, synth


def orc_catalog(orc, sites):
    from paper_1108_1785_b200 import Cidr
    prefixes, owners = [], []
    for sid, cl in enumerate(sites):
        for text in cl:
            c = Cidr.parse(text)
            p = c.first_prefix24()
            while p <= c.last_prefix24():
                prefixes.append(p)
                owners.append(sid)
                p += 256
    return orc.catalog(np.array(prefixes, np.uint32), np.array(owners, np.uint32))


@pytest.mark.parametrize("name", G.ANALYSIS_SETS)
def test_oracle_hosts_reproduce_reference_fixture(orc, name):
    z = G.load(name)
    got = orc.host_stats(G.cols(z), orc_catalog(orc, G.sites(z)), G.params(z), hist=True)
    G.assert_hosts_equal(got, G.hosts_expected(name))


def test_oracle_hosts_sum_to_sites(orc):
    """Finalize's merge: a site's histogram is the sum of its hosts' (:279-286)."""
    sites, cols = parity.engine_stress_set(20_000, seed=5)
    cat = SiteCatalog()
    for i, c in enumerate(sites):
        cat.register_site(f"s{i}", c)
    p, s = cat.entries_arrays()
    oc = orc.catalog(p, s)
    h = orc.host_stats(cols, oc)
    site = orc.analyze(cols, oc, cat.site_count())
    cnt = np.zeros(cat.site_count(), np.uint64)
    np.add.at(cnt, h["site"], h["count"])
    np.testing.assert_array_equal(cnt, site["count"])


# ---- GPU ----------------------------------------------------------------------

def catalog_of(sites):
    cat = SiteCatalog()
    for i, c in enumerate(sites):
        cat.register_site(f"site{i}", c)
    return cat


def host_dict(res):
    t = res.host_table
    d = {"site": t["site"], "host": t["host"], "count": t["flow_count"], "min": t["min_bps"],
         "max": t["max_bps"], "avg": t["avg_bps"], "median": t["median_bps"],
         "ubps_lo": t["rate_ubps_lo"], "ubps_hi": t["rate_ubps_hi"]}
    if res.host_histograms is not None:
        d["hist"] = res.host_histograms
    return d


def oracle_hosts(orc, cat, cols, params=(96, 20, 100)):
    p, s = cat.entries_arrays()
    return orc.host_stats(cols, orc.catalog(p, s), params)


def assert_hosts_match_oracle(res, want):
    got = host_dict(res)
    G.assert_hosts_equal(got, want, check_hist=False)
    np.testing.assert_array_equal(got["ubps_lo"], want["ubps_lo"])
    np.testing.assert_array_equal(got["ubps_hi"], want["ubps_hi"])


@pytest.fixture
def hosts_engine(engine):
    engine.set_hosts(True)
    yield engine
    engine.reset()
    engine.set_hosts(False)


@pytest.mark.gpu
@pytest.mark.parametrize("path", ["host_soa", "device_soa", "host_aos"])
@pytest.mark.parametrize("name", G.ANALYSIS_SETS)
def test_gpu_hosts_reproduce_reference_fixture(hosts_engine, name, path):
    z = G.load(name)
    cat = catalog_of(G.sites(z))
    cols = G.cols(z)
    batch = {"host_soa": lambda: FlowBatch(*cols), "device_soa": lambda: FlowBatch(*cols).to_device(),
             "host_aos": lambda: FlowRecords(synth.to_aos(cols))}[path]()
    res = hosts_engine.aggregate(batch, cat, FilterParams(*G.params(z)), histograms=True)
    want = G.hosts_expected(name)
    G.assert_hosts_equal(host_dict(res), want)
    rows, bks, cnt = hosts_engine.host_histogram_entries()  # sparse form of the same histograms
    np.testing.assert_array_equal(rows, want["hist_row"])
    np.testing.assert_array_equal(bks, want["hist_bucket"])
    np.testing.assert_array_equal(cnt, want["hist_count"])
    # SiteResult.hosts view: every present site holds exactly its rows.
    n_rows = sum(len(sr.hosts) for sr in res.sites.values())
    assert n_rows == want["n"]


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["off", "force", "auto"])
@pytest.mark.parametrize("name,n", [("D1", 200_000), ("D2", 300_000), ("D3", 1_000_000)])
def test_gpu_hosts_match_oracle(hosts_engine, orc, name, n, mode):
    w = synth.workload(name)
    cols = synth.generate(w, n)
    cat = SiteCatalog()
    w.sites.register(cat)
    hosts_engine.set_hot_mode(mode)
    try:
        res = hosts_engine.aggregate(FlowBatch(*cols).to_device(), cat)
    finally:
        hosts_engine.set_hot_mode("auto")
    assert_hosts_match_oracle(res, oracle_hosts(orc, cat, cols))


@pytest.mark.gpu
def test_gpu_hosts_split_batches_and_window(hosts_engine, orc):
    """Three accumulate calls (three log slices) and a fused window equal the
    oracle on the concatenated / snapshotted input."""
    w = synth.workload("D2")
    cols = synth.generate(w, 500_000)
    cat = SiteCatalog()
    w.sites.register(cat)
    cuts = [0, 123_457, 333_333, 500_000]
    for a, b in zip(cuts[:-1], cuts[1:]):
        hosts_engine.accumulate(FlowBatch(*[c[a:b] for c in cols]).to_device(), cat)
    res = hosts_engine.finalize(cat)
    assert_hosts_match_oracle(res, oracle_hosts(orc, cat, cols))
    end = cols[5]
    lo, hi = int(np.percentile(end, 20)), int(np.percentile(end, 70))
    res = hosts_engine.aggregate_window(FlowBatch(*cols).to_device(), cat, lo, hi)
    m = (end >= lo) & (end < hi)
    assert_hosts_match_oracle(res, oracle_hosts(orc, cat, tuple(c[m] for c in cols)))


@pytest.mark.gpu
def test_gpu_hosts_wide_registry(hosts_engine, orc):
    """>= 2^18 sites: K2's wide log (separate bucket column) feeds the post-pass."""
    rng = np.random.default_rng(11)
    n_sites = 300_000
    base = 0x20000000
    cat = SiteCatalog()
    for i in range(n_sites):
        a = base + i * 256
        cat.register_site(f"w{i}", [f"{a >> 24}.{(a >> 16) & 255}.{(a >> 8) & 255}.0/24"])
    n = 400_000
    site = rng.integers(0, n_sites, n)
    src = (base + site * 256 + rng.integers(0, 4, n)).astype(np.uint32)
    dst = rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32)
    flip = rng.random(n) < 0.3
    src[flip], dst[flip] = dst[flip], src[flip].copy()
    cols = parity.make_cols(src, dst, rng.integers(20, 200, n), rng.integers(20_000, 2_000_000, n),
                            rng.integers(100, 100_000, n))
    res = hosts_engine.aggregate(FlowBatch(*cols).to_device(), cat)
    assert_hosts_match_oracle(res, oracle_hosts(orc, cat, cols))


@pytest.mark.gpu
def test_gpu_hosts_both_endpoints_and_empty(hosts_engine, orc):
    """Both endpoints registered: the host is src (src lookup first); a src
    whose /16 holds sites but whose /24 does not falls through to dst."""
    cat = catalog_of([["10.1.1.0/24"], ["10.1.2.0/24"], ["10.2.0.0/16"]])
    ip = lambda a, b, c, d: (a << 24) | (b << 16) | (c << 8) | d
    src = np.array([ip(10, 1, 1, 5), ip(10, 1, 3, 9), ip(10, 2, 7, 7), ip(10, 1, 2, 4), ip(9, 9, 9, 9)], np.uint32)
    dst = np.array([ip(10, 1, 2, 6), ip(10, 1, 2, 8), ip(10, 1, 1, 1), ip(10, 9, 9, 9), ip(8, 8, 8, 8)], np.uint32)
    cols = parity.make_cols(src, dst, np.full(5, 50), np.full(5, 500_000), np.full(5, 1000))
    res = hosts_engine.aggregate(FlowBatch(*cols), cat)
    want = oracle_hosts(orc, cat, cols)
    assert_hosts_match_oracle(res, want)
    assert {(int(s), int(h)) for s, h in zip(want["site"], want["host"])} == {
        (0, ip(10, 1, 1, 5)), (1, ip(10, 1, 2, 8)), (2, ip(10, 2, 7, 7)), (1, ip(10, 1, 2, 4))}
    # No Forward flows: zero rows.
    res = hosts_engine.aggregate(FlowBatch(*[c[4:] for c in cols]), cat)
    assert len(res.host_table) == 0
    res = hosts_engine.aggregate(FlowBatch(*[c[:0] for c in cols]), cat)
    assert len(res.host_table) == 0


@pytest.mark.gpu
def test_gpu_hosts_mode_switching(engine):
    cat = catalog_of([["10.1.1.0/24"]])
    cols = parity.make_cols(np.array([0x0A010105], np.uint32), np.array([1], np.uint32),
                            np.array([50]), np.array([500_000]), np.array([1000]))
    res = engine.aggregate(FlowBatch(*cols), cat)
    assert res.host_table is None and res.sites[0].hosts == {}
    engine.set_hosts(True)
    try:
        engine.accumulate(FlowBatch(*cols), cat)
        with pytest.raises(Exception):
            engine.set_hosts(False)  # only between accumulations
        res = engine.finalize(cat)
        assert list(res.sites[0].hosts) == [0x0A010105]
        assert res.sites[0].hosts[0x0A010105].stats.flow_count == 1
    finally:
        engine.reset()
        engine.set_hosts(False)


@pytest.mark.gpu
@pytest.mark.slow
def test_gpu_hosts_large_properties(hosts_engine):
    """12M records over 64 /16 sites (~millions of host rows: the 64-bit
    sort-key path): the host rows partition every site's flows -- counts,
    u128 micro-bps sums, min and max recombine to the site row exactly; rows
    are strictly (site, host) ordered; every median lies in [min, max]."""
    rng = np.random.default_rng(12)
    cat = catalog_of([[f"10.{i}.0.0/16"] for i in range(64)])
    n = 12_000_001
    src = (0x0A000000 + (rng.integers(0, 64, n) << 16) + rng.integers(0, 65536, n)).astype(np.uint32)
    dst = rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32)
    flip = rng.random(n) < 0.4
    src[flip], dst[flip] = dst[flip], src[flip].copy()
    cols = parity.make_cols(src, dst, rng.integers(1, 400, n), rng.integers(1, 2**32, n, dtype=np.uint64),
                            rng.integers(1, 3_600_000, n), end=4_000_000_000)
    res = hosts_engine.aggregate(FlowBatch(*cols).to_device(), cat)
    t, st = res.host_table, res.table
    assert len(t) > 2**18
    key = t["site"].astype(np.uint64) << np.uint64(32) | t["host"].astype(np.uint64)
    assert np.all(np.diff(key) > 0)
    n = len(st)
    cnt = np.zeros(n, np.uint64)
    np.add.at(cnt, t["site"], t["flow_count"])
    np.testing.assert_array_equal(cnt, st["flow_count"])
    mn = np.full(n, np.inf)
    mx = np.zeros(n)
    np.minimum.at(mn, t["site"], t["min_bps"])
    np.maximum.at(mx, t["site"], t["max_bps"])
    pres = st["flow_count"] > 0
    np.testing.assert_array_equal(mn[pres], st["min_bps"][pres])
    np.testing.assert_array_equal(mx[pres], st["max_bps"][pres])
    lo = [0] * n
    for s, a, b in zip(t["site"].tolist(), t["rate_ubps_lo"].tolist(), t["rate_ubps_hi"].tolist()):
        lo[s] += b << 64 | a
    want = [int(b) << 64 | int(a) for a, b in zip(st["rate_ubps_lo"], st["rate_ubps_hi"])]
    assert lo == want
    assert np.all((t["median_bps"] >= t["min_bps"]) & (t["median_bps"] <= t["max_bps"]))
    rows, bks, c = hosts_engine.host_histogram_entries()  # 64-bit keys: sparse histograms sum to the counts
    per_row = np.zeros(len(t), np.uint64)
    np.add.at(per_row, rows, c)
    np.testing.assert_array_equal(per_row, t["flow_count"])
    assert np.all(bks <= 10000)


@pytest.mark.gpu
def test_gpu_host_results_c_abi_errors(hosts_engine):
    """The C-ABI's capacity rules (gnetmon.h): rows and sparse entries report
    GNM_ERR_CAPACITY when the caller's arrays are short, the NULL query form
    only sets the count, and rows outlive later accumulate calls until the
    next finalize."""
    import ctypes as C
    from paper_1108_1785_b200 import _lib
    cat = catalog_of([["10.1.1.0/24"], ["10.1.2.0/24"]])
    ip = lambda a, b, c, d: (a << 24) | (b << 16) | (c << 8) | d
    src = np.array([ip(10, 1, 1, 5), ip(10, 1, 1, 6), ip(10, 1, 2, 7)], np.uint32)
    cols = parity.make_cols(src, np.full(3, 1, np.uint32), np.full(3, 50), np.full(3, 500_000), np.full(3, 1000))
    hosts_engine.aggregate(FlowBatch(*cols), cat)
    h = hosts_engine.handle
    assert _lib.lib.gnm_host_count(h) == 3
    rows = np.zeros(2, _lib.HOST_STATS_DTYPE)
    assert _lib.lib.gnm_host_results(h, rows.ctypes.data, 2, None) == _lib.ERR_CAPACITY
    n = C.c_uint64()
    assert _lib.lib.gnm_host_histogram_entries(h, None, None, None, 0, C.byref(n)) == _lib.OK
    assert n.value == 3
    a = np.zeros(2, np.uint32)
    assert _lib.lib.gnm_host_histogram_entries(h, a.ctypes.data, a.ctypes.data, a.ctypes.data, 2,
                                               C.byref(n)) == _lib.ERR_CAPACITY
    hosts_engine.accumulate(FlowBatch(*cols), cat)  # rows stay valid until the next finalize
    assert _lib.lib.gnm_host_count(h) == 3
    hosts_engine.reset()
    assert _lib.lib.gnm_host_count(h) == 0


@pytest.mark.gpu
def test_gpu_hosts_union_path_single_context(hosts_engine):
    """The cross-context path with one context (union = its own keys, no
    collective): gnm_hosts_local_keys -> set_keys -> prepare_median ->
    finalize gives the same rows as the local path; the histograms of union
    rows count this context's own flows (here: all of them) over the union
    rows, so they equal the local path's."""
    w = synth.workload("D2")
    cols = synth.generate(w, 300_000)
    cat = SiteCatalog()
    w.sites.register(cat)
    want = hosts_engine.aggregate(FlowBatch(*cols).to_device(), cat).host_table
    want_e = hosts_engine.host_histogram_entries()
    hosts_engine.accumulate(FlowBatch(*cols).to_device(), cat)
    keys = hosts_engine.hosts_local_keys(cat)
    t = hosts_engine.hosts_set_keys(keys.clone())
    assert t["n"] == len(want)
    hosts_engine.hosts_prepare_median()
    res = hosts_engine.finalize(cat)
    np.testing.assert_array_equal(res.host_table, want)
    for x, y in zip(hosts_engine.host_histogram_entries(), want_e):
        np.testing.assert_array_equal(x, y)


@pytest.mark.gpu
@pytest.mark.slow
def test_gpu_hosts_full_size_d3(hosts_engine, orc):
    """Per-host rows at D3's full size (100M records, 80k (site, host) rows)
    equal the oracle's restatement bit for bit."""
    w = synth.workload("D3")
    cols = synth.generate(w, w.n)
    cat = SiteCatalog()
    w.sites.register(cat)
    res = hosts_engine.aggregate(FlowBatch(*cols).to_device(), cat)
    assert_hosts_match_oracle(res, oracle_hosts(orc, cat, cols))

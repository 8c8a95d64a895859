"""GPU parity: the sm_100a path (through the C-ABI) against the CPU oracle,
bit-exact on every output of the site-level AnalysisResult."""
import numpy as np
import pytest

import parity
from paper_1108_1785_b200 import (FilterParams, FlowBatch, FlowRecords, SiteCatalog,
                                  aggregate_partitioned, synth)

pytestmark = pytest.mark.gpu


def catalog_of(sites):
    cat = SiteCatalog()
    for i, cidrs in enumerate(sites):
        cat.register_site(f"site{i}", cidrs)
    return cat


def layout_catalog(layout):
    cat = SiteCatalog()
    layout.register(cat)
    return cat


@pytest.mark.parametrize("on_device", [False, True])
def test_engine_stress_set_bit_exact(engine, orc, on_device):
    sites, cols = parity.engine_stress_set()
    cat = catalog_of(sites)
    batch = FlowBatch(*cols)
    if on_device:
        batch = batch.to_device()
    res = engine.aggregate(batch, cat, histograms=True)
    parity.assert_matches_oracle(res, parity.oracle_reference(orc, cat, cols))
    assert res.tallies.total() == len(cols[0])


def test_edge_set_bit_exact(engine, orc):
    sites, cols = parity.edge_set()
    cat = catalog_of(sites)
    res = engine.aggregate(FlowBatch(*cols), cat, histograms=True)
    parity.assert_matches_oracle(res, parity.oracle_reference(orc, cat, cols))


def test_tiny_durations_third_limb(engine, orc):
    sites, cols = parity.tiny_duration_set()
    cat = catalog_of(sites)
    params = FilterParams(min_duration_ms=0, min_packets=1)
    res = engine.aggregate(FlowBatch(*cols), cat, params, histograms=True)
    acc = parity.oracle_reference(orc, cat, cols, (96, 1, 0))
    assert acc["ubps_hi"].max() > 0  # the quotient really exceeded 2^64
    parity.assert_matches_oracle(res, acc)


@pytest.mark.parametrize("name,n", [("D1", 100_000), ("D2", 300_000), ("D3", 400_000)])
def test_workload_shapes_bit_exact(engine, orc, name, n):
    w = synth.workload(name)
    cols = synth.generate(w, n)
    cat = layout_catalog(w.sites)
    res = engine.aggregate(FlowBatch(*cols).to_device(), cat, histograms=(name != "D3"))
    parity.assert_matches_oracle(res, parity.oracle_reference(orc, cat, cols))


@pytest.mark.parametrize("params", [FilterParams(), FilterParams(ack_avg_size_max=200),
                                    FilterParams(min_packets=50, min_duration_ms=500),
                                    FilterParams(ack_avg_size_max=0xFFFFFFFF)])
def test_filter_params(engine, orc, params):
    sites, cols = parity.engine_stress_set(20_000, seed=17)
    cat = catalog_of(sites)
    res = engine.aggregate(FlowBatch(*cols), cat, params)
    acc = parity.oracle_reference(orc, cat, cols, (params.ack_avg_size_max, params.min_packets,
                                                   params.min_duration_ms))
    parity.assert_matches_oracle(res, acc)


def test_classify_matches_oracle(engine, orc):
    sites, cols = parity.engine_stress_set()
    cat = catalog_of(sites)
    got = engine.classify(FlowBatch(*cols), cat)
    p, s = cat.entries_arrays()
    want = orc.classify(cols, orc.catalog(p, s))
    np.testing.assert_array_equal(got, want)


def test_classify_d2_mixed_prefixes(engine, orc):
    w = synth.workload("D2")
    cols = synth.generate(w, 200_000)
    cat = layout_catalog(w.sites)
    got = engine.classify(FlowBatch(*cols).to_device(), cat)
    p, s = cat.entries_arrays()
    np.testing.assert_array_equal(got, orc.classify(cols, orc.catalog(p, s)))


def test_aos_equals_soa(engine):
    w = synth.workload("D2")
    cols = synth.generate(w, 100_000)
    cat = layout_catalog(w.sites)
    soa = engine.aggregate(FlowBatch(*cols), cat, histograms=True)
    aos_host = engine.aggregate(FlowRecords(synth.to_aos(cols)), cat, histograms=True)
    import torch
    aos_dev = engine.aggregate(FlowRecords(torch.from_numpy(synth.to_aos(cols)).cuda()), cat,
                               histograms=True)
    for r in (aos_host, aos_dev):
        np.testing.assert_array_equal(r.table, soa.table)
        np.testing.assert_array_equal(r.histograms, soa.histograms)
        assert r.tallies == soa.tallies


def test_partition_and_chunk_independence(engine):
    """acceptance.cpp:328-362 / engine_test.cpp:282-305 on the GPU: any batch
    split and any loader chunking gives the identical result."""
    sites, cols = parity.engine_stress_set(20_000, seed=41)
    cat = catalog_of(sites)
    batch = FlowBatch(*cols)
    whole = engine.aggregate(batch, cat, histograms=True)
    rng = np.random.default_rng(6)
    for _ in range(5):
        cuts = sorted(rng.integers(0, len(batch) + 1, rng.integers(1, 8)).tolist())
        part = aggregate_partitioned(batch, cat, FilterParams(), cuts, histograms=True)
        np.testing.assert_array_equal(part.table, whole.table)
        np.testing.assert_array_equal(part.histograms, whole.histograms)
    engine.set_chunk_records(1500)
    try:
        chunked = engine.aggregate(batch, cat, histograms=True)
    finally:
        engine.set_chunk_records(1 << 22)
    np.testing.assert_array_equal(chunked.table, whole.table)


def test_empty_and_no_forward(engine):
    cat = catalog_of([["10.1.2.0/24"]])
    empty = parity.make_cols([], [], [], [], [])
    r = engine.aggregate(FlowBatch(*empty), cat)
    assert r.sites == {} and r.tallies.total() == 0
    # engine_test.cpp:330-342: ack, admin, unmatched, no forward flow.
    cols = parity.make_cols([0x0A010203, 0x0A010203, 0xC0000001], [0, 0, 0xC0000002],
                            [100, 5, 100], [4000, 4000, 1_000_000], [1000, 50, 1000])
    r = engine.aggregate(FlowBatch(*cols), cat)
    assert r.sites == {}
    assert (r.tallies.pure_ack, r.tallies.administrative, r.tallies.unmatched,
            r.tallies.forward) == (1, 1, 1, 0)


@pytest.mark.parametrize("mode", ["off", "force", "auto"])
def test_hot_site_modes_bit_exact(engine, orc, mode):
    """Block-private (shared-memory) accumulation of hot sites with 32-bit
    carry chains must equal the oracle: full-range octets overflow every
    limb of the per-block accumulators."""
    sites, cols = parity.engine_stress_set(200_000, seed=11)
    cat = catalog_of(sites)
    engine.set_hot_mode(mode)
    try:
        res = engine.aggregate(FlowBatch(*cols).to_device(), cat, histograms=True)
        res3 = engine.aggregate(FlowBatch(*parity.tiny_duration_set()[1]).to_device(),
                                catalog_of(parity.tiny_duration_set()[0]),
                                FilterParams(min_duration_ms=0, min_packets=1))
    finally:
        engine.set_hot_mode("auto")
    parity.assert_matches_oracle(res, parity.oracle_reference(orc, cat, cols))
    tcat = catalog_of(parity.tiny_duration_set()[0])
    parity.assert_matches_oracle(res3, parity.oracle_reference(orc, tcat, parity.tiny_duration_set()[1],
                                                               (96, 1, 0)))


@pytest.mark.parametrize("mode", ["off", "force", "auto"])
def test_zipf_d3_hot_modes(engine, orc, mode):
    """D3 shape (10k Zipf sites) large enough for the auto planner to engage."""
    w = synth.workload("D3")
    cols = synth.generate(w, 2_000_000)
    cat = layout_catalog(w.sites)
    engine.set_hot_mode(mode)
    try:
        res = engine.aggregate(FlowBatch(*cols).to_device(), cat)
    finally:
        engine.set_hot_mode("auto")
    parity.assert_matches_oracle(res, parity.oracle_reference(orc, cat, cols))


def test_state_resets_between_calls(engine, orc):
    """The device partials are all-zero at rest: back-to-back calls on
    different data and registries do not leak into each other."""
    sites, cols = parity.engine_stress_set(10_000, seed=3)
    cat = catalog_of(sites)
    for _ in range(3):
        r = engine.aggregate(FlowBatch(*cols), cat)
    parity.assert_matches_oracle(r, parity.oracle_reference(orc, cat, cols))
    w = synth.workload("D1")
    c2 = synth.generate(w, 50_000)
    cat2 = layout_catalog(w.sites)
    r2 = engine.aggregate(FlowBatch(*c2), cat2)
    parity.assert_matches_oracle(r2, parity.oracle_reference(orc, cat2, c2))
    r3 = engine.aggregate(FlowBatch(*cols), cat)
    np.testing.assert_array_equal(r3.table, r.table)


@pytest.mark.parametrize("n", [300_007, 12_000_001])
def test_multi_cta_remainders_and_epochs(engine, orc, n):
    """Sizes that span several persistent CTAs, the < 64-record remainder
    and (12M: > 29 rounds of 32 tiles per CTA) K2 epochs with limb
    normalization, on the engine stress set (full-range octets push the
    16-bit limbs of the few hot sites past the flush bound) and the D3
    shape."""
    sites, cols = parity.engine_stress_set(n, seed=23)
    cat = catalog_of(sites)
    res = engine.aggregate(FlowBatch(*cols).to_device(), cat, histograms=(n < 1_000_000))
    parity.assert_matches_oracle(res, parity.oracle_reference(orc, cat, cols),
                                 check_hist=(n < 1_000_000))
    w = synth.workload("D3")
    cols = synth.generate(w, n)
    cat = layout_catalog(w.sites)
    res = engine.aggregate(FlowBatch(*cols).to_device(), cat)
    parity.assert_matches_oracle(res, parity.oracle_reference(orc, cat, cols))


def _window_mask(cols, lo, hi):
    end = cols[5]
    return (end >= np.uint64(lo)) & (end < np.uint64(hi))


@pytest.mark.parametrize("on_device", [False, True])
def test_window_fused_snapshot_bit_exact(engine, orc, on_device):
    """gnm_analyze_window / gnm_accumulate_window = FlowStore::snapshot
    (flow_store.cpp:62-80: end_ms in [start, end)) fused into K1/K2: equal to
    the oracle on the host-filtered records, tallies included, for a
    partial, an empty, a full and a one-millisecond window."""
    w = synth.workload("D2")
    cols = synth.generate(w, 400_000)
    cat = layout_catalog(w.sites)
    end = cols[5]
    lo_all, hi_all = int(end.min()), int(end.max()) + 1
    mid = (lo_all + hi_all) // 2
    windows = [(lo_all + (hi_all - lo_all) // 4, mid), (hi_all + 10, hi_all + 20), (0, 2**64 - 1),
               (int(end[12345]), int(end[12345]) + 1)]
    batch = FlowBatch(*cols)
    if on_device:
        batch = batch.to_device()
    for lo, hi in windows:
        m = _window_mask(cols, lo, hi)
        sub = tuple(np.ascontiguousarray(c[m]) for c in cols)
        want = parity.oracle_reference(orc, cat, sub)
        got = engine.aggregate_window(batch, cat, lo, hi, histograms=True)
        parity.assert_matches_oracle(got, want)
        assert got.tallies.total() == int(m.sum())
        assert (got.window_start_ms, got.window_end_ms) == (lo, hi)
    # split accumulation: two batches, one window
    lo, hi = windows[0]
    engine.accumulate(FlowBatch(*[c[:150_000] for c in cols]), cat, window=(lo, hi))
    engine.accumulate(FlowBatch(*[c[150_000:] for c in cols]), cat, window=(lo, hi))
    got = engine.finalize(cat, lo, hi)
    m = _window_mask(cols, lo, hi)
    parity.assert_matches_oracle(got, parity.oracle_reference(orc, cat, tuple(np.ascontiguousarray(c[m]) for c in cols)))


@pytest.mark.parametrize("mode", ["force", "auto"])
def test_sampled_min_max_respects_window(engine, orc, mode):
    """K1 reduces its sampled flows' rates into the sites' min/max (they
    seed K2's hot-slot caches): records the window drops carry the most
    extreme rates of the batch here, so a sample that ignored the window
    (or the class filter) would show up in min_bps / max_bps."""
    w = synth.workload("D3")
    cols = [c.copy() for c in synth.generate(w, 600_000)]
    cat = layout_catalog(w.sites)
    end = cols[5]
    lo, hi = int(np.percentile(end, 20)), int(np.percentile(end, 80))
    out = ~_window_mask(cols, lo, hi)
    idx = np.flatnonzero(out)
    # Outside the window: half very fast (4e9 octets in 1 s), half very slow
    # (2048 octets over ~11 days), all Forward-shaped for the hot sites.
    fast, slow = idx[0::2], idx[1::2]
    cols[3][fast] = np.uint32(4_000_000_000)
    cols[2][fast] = np.uint32(25)
    cols[4][fast] = cols[5][fast] - np.uint64(1000)
    cols[3][slow] = np.uint32(2048)
    cols[2][slow] = np.uint32(20)
    cols[4][slow] = cols[5][slow] - np.uint64(1_000_000_000)
    batch = FlowBatch(*cols).to_device()
    engine.set_hot_mode(mode)
    try:
        got = engine.aggregate_window(batch, cat, lo, hi)
        full = engine.aggregate(batch, cat)
    finally:
        engine.set_hot_mode("auto")
    m = ~out
    parity.assert_matches_oracle(got, parity.oracle_reference(
        orc, cat, tuple(np.ascontiguousarray(c[m]) for c in cols)))
    # and the unwindowed call does see the extremes
    parity.assert_matches_oracle(full, parity.oracle_reference(orc, cat, tuple(cols)))


def test_window_fused_aos(engine, orc):
    sites, cols = parity.engine_stress_set(50_000, seed=31)
    cat = catalog_of(sites)
    end = cols[5]
    lo = int(np.percentile(end, 30))
    hi = int(np.percentile(end, 80))
    from paper_1108_1785_b200 import FlowRecords
    got = engine.aggregate_window(FlowRecords(synth.to_aos(cols)), cat, lo, hi)
    m = _window_mask(cols, lo, hi)
    parity.assert_matches_oracle(got, parity.oracle_reference(orc, cat, tuple(np.ascontiguousarray(c[m]) for c in cols)))


def test_graph_replay_matches_plain_calls(engine, orc):
    """Repeated device-batch calls replay a captured CUDA graph: identical
    results to graphs off, across in-place data changes, a registry switch
    in between (partials / table / log reallocated), hot-mode changes and a
    fused window."""
    import torch
    from paper_1108_1785_b200 import Engine
    w = synth.workload("D2")
    cols = synth.generate(w, 400_000)
    cat = layout_catalog(w.sites)
    dev = [torch.from_numpy(c.view(np.int32 if c.dtype.itemsize == 4 else np.int64).copy()).cuda() for c in cols]
    batch = FlowBatch(*dev)
    plain = Engine(0)
    plain.set_graphs(False)
    want = plain.aggregate(batch, cat)
    for _ in range(4):  # plain, capture, replays
        got = engine.aggregate(batch, cat)
        np.testing.assert_array_equal(got.table, want.table)
    # contents change in place: the replay reads the new data
    dev[3].mul_(2)
    want2 = plain.aggregate(batch, cat)
    got2 = engine.aggregate(batch, cat)
    np.testing.assert_array_equal(got2.table, want2.table)
    assert not np.array_equal(got2.table, want.table)
    # another registry (bigger) in between, then the first again
    big = layout_catalog(synth.workload("D3").sites)
    engine.aggregate(FlowBatch(*synth.generate(synth.workload("D3"), 300_000)).to_device(), big)
    for _ in range(3):
        np.testing.assert_array_equal(engine.aggregate(batch, cat).table, want2.table)
    for mode in ("off", "force", "auto"):
        engine.set_hot_mode(mode)
        for _ in range(3):
            np.testing.assert_array_equal(engine.aggregate(batch, cat).table, want2.table)
    end = cols[5]
    lo, hi = int(np.percentile(end, 25)), int(np.percentile(end, 75))
    wantw = plain.aggregate_window(batch, cat, lo, hi)
    for _ in range(3):
        np.testing.assert_array_equal(engine.aggregate_window(batch, cat, lo, hi).table, wantw.table)
    plain.close()


def test_graph_replay_aos(engine):
    """Graph replay of repeated device AoS (64-byte FlowRecord) calls."""
    import torch
    from paper_1108_1785_b200 import Engine
    w = synth.workload("D1")
    cols = synth.generate(w, 200_000)
    cat = layout_catalog(w.sites)
    rows = torch.from_numpy(synth.to_aos(cols)).cuda()
    plain = Engine(0)
    plain.set_graphs(False)
    want = plain.aggregate(FlowRecords(rows), cat)
    for _ in range(4):
        np.testing.assert_array_equal(engine.aggregate(FlowRecords(rows), cat).table, want.table)
    plain.close()


def test_fresh_registries_never_reuse_a_stale_device_table(engine):
    """Registries created and dropped in a loop (their handles' addresses get
    recycled): every call sees its own registry's table, because registry
    versions are unique across the process."""
    import gc
    for i in range(24):
        cat = SiteCatalog()
        cat.register_site("only", [f"10.{i}.1.0/24"])
        src = np.array([(10 << 24) | (i << 16) | (1 << 8) | 5, (10 << 24) | (((i + 1) % 24) << 16) | (1 << 8) | 5],
                       np.uint32)
        cols = parity.make_cols(src, np.full(2, 1, np.uint32), np.full(2, 50), np.full(2, 500_000), np.full(2, 1000))
        got = engine.classify(FlowBatch(*cols), cat)
        assert int(got[0]) == 0 and int(got[1]) >> 30 == 3, (i, got)
        del cat
        gc.collect()


def test_graph_cache_ring_of_batches(engine):
    """A ring of streaming batches (different buffers and windows, cycled)
    replays one graph per input set: identical to plain calls."""
    import torch
    from paper_1108_1785_b200 import Engine
    w = synth.workload("D5")
    cat = layout_catalog(w.sites)
    ring = []
    for j in range(3):
        cols = synth.generate(w, 150_000, index_offset=j * 150_000)
        dev = [torch.from_numpy(c.view(np.int32 if c.dtype.itemsize == 4 else np.int64).copy()).cuda() for c in cols]
        lo = int(np.percentile(cols[5], 5 + 10 * j))
        ring.append((FlowBatch(*dev), lo, lo + 60_000_000))
    plain = Engine(0)
    plain.set_graphs(False)
    want = [plain.aggregate_window(b, cat, lo, hi).table for b, lo, hi in ring]
    for rep in range(4):
        for (b, lo, hi), t in zip(ring, want):
            np.testing.assert_array_equal(engine.aggregate_window(b, cat, lo, hi).table, t)
    plain.close()


@pytest.mark.slow
@pytest.mark.parametrize("name", ["D1", "D2", "D3"])
def test_full_size_configs_bit_exact(engine, orc, name):
    """BASELINE.json configs[0..2] at their full sizes (D1 100k records / 256
    sites, D2 1M / 1k mixed prefixes, D3 100M / 10k Zipf sites): the whole
    site table (counts, byte and u128 micro-bps sums, min / max / avg /
    median) and the tallies equal the C oracle's bit for bit."""
    w = synth.workload(name)
    cols = synth.generate(w, w.n)
    cat = layout_catalog(w.sites)
    res = engine.aggregate(FlowBatch(*cols).to_device(), cat)
    assert res.tallies.total() == w.n
    parity.assert_matches_oracle(res, parity.oracle_reference(orc, cat, cols), check_hist=False)


@pytest.mark.slow
def test_d4_one_billion_records_chunked(engine, orc):
    """BASELINE.json configs[3] (D4: 1B records with D3's distribution) on one
    GPU through the split API: ten 100M-record index shards accumulated into
    one context (ten K2 launches, one 1B-entry log), finalized once, equal
    the C oracle run over the same shards bit for bit."""
    w = synth.workload("D4")
    cat = layout_catalog(w.sites)
    p, s = cat.entries_arrays()
    oc = orc.catalog(p, s)
    acc = None
    shard = w.n // 10
    for k in range(10):
        cols = synth.generate(w, shard, index_offset=k * shard)
        engine.accumulate(FlowBatch(*cols).to_device(), cat)
        acc = orc.aggregate(cols, oc, cat.site_count(), acc=acc)
        del cols
    res = engine.finalize(cat)
    assert res.tallies.total() == w.n
    parity.assert_matches_oracle(res, orc.finalize(acc), check_hist=False)

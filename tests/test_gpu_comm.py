"""Multi-GPU inside the library (gnetmon.h gnm_ctx_comm_* / gnm_group_*):
the two-round combine runs in gnm_finalize over the context's communicator.

A test box has one GPU and NCCL refuses two ranks on one device, so:
* the loopback group runs the exact in-library orchestration (shards by the
  reference's worker boundaries, one host thread per rank, round 1 / K3a+K2b
  / round 2 / K3b, the per-host key union and its two rounds) with 2-3 ranks
  on cuda:0, exchanging through host memory -- compared bit for bit with one
  engine over the whole batch, and with the C oracle;
* NCCL itself runs at world size 1: a one-device clique (ncclCommInitAll)
  and a per-process communicator (ncclCommInitRank), including CUDA-graph
  capture and replay of the collectives.
"""
import numpy as np
import pytest

import parity

pytestmark = pytest.mark.gpu


def _setup(name="D1", n=None, seed_sites=None):
    from paper_1108_1785_b200 import FlowBatch, SiteCatalog, synth
    w = synth.workload(name)
    cols = synth.generate(w, n or w.n)
    cat = SiteCatalog()
    w.sites.register(cat)
    return cat, cols, FlowBatch(*cols)


def _same_sites(a, b):
    assert np.array_equal(a.table, b.table), "site rows differ"
    assert a.tallies == b.tallies


def _same_hosts(a, b):
    assert len(a.host_table) == len(b.host_table)
    assert a.host_table.tobytes() == b.host_table.tobytes(), "host rows differ"


@pytest.mark.parametrize("ranks", [2, 3])
def test_loopback_group_equals_one_engine(engine, ranks):
    from paper_1108_1785_b200 import Group
    cat, cols, batch = _setup("D2", 400_000)
    want = engine.aggregate(batch, cat, histograms=True)
    with Group([0] * ranks, kind="loopback") as g:
        got = g.aggregate(batch, cat, histograms=True)
        _same_sites(got, want)
        assert np.array_equal(got.histograms, want.histograms)
        # device-resident input, a second call on the same group
        dev = batch.to_device("cuda:0")
        _same_sites(g.aggregate(dev, cat), want)


def test_loopback_group_skewed_d3_slice(engine, orc):
    """Zipf sites with hot-slot accumulation on every rank, against the oracle."""
    from paper_1108_1785_b200 import Group
    cat, cols, batch = _setup("D3", 3_000_000)
    want = engine.aggregate(batch.to_device("cuda:0"), cat)
    with Group([0, 0], kind="loopback") as g:
        got = g.aggregate(batch.to_device("cuda:0"), cat)
    _same_sites(got, want)
    parity.assert_matches_oracle(got, parity.oracle_reference(orc, cat, cols), check_hist=False)


def test_loopback_group_hosts_union(engine):
    """Per-host rows across ranks: the key union, the two rounds over the
    union's rows, and the ranks' host histograms summed."""
    from paper_1108_1785_b200 import Group
    cat, cols, batch = _setup("D2", 300_000)
    engine.set_hosts(True)
    try:
        want = engine.aggregate(batch, cat)
        we = engine.host_histogram_entries()
    finally:
        engine.set_hosts(False)
    with Group([0, 0, 0], kind="loopback") as g:
        g.set_hosts(True)
        got = g.aggregate(batch, cat)
        ge = g.host_histogram_entries()
    _same_sites(got, want)
    _same_hosts(got, want)
    for x, y in zip(ge, we):
        assert np.array_equal(x, y)


def test_loopback_group_aos_and_edges(engine):
    from paper_1108_1785_b200 import FlowRecords, Group, SiteCatalog, FilterParams, synth
    sites, cols = parity.engine_stress_set()
    cat = SiteCatalog()
    for i, c in enumerate(sites):
        cat.register_site(f"s{i}", c)
    rows = FlowRecords(synth.to_aos(cols))
    for p in (None, FilterParams(ack_avg_size_max=200, min_packets=50, min_duration_ms=500)):
        want = engine.aggregate(rows, cat, p)
        with Group([0, 0], kind="loopback") as g:
            _same_sites(g.aggregate(rows, cat, p), want)


def test_loopback_group_more_ranks_than_records(engine):
    from paper_1108_1785_b200 import Group
    cat, cols, batch = _setup("D1", 3)
    want = engine.aggregate(batch, cat)
    with Group([0] * 5, kind="loopback") as g:
        g.set_hosts(True)
        got = g.aggregate(batch, cat)
    _same_sites(got, want)


def test_nccl_clique_single_device(engine):
    from paper_1108_1785_b200 import Group
    cat, cols, batch = _setup("D1")
    want = engine.aggregate(batch, cat)
    engine.set_hosts(True)
    try:
        want_h = engine.aggregate(batch, cat)
    finally:
        engine.set_hosts(False)
    with Group([0], kind="nccl") as g:
        _same_sites(g.aggregate(batch, cat), want)
        g.set_hosts(True)
        got = g.aggregate(batch, cat)
    _same_sites(got, want_h)
    _same_hosts(got, want_h)


def test_nccl_per_process_comm_with_graph_replay(engine):
    """ncclCommInitRank at world size 1 on a fresh engine; repeated calls on
    one device batch capture the collectives into the CUDA graph and replay
    it (calls 2 and 3+), each result identical to the plain engine's."""
    from paper_1108_1785_b200 import Engine
    cat, cols, batch = _setup("D3", 2_000_000)
    dev = batch.to_device("cuda:0")
    want = engine.aggregate(dev, cat)
    with Engine(0) as e:
        e.comm_init(1, 0, Engine.comm_unique_id())
        assert e.comm_size() == 1
        k0 = e.timing()["kernel_launches"]
        for _ in range(4):
            _same_sites(e.aggregate(dev, cat), want)
        assert e.timing()["kernel_launches"] > k0
        e.comm_destroy()
        assert e.comm_size() == 1
        _same_sites(e.aggregate(dev, cat), want)


def test_comm_rejects_manual_prepare(engine):
    from paper_1108_1785_b200 import Engine, GnmError
    cat, cols, batch = _setup("D1", 1000)
    with Engine(0) as e:
        e.comm_init(1, 0, Engine.comm_unique_id())
        e.accumulate(batch, cat)
        with pytest.raises(GnmError):
            e.prepare_median(cat)
        e.reset()


def test_failed_rank_aborts_the_group_instead_of_hanging():
    """One loopback rank fails between its accumulation and the combine
    (GNM_TEST_FAIL_RANK): the other rank's collective is aborted, the call
    returns an error promptly, and the group refuses further work."""
    import os
    import subprocess
    import sys
    prog = (
        "import sys; sys.path.insert(0, '.')\n"
        "from paper_1108_1785_b200 import Group, GnmError, FlowBatch, SiteCatalog, synth\n"
        "w = synth.workload('D1'); cat = SiteCatalog(); w.sites.register(cat)\n"
        "b = FlowBatch(*synth.generate(w, 20000))\n"
        "g = Group([0, 0], kind='loopback')\n"
        "try:\n"
        "    g.aggregate(b, cat); print('NO ERROR')\n"
        "except GnmError as e:\n"
        "    print('FIRST', e.status, str(e)[:120])\n"
        "try:\n"
        "    g.aggregate(b, cat); print('NO ERROR 2')\n"
        "except GnmError as e:\n"
        "    print('SECOND', e.status, str(e)[:120])\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", prog], cwd=root, capture_output=True, text=True, timeout=120,
                         env=dict(os.environ, GNM_TEST_FAIL_RANK="1"))
    assert "FIRST" in out.stdout and "injected failure" in out.stdout, out.stdout + out.stderr
    assert "SECOND 13" in out.stdout, out.stdout + out.stderr

"""The reference's specification examples and the
toolkit scenario checks (toolkit_test.cpp:98-131), re-expressed: on the CPU
oracle and the host-side warning rule (CPU), and through the sm_100a path
(GPU). SPEC paths are relative to /root/reference, the tests to
/root/reference/proj/tests."""
import numpy as np
import pytest

import parity
from paper_1108_1785_b200 import (AnalysisResult, FilterParams, FlowBatch, RateStats, SiteCatalog,
                                  WarningState, evaluate_warnings)

IP = lambda a, b, c, d: (a << 24) | (b << 16) | (c << 8) | d  # noqa: E731
SITE_A, SITE_B = ["10.1.2.0/24"], ["10.9.0.0/24"]


def _catalog():
    cat = SiteCatalog()
    cat.register_site("SiteA", SITE_A)
    cat.register_site("SiteB", SITE_B)
    return cat


def _flows(rows, end=10_000_000):
    """rows: (src, dst, pkts, octets, duration_ms)."""
    src, dst, pkts, octs, dur = (np.array(c) for c in zip(*rows))
    return parity.make_cols(src.astype(np.uint32), dst.astype(np.uint32), pkts, octs, dur, end=end)


# classify: PureAck, then Administrative, then attribution.
CLASSIFY = [((IP(10, 1, 2, 3), IP(8, 8, 8, 8), 100, 4000, 1000), 1),             # avg 40 B -> PureAck
            ((IP(10, 1, 2, 3), IP(8, 8, 8, 8), 5, 4000, 50), 2),                 # 5 pkts, 50 ms -> Admin
            ((IP(10, 1, 2, 3), IP(8, 8, 8, 8), 10**6, 1_400_000_000, 10**4), 0)]  # bulk -> Forward
# attribute: src first; host = the matched address.
ATTRIBUTE = [((IP(10, 1, 2, 3), IP(8, 8, 8, 8)), (0, IP(10, 1, 2, 3))),
             ((IP(7, 7, 7, 7), IP(8, 8, 8, 8)), None),
             ((IP(10, 1, 2, 3), IP(10, 9, 0, 1)), (0, IP(10, 1, 2, 3)))]
# flow_rate and bucket_index (:271-278).
RATES = [(1_000_000, 8000, 1_000_000.0), (125_000_000, 1000, 1e9)]
BUCKETS = [(0.0, 0), (9_999.0, 0), (10_000.0, 1), (1e8, 10000), (99_995_000.0, 9999)]


def _oracle_catalog(orc):
    p, s = _catalog().entries_arrays()
    return orc.catalog(p, s)


def test_spec_scalar_examples_on_oracle(orc):
    oc = _oracle_catalog(orc)
    for row, cls in CLASSIFY:
        assert orc.classify(_flows([row]), oc)[0] >> 30 == cls
    for (src, dst), want in ATTRIBUTE:
        got = orc.classify(_flows([(src, dst, 100, 1_000_000, 2000)]), oc)[0]
        if want is None:
            assert got >> 30 == 3
        else:
            assert got >> 30 == 0 and got & 0x3FFFFFFF == want[0]
    for oct_, dur, rate in RATES:
        assert orc.flow_rate(oct_, dur) == rate
    for rate, b in BUCKETS:
        assert orc.bucket_index(rate) == b
    # median_from_histogram
    h = np.zeros(10001, np.uint32)
    h[200] = 1
    assert orc.median_bps(h, 1) == 2_005_000.0
    h[:] = 0
    h[0], h[500] = 3, 2
    assert orc.median_bps(h, 5) == 5_000.0
    h[:] = 0
    h[10000] = 7
    assert orc.median_bps(h, 7) == 100_000_000.0


def _result_with_median(median):
    return AnalysisResult.from_site_stats(2, {0: RateStats(median_bps=median, min_bps=median, max_bps=median,
                                                           avg_bps=median, flow_count=10)})


def test_spec_warning_examples_host_rule():
    """evaluate_warnings and detection latency (:367-373)."""
    cat = _catalog()
    ws = WarningState()
    assert evaluate_warnings(_result_with_median(900_000), cat, ws) == []
    w = evaluate_warnings(_result_with_median(900_000), cat, ws)
    assert [x.site for x in w] == [0] and w[0].consecutive_bad_hours == 2
    for _ in range(3):
        evaluate_warnings(_result_with_median(500_000), cat, ws)
    assert ws.streak(0) == 5
    assert evaluate_warnings(_result_with_median(50_000_000), cat, ws) == [] and ws.streak(0) == 0
    evaluate_warnings(_result_with_median(500_000), cat, ws)
    assert evaluate_warnings(_result_with_median(1_000_000), cat, ws) == [] and ws.streak(0) == 0  # strict <
    for hours, warnings in ((2, 1), (4, 3), (1, 0)):
        ws = WarningState()
        n = 0
        for h in range(hours + 2):
            bad = 1 <= h <= hours
            n += len(evaluate_warnings(_result_with_median(500_000 if bad else 5_000_000), cat, ws))
        assert n == warnings, (hours, n)


@pytest.mark.gpu
def test_spec_examples_on_gpu(engine):
    cat = _catalog()
    got = engine.classify(FlowBatch(*_flows([r for r, _ in CLASSIFY])), cat, FilterParams())
    assert [int(x) >> 30 for x in got] == [c for _, c in CLASSIFY]
    rows = [(s, d, 100, 1_000_000, 2000) for (s, d), _ in ATTRIBUTE]
    got = engine.classify(FlowBatch(*_flows(rows)), cat, FilterParams())
    for g, (_, want) in zip(got, ATTRIBUTE):
        assert (int(g) >> 30 == 3) if want is None else (int(g) >> 30 == 0 and int(g) & 0x3FFFFFFF == want[0])
    # rates: a site holding one flow reports it as min = max (exact f64)
    for oct_, dur, rate in RATES:
        res = engine.aggregate(FlowBatch(*_flows([(IP(10, 1, 2, 3), 1, 100, oct_, dur)])), cat,
                               FilterParams(min_packets=1))
        assert res.sites[0].stats.min_bps == rate == res.sites[0].stats.max_bps
    # buckets: octets over 8000 ms give rate = octets bps exactly
    for rate, b in BUCKETS[1:]:
        res = engine.aggregate(FlowBatch(*_flows([(IP(10, 1, 2, 3), 1, 20, int(rate), 8000)])), cat,
                               histograms=True)
        assert int(np.nonzero(res.histograms[0])[0][0]) == b
    # medians, clamped into [min, max] by stats_from
    res = engine.aggregate(FlowBatch(*_flows([(IP(10, 1, 2, 3), 1, 20, 2_000_000, 8000)])), cat)
    assert res.sites[0].stats.median_bps == 2_000_000.0  # 2,005,000 clamped to max
    rows = [(IP(10, 1, 2, 3), 1, 20, 5_000, 8000)] * 3 + [(IP(10, 1, 2, 3), 1, 20, 5_005_000, 8000)] * 2
    assert engine.aggregate(FlowBatch(*_flows(rows)), cat).sites[0].stats.median_bps == 5_000.0
    rows = [(IP(10, 1, 2, 3), 1, 20, 150_000_000 + i, 8000) for i in range(3)]
    st = engine.aggregate(FlowBatch(*_flows(rows)), cat).sites[0].stats
    assert st.median_bps == st.min_bps == 150_000_000.0  # 1e8 cap clamped up to min


@pytest.mark.gpu
def test_toolkit_small_scenario_on_gpu(engine, ref):
    """toolkit_test.cpp:98-131: the reference's generator, 1 h of SiteA
    (10.1.1.0/24, 4 hosts, fixed 2 Mbps, 1000 flows, 25% ack, 10% admin),
    seed 42: 250 / 100 / 650 / 0 tallies, every Forward flow at exactly
    2 Mbps in bucket 200."""
    rec = ref.generate([{"cidr": "10.1.1.0/24", "hosts": 4, "fixed_bps": 2_000_000.0, "flows_per_hour": 1000,
                         "ack": 0.25, "admin": 0.10}], duration_hours=1, seed=42)
    cols = ref.record_columns(rec)
    cat = SiteCatalog()
    cat.register_site("SiteA", ["10.1.1.0/24"])
    res = engine.aggregate(FlowBatch(*cols), cat, histograms=True)
    t = res.tallies
    assert (t.pure_ack, t.administrative, t.forward, t.unmatched) == (250, 100, 650, 0)
    st = res.sites[0].stats
    assert st.min_bps == st.max_bps == st.median_bps == 2_000_000.0 and st.flow_count == 650
    assert res.histograms[0][200] == 650

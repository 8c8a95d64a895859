"""GPU parity against the golden fixtures produced by the unmodified
reference (tests/golden/): bit-exact per-site counts, byte and micro-bps
sums, min/max/avg/median, histograms, tallies and per-record class/site,
through every input path of the C-ABI (host SoA, device SoA, host AoS), and
the criterion-7 warning scenarios end to end."""
import numpy as np
import pytest
import torch

import golden_io as G
import parity
from paper_1108_1785_b200 import (FilterParams, FlowBatch, FlowRecords, SiteCatalog, WarningState,
                                  evaluate_warnings, synth)

pytestmark = pytest.mark.gpu


def catalog(z):
    cat = SiteCatalog()
    for i, c in enumerate(G.sites(z)):
        cat.register_site(f"site{i}", c)
    return cat


def to_acc(res):
    t = res.table
    return {"count": t["flow_count"], "octets": t["octets"], "ubps_lo": t["rate_ubps_lo"],
            "ubps_hi": t["rate_ubps_hi"], "min": t["min_bps"], "max": t["max_bps"],
            "avg": t["avg_bps"], "median": t["median_bps"], "hist": res.histograms,
            "tallies": np.array([res.tallies.forward, res.tallies.pure_ack,
                                 res.tallies.administrative, res.tallies.unmatched], np.uint64)}


@pytest.mark.parametrize("path", ["host_soa", "device_soa", "host_aos"])
@pytest.mark.parametrize("name", G.ANALYSIS_SETS)
def test_gpu_reproduces_reference_fixture(engine, name, path):
    z = G.load(name)
    cat = catalog(z)
    ack, minp, mind = G.params(z)
    params = FilterParams(ack, minp, mind)
    cols = G.cols(z)
    if path == "host_soa":
        batch = FlowBatch(*cols)
    elif path == "device_soa":
        batch = FlowBatch(*cols).to_device()
    else:
        batch = FlowRecords(synth.to_aos(cols))
    res = engine.aggregate(batch, cat, params, histograms=True)
    G.assert_acc_equal(to_acc(res), G.expected(z))
    assert set(res.sites) == set(np.nonzero(z["count"])[0].tolist())


@pytest.mark.parametrize("name", G.ANALYSIS_SETS)
def test_gpu_classification_matches_reference(engine, name):
    z = G.load(name)
    ack, minp, mind = G.params(z)
    got = engine.classify(FlowBatch(*G.cols(z)), catalog(z), FilterParams(ack, minp, mind))
    np.testing.assert_array_equal(got, z["assign"])


def test_gpu_warning_scenarios_match_reference(engine):
    """acceptance.cpp:367-418 (criterion 7): windows cut like
    FlowStore::snapshot (end_ms in [start, end)), analysed on the GPU, the
    streak rule on the host: warning hours must equal the reference's."""
    z = np.load(G.GOLDEN + "/warnings.npz")
    base, hour = int(z["base"]), int(z["hour"])
    for name in ("two", "one", "four"):
        c = z[f"{name}_cols"]
        cat = SiteCatalog()
        cat.register_site("SiteA", ["10.1.1.0/24"])
        st = WarningState()
        hours = []
        for h in range(len(z[f"{name}_rates"])):
            s0, s1 = base + h * hour, base + (h + 1) * hour
            m = (c[5] >= s0) & (c[5] < s1)
            cols = [np.ascontiguousarray(c[i][m].astype(np.uint32 if i < 4 else np.uint64))
                    for i in range(6)]
            res = engine.aggregate(FlowBatch(*cols), cat, window_start_ms=s0, window_end_ms=s1)
            assert res.window_start_ms == s0 and res.window_end_ms == s1
            assert res.sites[0].stats.median_bps == z[f"{name}_medians"][h]
            if evaluate_warnings(res, cat, st):
                hours.append(h)
        assert hours == z[f"{name}_warn_hours"].tolist()


def test_device_partials_zero_copy_views(engine):
    """gnm_get_partials exposes the accumulation for a cross-GPU all-reduce;
    reducing the view with itself (x2) doubles every count/sum, as two equal
    ranks would."""
    sites, cols = parity.engine_stress_set(20_000, seed=5)
    cat = SiteCatalog()
    for i, c in enumerate(sites):
        cat.register_site(f"s{i}", c)
    single = engine.aggregate(FlowBatch(*cols), cat)
    engine.accumulate(FlowBatch(*cols).to_device(), cat)
    t = engine.device_tensors(cat)
    torch.cuda.synchronize()  # K2 ran on the engine's stream
    t["sums"].mul_(2)          # round 1 of two equal ranks
    t["coarse"].mul_(2)
    torch.cuda.synchronize()
    engine.prepare_median(cat)
    torch.cuda.synchronize()
    t["fine"].mul_(2)          # round 2
    torch.cuda.synchronize()
    doubled = engine.finalize(cat)
    np.testing.assert_array_equal(doubled.table["flow_count"], 2 * single.table["flow_count"])
    np.testing.assert_array_equal(doubled.table["octets"], 2 * single.table["octets"])
    np.testing.assert_array_equal(doubled.table["min_bps"], single.table["min_bps"])
    assert doubled.tallies.forward == 2 * single.tallies.forward
    # the lower median of a doubled multiset is the same element
    np.testing.assert_array_equal(doubled.table["median_bps"], single.table["median_bps"])

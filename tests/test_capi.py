"""The C-ABI boundary without a GPU: the library loads, exports every symbol
include/gnetmon.h declares, fails loudly (no CPU fallback) when no device is
present, and its host-side warning rule matches monitor_test.cpp."""
import ctypes as C
import os
import re

import numpy as np
import pytest
import torch

from paper_1108_1785_b200 import _lib
from paper_1108_1785_b200.flowmon import (AnalysisResult, FilterParams, GnmError, RateStats,
                                          SiteCatalog, WarningState, evaluate_warnings)

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include",
                      "gnetmon.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gnm_[a-z0-9_]+)\s*\(", text)))


def test_header_and_binding_agree():
    decl = declared_functions()
    assert decl, "no functions parsed from gnetmon.h"
    assert sorted(_lib.SYMBOLS) == decl


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(_lib.LIB_PATH)
    for name in declared_functions():
        assert hasattr(lib, name), name


def test_abi_version_and_defaults():
    assert _lib.lib.gnm_abi_version() == 4
    p = _lib.gnm_filter_params()
    _lib.lib.gnm_filter_params_default(C.byref(p))
    assert (p.ack_avg_size_max, p.min_packets, p.min_duration_ms, p.workers) == (96, 20, 100, 1)
    assert FilterParams() == FilterParams(96, 20, 100, 1)


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure mode")
def test_no_device_fails_loudly():
    from paper_1108_1785_b200 import Engine
    with pytest.raises(GnmError) as e:
        Engine(0)
    assert e.value.status == _lib.ERR_NO_DEVICE
    assert "no CPU fallback" in str(e.value)


def result_with_median(n_sites, site, median, flows):
    """monitor_test.cpp:23-47 result_with_median."""
    return AnalysisResult.from_site_stats(n_sites, {site: RateStats(median_bps=median,
                                                                    flow_count=flows)})


def one_site():
    c = SiteCatalog()
    c.register_site("SiteA", ["10.1.1.0/24"])
    return c


def test_streak_below_threshold_twice_warns():
    cat, st = one_site(), WarningState()
    bad = result_with_median(1, 0, 500_000.0, 10)
    good = result_with_median(1, 0, 5_000_000.0, 10)
    assert evaluate_warnings(bad, cat, st) == [] and st.streak(0) == 1
    w = evaluate_warnings(bad, cat, st)
    assert len(w) == 1 and w[0].site == 0 and w[0].site_name == "SiteA"
    assert w[0].median_bps == 500_000.0 and w[0].consecutive_bad_hours == 2
    w = evaluate_warnings(bad, cat, st)
    assert len(w) == 1 and w[0].consecutive_bad_hours == 3
    assert evaluate_warnings(good, cat, st) == [] and st.streak(0) == 0
    assert evaluate_warnings(bad, cat, st) == [] and st.streak(0) == 1


def test_threshold_is_strict():
    cat, st = one_site(), WarningState()
    evaluate_warnings(result_with_median(1, 0, 999_999.0, 5), cat, st)
    assert st.streak(0) == 1
    evaluate_warnings(result_with_median(1, 0, 1_000_000.0, 5), cat, st)
    assert st.streak(0) == 0


@pytest.mark.parametrize("idle", ["absent", "zero_flows"])
def test_zero_flow_hours_freeze_streak(idle):
    cat, st = one_site(), WarningState()
    bad = result_with_median(1, 0, 200_000.0, 8)
    evaluate_warnings(bad, cat, st)
    assert st.streak(0) == 1
    idle_res = AnalysisResult() if idle == "absent" else result_with_median(1, 0, 0.0, 0)
    assert evaluate_warnings(idle_res, cat, st) == [] and st.streak(0) == 1
    w = evaluate_warnings(bad, cat, st)
    assert len(w) == 1 and w[0].consecutive_bad_hours == 2


def test_streaks_are_per_site():
    cat = SiteCatalog()
    cat.register_site("SiteA", ["10.1.1.0/24"])
    cat.register_site("SiteB", ["10.2.2.0/24"])
    st = WarningState()
    mixed = AnalysisResult.from_site_stats(2, {0: RateStats(median_bps=100_000.0, flow_count=4),
                                               1: RateStats(median_bps=9_000_000.0, flow_count=4)})
    evaluate_warnings(mixed, cat, st)
    evaluate_warnings(mixed, cat, st)
    w = evaluate_warnings(mixed, cat, st)
    assert len(w) == 1 and w[0].site_name == "SiteA" and st.streak(1) == 0


def test_warning_rule_matches_oracle_random(orc):
    rng = np.random.default_rng(9)
    n = 50
    cat = SiteCatalog()
    for i in range(n):
        cat.register_site(f"s{i}", [f"10.{i}.0.0/24"])
    st = WarningState()
    streak = np.zeros(n, np.uint32)
    for hour in range(30):
        count = rng.integers(0, 3, n).astype(np.uint64)
        med = rng.choice([5e5, 999_999.0, 1e6, 2e6], n)
        res = AnalysisResult.from_site_stats(n, {s: RateStats(median_bps=float(med[s]),
                                                              flow_count=int(count[s]))
                                                 for s in range(n)})
        got = {w.site for w in evaluate_warnings(res, cat, st)}
        want = set(np.nonzero(orc.evaluate_warnings(count, np.where(count > 0, med, 0.0),
                                                    streak))[0].tolist())
        assert got == want
        assert [st.streak(s) for s in range(n)] == streak.tolist()


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure mode")
def test_multi_gpu_group_fails_loudly_without_devices():
    """gnm_group_create (one context per device + a communicator clique)
    reports the missing device instead of falling back to the CPU."""
    from paper_1108_1785_b200 import Group
    for kind in ("nccl", "loopback"):
        with pytest.raises(GnmError) as e:
            Group([0, 0], kind=kind)
        assert e.value.status == _lib.ERR_NO_DEVICE


def test_multi_gpu_argument_validation():
    L = _lib.lib
    h = C.c_void_p()
    devs = (C.c_int * 2)(0, 0)
    assert L.gnm_group_create(devs, 0, _lib.GROUP_NCCL, C.byref(h)) == _lib.ERR_INVALID_ARGUMENT
    assert L.gnm_group_create(devs, 2, 7, C.byref(h)) == _lib.ERR_INVALID_ARGUMENT
    assert L.gnm_group_size(None) == 0 and L.gnm_group_ctx(None, 0) is None
    assert L.gnm_group_host_count(None) == 0
    assert L.gnm_ctx_comm_size(None) == 1
    assert L.gnm_ctx_comm_init(None, 1, 0, None) == _lib.ERR_INVALID_ARGUMENT
    assert L.gnm_group_analyze(None, None, None, None, None) == _lib.ERR_INVALID_ARGUMENT

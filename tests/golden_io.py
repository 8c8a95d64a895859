"""Loading helpers for the golden fixtures (tests/golden/, made by
tests/golden/make_golden.py from the unmodified reference)."""
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
ANALYSIS_SETS = ["engine_stress", "edge", "tiny_duration", "d1_small", "d2_small", "d3_small"]


def load(name):
    return np.load(os.path.join(GOLDEN, f"{name}.npz"))


def sites(z):
    return [s.split("|") for s in z["sites"].tolist()]


def cols(z):
    return tuple(np.ascontiguousarray(z[k]) for k in ("src", "dst", "pkts", "octets", "start", "end"))


def params(z):
    return tuple(int(x) for x in z["params"])


def dense_hist(z):
    n = len(z["count"])
    h = np.zeros((n, 10001), np.uint32)
    h[z["hist_site"], z["hist_bucket"]] = z["hist_count"]
    return h


def expected(z):
    """The reference's result in the oracle dict layout (Oracle.finalize)."""
    st = z["stats"]
    return {"count": z["count"], "octets": z["octet_sum"], "ubps_lo": z["ubps_lo"],
            "ubps_hi": z["ubps_hi"], "min": st[:, 0], "max": st[:, 1], "avg": st[:, 2],
            "median": st[:, 3], "hist": dense_hist(z), "tallies": z["tallies"]}


def assert_acc_equal(got, want, check_hist=True):
    """Bit-exact comparison of two result dicts (oracle layout)."""
    pres = want["count"] > 0
    np.testing.assert_array_equal(got["count"], want["count"])
    np.testing.assert_array_equal(got["octets"], want["octets"])
    np.testing.assert_array_equal(got["ubps_lo"], want["ubps_lo"])
    np.testing.assert_array_equal(got["ubps_hi"], want["ubps_hi"])
    for k in ("min", "max", "avg", "median"):
        np.testing.assert_array_equal(np.asarray(got[k])[pres].view(np.uint64),
                                      np.asarray(want[k])[pres].view(np.uint64), err_msg=k)
    np.testing.assert_array_equal(np.asarray(got["tallies"], np.uint64), want["tallies"])
    if check_hist:
        np.testing.assert_array_equal(got["hist"], want["hist"])


def hosts_expected(name):
    """The reference's SiteResult::hosts rows for an analysis fixture
    (hosts.npz, make_golden.py hosts_fixture), in (site, host) order."""
    z = np.load(os.path.join(GOLDEN, "hosts.npz"))
    st = z[f"{name}_stats"]
    n = len(st)
    rows, bks, cnts = z[f"{name}_hist_row"], z[f"{name}_hist_bucket"], z[f"{name}_hist_count"]
    return {"site": z[f"{name}_site"], "host": z[f"{name}_host"], "count": z[f"{name}_count"],
            "min": st[:, 0], "max": st[:, 1], "avg": st[:, 2], "median": st[:, 3], "sum_bps": st[:, 4],
            "hist_row": rows, "hist_bucket": bks, "hist_count": cnts, "n": n}


def dense_host_hist(h):
    d = np.zeros((len(h["count"]), 10001), np.uint32)
    d[h["hist_row"], h["hist_bucket"]] = h["hist_count"]
    return d


def assert_hosts_equal(got, want, check_hist=True):
    """Bit-exact comparison of per-host rows (dict layout of Oracle.host_stats)."""
    for k in ("site", "host", "count"):
        np.testing.assert_array_equal(np.asarray(got[k]).astype(np.uint64),
                                      np.asarray(want[k]).astype(np.uint64), err_msg=k)
    for k in ("min", "max", "avg", "median"):
        np.testing.assert_array_equal(np.asarray(got[k], np.float64).view(np.uint64),
                                      np.asarray(want[k], np.float64).view(np.uint64), err_msg=k)
    if "sum_bps" in want and "ubps_lo" in got:
        sb = [float(int(h) << 64 | int(lo)) / 1e6 for lo, h in zip(got["ubps_lo"], got["ubps_hi"])]
        np.testing.assert_array_equal(np.array(sb).view(np.uint64),
                                      np.asarray(want["sum_bps"]).view(np.uint64), err_msg="sum_bps")
    if check_hist:
        np.testing.assert_array_equal(got["hist"] if "hist" in got else dense_host_hist(got),
                                      dense_host_hist(want))

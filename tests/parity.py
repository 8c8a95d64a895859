"""Shared parity helpers: workloads mirroring the reference's own tests and
the exact comparison of a GPU result with the CPU oracle."""
from __future__ import annotations

import numpy as np

U32 = 2**32


def make_cols(src, dst, pkts, octets, dur, end=1_000_000):
    """engine_test.cpp:16-27 make_flow, vectorised: start = end - duration (u64 wrap)."""
    n = len(src)
    end = np.broadcast_to(np.asarray(end, np.uint64), (n,)).copy()
    dur = np.asarray(dur, np.uint64)
    start = end - dur
    return (np.asarray(src, np.uint32), np.asarray(dst, np.uint32), np.asarray(pkts, np.uint32),
            np.asarray(octets, np.uint32), start, end)


def engine_stress_set(n: int = 50_000, seed: int = 37):
    """engine_test.cpp:232-248 shape: 3/4 of sources in SiteA 10.1.2.0/24 or
    SiteB 10.9.0.0/22, full-range u32 octets (hits the u128 path and
    octets<pkts), pkts 1..5000, durations 1..20000 ms."""
    rng = np.random.default_rng(seed)
    host = np.where(rng.integers(0, 2, n) == 0, 0x0A010200,
                    0x0A090000 + 256 * rng.integers(0, 4, n)) + rng.integers(1, 255, n)
    registered = rng.integers(0, 4, n) != 0
    src = np.where(registered, host, rng.integers(0, U32, n))
    dst = rng.integers(0, U32, n)
    cols = make_cols(src, dst, rng.integers(1, 5001, n), rng.integers(0, U32, n),
                     rng.integers(1, 20001, n), end=2_000_000_000)
    return [["10.1.2.0/24"], ["10.9.0.0/22"]], cols


def edge_set():
    """Hand-built edge cases of SURVEY.md §8(a'): zero packets, octets <
    pkts, end < start (u64 wrap), zero and tiny durations, the u128 ubps
    product and quotient, bucket boundaries, the overflow bucket, src-first
    attribution, unregistered endpoints, /26 round-up, top /24 of the space,
    a /16 site (uniform radix node) and a mixed /16."""
    sites = [["10.1.2.128/26"], ["10.9.0.0/22"], ["172.16.0.0/16"], ["255.255.255.0/24"],
             ["10.1.3.0/24"]]
    A, B, C16, TOP, D = 0x0A010205, 0x0A090101, 0xAC10FFFE, 0xFFFFFF01, 0x0A0103FE
    R = 0xC6336401  # unregistered
    rows = [
        # src, dst, pkts, octets, duration
        (A, R, 0, 100000, 1000),            # d_pkts == 0 -> Administrative
        (A, R, 5, 3, 1000),                  # octets < pkts -> PureAck
        (A, R, 100, 9700, 1000),             # exactly 97*pkts -> not ACK
        (A, R, 100, 9699, 1000),             # 96.99 avg -> ACK
        (A, R, 19, 100000, 1000),            # pkts < 20 -> Admin
        (A, R, 20, 100000, 99),              # dur < 100 -> Admin
        (A, R, 20, 100000, 100),             # dur == 100 -> Forward
        (A, R, 20, 100000, 0),               # dur == 0 -> Admin
        (R, B, 1000, 2**32 - 1, 1000),       # u128 product branch, dst attribution
        (R, B, 1000, 2305843009, 1000),      # last u64-product octets
        (R, B, 1000, 2305843010, 1000),      # first u128-product octets
        (C16, R, 1000, 125_000_000, 1000),   # 1e9 bps -> overflow bucket
        (C16, R, 100, 1_000_000, 8000),      # exactly 1 Mbps -> bucket 100
        (C16, R, 100, 12_500, 10),           # 10 kbps * 1000 boundary at dur 10
        (C16, R, 1000, 12_499_375, 1000),    # 99,995,000 bps -> bucket 9999
        (TOP, R, 1000, 10_000_000, 1000),    # top /24
        (A, D, 1000, 10_000_000, 2000),      # both registered: src wins
        (D, A, 1000, 10_000_000, 2000),      # both registered: src wins (other way)
        (R, R, 1000, 10_000_000, 2000),      # unmatched
        (0x0A010201, R, 1000, 10_000_000, 2000),  # 10.1.2.1 (below /26 but same /24)
        (0x0A0101FF, R, 1000, 10_000_000, 2000),  # 10.1.1.255 unregistered neighbour
        (0x0A090400, R, 1000, 10_000_000, 2000),  # 10.9.4.0 just past the /22
        (0x0A08FFFF, R, 1000, 10_000_000, 2000),  # 10.8.255.255 just before the /22
        (D, R, 1000, 80_000, 8000),          # 10 kbps -> bucket 1
        (D, R, 1000, 79_999, 8000),          # just under -> bucket 0
    ]
    src, dst, pkts, octs, dur = (np.array(c) for c in zip(*rows))
    cols = list(make_cols(src, dst, pkts, octs, dur, end=10_000_000))
    # end < start: the u64 duration wraps to a huge value (passes the filters).
    wrap = make_cols([A], [R], [1000], [10_000_000], [0], end=5_000)
    wrap[4][0] = np.uint64(6_000)  # start > end
    for i in range(6):
        cols[i] = np.concatenate([cols[i], wrap[i]])
    return sites, tuple(cols)


def tiny_duration_set(n: int = 4000, seed: int = 5):
    """min_duration_ms = 0 exercises dur = 1 ms with full-range octets, whose
    micro-bps QUOTIENT exceeds 2^64 (the third limb)."""
    rng = np.random.default_rng(seed)
    src = 0x0A010200 + rng.integers(1, 255, n)
    cols = make_cols(src, rng.integers(0, U32, n), rng.integers(1, 100, n),
                     rng.integers(2**31, U32, n), rng.integers(1, 4, n), end=2_000_000)
    return [["10.1.2.0/24"]], cols


def oracle_reference(orc, catalog, cols, params=(96, 20, 100)):
    p, s = catalog.entries_arrays()
    oc = orc.catalog(p, s)
    return orc.analyze(cols, oc, catalog.site_count(), params)


def assert_matches_oracle(result, acc, threshold=1e6, check_hist=True):
    """Bit-exact comparison of an AnalysisResult with the oracle."""
    t = result.table
    n = len(acc["count"])
    assert len(t) == n
    np.testing.assert_array_equal(t["flow_count"], acc["count"], err_msg="flow counts")
    np.testing.assert_array_equal(t["octets"], acc["octets"], err_msg="byte sums")
    np.testing.assert_array_equal(t["rate_ubps_lo"], acc["ubps_lo"], err_msg="ubps sum lo")
    np.testing.assert_array_equal(t["rate_ubps_hi"], acc["ubps_hi"], err_msg="ubps sum hi")
    pres = acc["count"] > 0
    for k_gpu, k_orc in (("min_bps", "min"), ("max_bps", "max"), ("avg_bps", "avg"),
                         ("median_bps", "median")):
        np.testing.assert_array_equal(t[k_gpu][pres].view(np.uint64),
                                      np.asarray(acc[k_orc])[pres].view(np.uint64),
                                      err_msg=k_gpu)
    np.testing.assert_array_equal(t["below_threshold"][pres].astype(bool),
                                  np.asarray(acc["median"])[pres] < threshold)
    assert not t["flow_count"][~pres].any()
    tl = result.tallies
    assert [tl.forward, tl.pure_ack, tl.administrative, tl.unmatched] == acc["tallies"].tolist()
    assert set(result.sites) == set(np.nonzero(pres)[0].tolist())
    if check_hist and result.histograms is not None:
        np.testing.assert_array_equal(result.histograms, acc["hist"], err_msg="histograms")

"""Pin the CPU oracle (oracle/gnm_oracle.c) to the reference: every golden
fixture produced by the unmodified reference must be reproduced bit-exactly,
plus the reference's own known answers (engine_test.cpp, acceptance.cpp)."""
import numpy as np
import pytest

import golden_io as G


@pytest.mark.parametrize("name", G.ANALYSIS_SETS)
def test_oracle_reproduces_reference_fixture(orc, name):
    z = G.load(name)
    sites = G.sites(z)
    # The oracle's catalog is the reference's hash table over the (prefix24,
    # site) entries in registration order (site_catalog.cpp:90-148).
    prefixes, owners = [], []
    from paper_1108_1785_b200 import Cidr
    for sid, cl in enumerate(sites):
        for text in cl:
            c = Cidr.parse(text)
            p = c.first_prefix24()
            while p <= c.last_prefix24():
                prefixes.append(p)
                owners.append(sid)
                p += 256
    oc = orc.catalog(np.array(prefixes, np.uint32), np.array(owners, np.uint32))
    got = orc.finalize(orc.aggregate(G.cols(z), oc, len(sites), G.params(z)))
    G.assert_acc_equal(got, G.expected(z))
    np.testing.assert_array_equal(orc.classify(G.cols(z), oc, G.params(z)), z["assign"])


def test_oracle_scalars_match_reference(orc):
    z = G.load("scalars")
    for i in range(0, len(z["octets"]), 7):
        o, d = int(z["octets"][i]), int(z["durations"][i])
        r = orc.flow_rate(o, d)
        assert np.float64(r).view(np.uint64) == np.float64(z["rate"][i]).view(np.uint64)
        assert orc.rate_ubps(o, d) == int(z["ubps_hi"][i]) << 64 | int(z["ubps_lo"][i])
        assert orc.bucket_index(r) == z["bucket"][i]
    for r, b in zip(z["probe_rates"], z["probe_bucket"]):
        assert orc.bucket_index(float(r)) == b
    off = 0
    for n, want in zip(z["median_lens"], z["median"]):
        rates = z["median_rates"][off:off + n]
        off += n
        row = np.zeros(10001, np.uint32)
        for r in rates:
            row[orc.bucket_index(float(r))] += 1
        assert orc.median_bps(row, int(n)) == want


def test_engine_test_known_answers(orc):
    """engine_test.cpp:121-208 known answers on the restatement."""
    assert orc.flow_rate(1_000_000, 8000) == 1_000_000.0
    assert orc.flow_rate(125_000_000, 1000) == 1e9
    for rate, b in ((0, 0), (9_999, 0), (10_000, 1), (99_995_000, 9999), (100_000_000, 10000),
                    (5e9, 10000)):
        assert orc.bucket_index(rate) == b
    for n in (0, 1, 17, 9999):
        assert orc.bucket_index(n * 10_000.0) == n
        assert orc.bucket_index((n + 1) * 10_000.0 - 0.001) == n
    row = np.zeros(10001, np.uint32)
    row[200] = 1
    assert orc.median_bps(row, 1) == 2_005_000.0
    row[:] = 0
    row[0], row[500] = 3, 2
    assert orc.median_bps(row, 5) == 5_000.0
    row[:] = 0
    row[10000] = 7
    assert orc.median_bps(row, 7) == 1e8


def test_rational_rate_oracle(orc):
    """engine_test.cpp:127-143: rate within 1e-9 relative of the exact
    rational, micro-bps the truncated rational."""
    from fractions import Fraction
    rng = np.random.default_rng(23)
    for _ in range(2000):
        o = int(rng.integers(0, 2**32))
        d = int(rng.integers(1, 1_000_001))
        exact = Fraction(8000 * o, d)
        r = orc.flow_rate(o, d)
        assert abs(Fraction(r) - exact) <= exact * Fraction(1, 10**9) + Fraction(1, 10**12)
        assert orc.rate_ubps(o, d) == (8_000_000_000 * o) // d


def test_warning_scenarios_match_reference(orc):
    """acceptance.cpp:367-418 criterion 7 on the oracle's rule, windowed like
    FlowStore::snapshot (flow_store.cpp:75)."""
    z = np.load(G.GOLDEN + "/warnings.npz")
    base, hour = int(z["base"]), int(z["hour"])
    oc = orc.catalog(np.array([0x0A010100], np.uint32), np.array([0], np.uint32))
    for name in ("two", "one", "four"):
        c = z[f"{name}_cols"]
        streak = np.zeros(1, np.uint32)
        hours = []
        for h in range(len(z[f"{name}_rates"])):
            m = (c[5] >= base + h * hour) & (c[5] < base + (h + 1) * hour)
            cols = tuple(c[i][m].astype(np.uint32 if i < 4 else np.uint64) for i in range(6))
            acc = orc.finalize(orc.aggregate(cols, oc, 1))
            assert acc["median"][0] == z[f"{name}_medians"][h]
            if orc.evaluate_warnings(acc["count"], acc["median"], streak).any():
                hours.append(h)
        assert hours == z[f"{name}_warn_hours"].tolist()


def test_oracle_matches_live_reference_random(orc, ref):
    """Where oracle/_ref is built: random engine_test-shaped inputs."""
    import parity
    for seed in (1, 2, 3):
        sites, cols = parity.engine_stress_set(5000, seed=seed)
        rc = ref.catalog(sites)
        p, s = ref.entries(rc)
        got = orc.finalize(orc.aggregate(cols, orc.catalog(p, s), len(sites)))
        d = ref.result(ref.aggregate(ref.records(cols), rc))
        lo, hi, octs = ref.site_sums(ref.records(cols), rc, len(sites))
        assert got["tallies"].tolist() == d["tallies"].tolist()
        for sid, x in d["sites"].items():
            assert got["count"][sid] == x["count"]
            assert (got["min"][sid], got["max"][sid], got["avg"][sid], got["median"][sid]) == (
                x["min"], x["max"], x["avg"], x["median"])
            np.testing.assert_array_equal(got["hist"][sid], x["hist"])
        np.testing.assert_array_equal(got["ubps_lo"], lo)
        np.testing.assert_array_equal(got["ubps_hi"], hi)
        np.testing.assert_array_equal(got["octets"], octs)


def test_integer_bucket_identity():
    """K2 computes bucket_index (rate_engine.cpp:119-125) as
    min(10000, floor(ubps / 1e10)) from the exact micro-bps instead of
    dividing the f64 rate by 1e4 (kernels.cu, bucket_of_ubps). Check the
    identity against the reference's double arithmetic (numpy float64 is the
    same IEEE round-to-nearest division) on random and adversarial inputs:
    octets/durations placed within +-2 of every bucket boundary
    4*oct == 5*dur*k, where double rounding would bite if it could."""
    rng = np.random.default_rng(7)
    n = 400_000
    oct_ = rng.integers(0, 2**32, n, dtype=np.uint64)
    dur = np.concatenate([rng.integers(1, 20_000, n // 4), rng.integers(1, 10**8, n // 4),
                          rng.integers(1, 2**63, n // 4, dtype=np.int64),
                          (rng.integers(1, 2**62, n // 4, dtype=np.int64) >> rng.integers(0, 62, n // 4))
                          + 1]).astype(np.uint64)
    # adversarial: oct = floor(5*dur*k/4) + d, d in [-2, 2]
    m = 200_000
    ad = rng.integers(1, 10**7, m).astype(np.uint64)
    k = rng.integers(0, 10002, m).astype(np.uint64)
    ao = (5 * ad * k) // 4 + rng.integers(-2, 3, m).astype(np.int64).astype(np.uint64)
    keep = ao < 2**32
    oct_ = np.concatenate([oct_, ao[keep]])
    dur = np.concatenate([dur, ad[keep]])
    rate = 8000.0 * oct_.astype(np.float64) / dur.astype(np.float64)
    b = rate / 10000.0
    ref = np.where(b >= 10000.0, 10000, b.astype(np.uint64))
    # floor(oct * 8e9 / dur) / 1e10 == floor(4 * oct / (5 * dur)) (nested
    # floors); 4*oct < 2^34 and 5*dur may be up to 2^66, so use Python ints.
    num = (4 * oct_.astype(object))
    den = (5 * dur.astype(object))
    got = np.minimum(np.array(num // den, dtype=object), 10000).astype(np.uint64)
    bad = np.nonzero(got != ref)[0]
    assert bad.size == 0, (oct_[bad[:5]], dur[bad[:5]], ref[bad[:5]], got[bad[:5]])

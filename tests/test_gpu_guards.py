"""Regression tests for the round-2 guards:
* the wide-registry bucket column of the log keeps its own capacity: wide
  (>= 2^18 sites) small batch, then a narrow registry on a bigger batch
  (the entry column grows alone), then the wide registry on a bigger batch
  again -- results stay exact (oracle);
* device FlowRecord rows must be 8-byte aligned (a clean error, not a
  misaligned-address fault);
* an accumulation whose Forward flows could wrap the u32 coarse counts
  (>= 2^32) fails finalize loudly instead of returning a wrong median.
"""
import numpy as np
import pytest

import parity

pytestmark = pytest.mark.gpu


def _wide_catalog(n_sites=300_000, base=0x20000000):
    from paper_1108_1785_b200 import SiteCatalog
    cat = SiteCatalog()
    for i in range(n_sites):
        a = base + i * 256
        cat.register_site(f"w{i}", [f"{a >> 24}.{(a >> 16) & 255}.{(a >> 8) & 255}.0/24"])
    return cat


def _wide_cols(n, n_sites=300_000, base=0x20000000, seed=1):
    rng = np.random.default_rng(seed)
    site = rng.integers(0, n_sites, n)
    src = (base + site * 256 + rng.integers(0, 4, n)).astype(np.uint32)
    return parity.make_cols(src, rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32),
                            rng.integers(20, 400, n), rng.integers(40_000, 2**31, n), rng.integers(100, 9000, n),
                            end=2_000_000_000)


def test_log_bucket_column_capacity_across_registries(orc):
    from paper_1108_1785_b200 import Engine, FlowBatch, synth
    wide = _wide_catalog()
    narrow_w = synth.workload("D1")
    from paper_1108_1785_b200 import SiteCatalog
    narrow = SiteCatalog()
    narrow_w.sites.register(narrow)
    with Engine(0) as eng:
        eng.set_graphs(False)
        small = _wide_cols(50_000, seed=2)
        parity.assert_matches_oracle(eng.aggregate(FlowBatch(*small), wide), parity.oracle_reference(orc, wide, small),
                                     check_hist=False)
        big_narrow = synth.generate(narrow_w, 3_000_000)
        parity.assert_matches_oracle(eng.aggregate(FlowBatch(*big_narrow), narrow),
                                     parity.oracle_reference(orc, narrow, big_narrow), check_hist=False)
        big_wide = _wide_cols(2_000_000, seed=3)
        parity.assert_matches_oracle(eng.aggregate(FlowBatch(*big_wide), wide),
                                     parity.oracle_reference(orc, wide, big_wide), check_hist=False)


def test_misaligned_device_rows_rejected(engine):
    import torch
    from paper_1108_1785_b200 import FlowRecords, GnmError, SiteCatalog, synth, _lib
    w = synth.workload("D1")
    cat = SiteCatalog()
    w.sites.register(cat)
    rows = torch.from_numpy(synth.to_aos(synth.generate(w, 1000))).cuda()
    buf = torch.zeros(rows.numel() + 4, dtype=torch.uint8, device="cuda")
    buf[4:].copy_(rows)
    with pytest.raises(GnmError) as e:
        engine.aggregate(FlowRecords(buf[4:]), cat)
    assert e.value.status == _lib.ERR_INVALID_ARGUMENT and "aligned" in str(e.value)
    # the context is still usable, and aligned rows give the reference's answer
    res = engine.aggregate(FlowRecords(rows), cat)
    assert res.tallies.total() == 1000


def test_coarse_count_wrap_guard():
    from paper_1108_1785_b200 import Engine, FlowBatch, GnmError, SiteCatalog, synth, _lib
    w = synth.workload("D1")
    cat = SiteCatalog()
    w.sites.register(cat)
    cols = synth.generate(w, 10_000)
    with Engine(0) as eng:
        eng.accumulate(FlowBatch(*cols), cat)
        t = eng.device_tensors(cat)
        n = cat.site_count()
        t["sums"][4 * n] += 2**32  # the Forward tally as if 2^32 more flows had been seen
        with pytest.raises(GnmError) as e:
            eng.finalize(cat)
        assert e.value.status == _lib.ERR_CAPACITY
        # the next accumulation starts clean
        res = eng.aggregate(FlowBatch(*cols), cat)
        assert res.tallies.total() == 10_000

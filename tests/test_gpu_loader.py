"""The host-batch loader's duration compaction (non-windowed SoA batches send
end - start as u32, 20 bytes per record): bit-identical to the uncompacted
path (GNM_NO_COMPACT) and to the oracle, including chunks that must fall back
because a duration needs 64 bits (end < start wraps), pinned and pageable
inputs, several chunk sizes, per-host mode, and the bytes it reports."""
import os

import numpy as np
import pytest

import parity

pytestmark = pytest.mark.gpu


def _with_wraps(cols, every):
    """Every `every`-th record gets end < start (a u64-wrapped duration)."""
    src, dst, pkts, octs, start, end = (np.array(c, copy=True) for c in cols)
    idx = np.arange(0, len(src), every)
    start[idx] = end[idx] + 1000
    return src, dst, pkts, octs, start, end


@pytest.mark.parametrize("chunk", [1024, 65536, 1 << 22])
def test_compacted_loader_matches_uncompacted_and_oracle(engine, orc, chunk):
    import torch
    from paper_1108_1785_b200 import FlowBatch, SiteCatalog, synth
    w = synth.workload("D2")
    cols = _with_wraps(synth.generate(w, 300_000), 50_000)  # a few chunks fall back
    cat = SiteCatalog()
    w.sites.register(cat)
    engine.set_chunk_records(chunk)
    try:
        want = parity.oracle_reference(orc, cat, cols)
        got = engine.aggregate(FlowBatch(*cols), cat)  # pageable numpy
        parity.assert_matches_oracle(got, want, check_hist=False)
        pinned = [torch.from_numpy(c.view(np.int32 if c.dtype.itemsize == 4 else np.int64)).pin_memory()
                  for c in cols]
        views = [p.numpy().view(c.dtype) for p, c in zip(pinned, cols)]
        got_p = engine.aggregate(FlowBatch(*views), cat)
        np.testing.assert_array_equal(got_p.table, got.table)
        os.environ["GNM_NO_COMPACT"] = "1"
        try:
            plain = engine.aggregate(FlowBatch(*cols), cat)
        finally:
            del os.environ["GNM_NO_COMPACT"]
        np.testing.assert_array_equal(plain.table, got.table)
    finally:
        engine.set_chunk_records(1 << 22)


def test_compacted_loader_hosts_mode_and_bytes(engine):
    from paper_1108_1785_b200 import FlowBatch, SiteCatalog, synth
    w = synth.workload("D1")
    cols = synth.generate(w, 200_000)
    cat = SiteCatalog()
    w.sites.register(cat)
    dev = engine.aggregate(FlowBatch(*cols).to_device("cuda:0"), cat)
    b0 = engine.timing()["h2d_bytes"]
    host = engine.aggregate(FlowBatch(*cols), cat)
    assert engine.timing()["h2d_bytes"] - b0 == 200_000 * 20  # no wide durations in D1
    np.testing.assert_array_equal(host.table, dev.table)
    engine.set_hosts(True)
    try:
        hd = engine.aggregate(FlowBatch(*cols).to_device("cuda:0"), cat)
        hh = engine.aggregate(FlowBatch(*cols), cat)
    finally:
        engine.set_hosts(False)
    assert hh.host_table.tobytes() == hd.host_table.tobytes()
    # a snapshot window keeps the timestamps (no compaction)
    lo, hi = int(np.percentile(cols[5], 20)), int(np.percentile(cols[5], 80))
    b1 = engine.timing()["h2d_bytes"]
    wh = engine.aggregate_window(FlowBatch(*cols), cat, lo, hi)
    assert engine.timing()["h2d_bytes"] - b1 == 200_000 * 32
    wd = engine.aggregate_window(FlowBatch(*cols).to_device("cuda:0"), cat, lo, hi)
    np.testing.assert_array_equal(wh.table, wd.table)


@pytest.mark.parametrize("chunk", [4096, 1 << 22])
def test_compacted_aos_rows(engine, orc, chunk):
    """Host FlowRecord rows (the drop-in's std::vector): the loader gathers
    the 20 hot bytes per row on host threads; chunks with a wrapped duration
    send whole rows. Pageable and pinned rows, per-host mode."""
    import torch
    from paper_1108_1785_b200 import FlowRecords, SiteCatalog, synth
    w = synth.workload("D1")
    cols = _with_wraps(synth.generate(w, 120_000), 30_000)
    cat = SiteCatalog()
    w.sites.register(cat)
    rows = synth.to_aos(cols)
    engine.set_chunk_records(chunk)
    try:
        want = parity.oracle_reference(orc, cat, cols)
        got = engine.aggregate(FlowRecords(rows), cat)
        parity.assert_matches_oracle(got, want, check_hist=False)
        pinned = torch.from_numpy(rows).pin_memory()
        np.testing.assert_array_equal(engine.aggregate(FlowRecords(pinned.numpy()), cat).table, got.table)
        dev = engine.aggregate(FlowRecords(torch.from_numpy(rows).cuda()), cat)
        np.testing.assert_array_equal(dev.table, got.table)
        engine.set_hosts(True)
        try:
            hh = engine.aggregate(FlowRecords(rows), cat)
            hd = engine.aggregate(FlowRecords(torch.from_numpy(rows).cuda()), cat)
        finally:
            engine.set_hosts(False)
        assert hh.host_table.tobytes() == hd.host_table.tobytes()
    finally:
        engine.set_chunk_records(1 << 22)

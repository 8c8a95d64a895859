"""FLOWARC1 archives (flow_store.cpp:144-207): archives written by the
unmodified reference's FlowStore::write_archive are decoded on the GPU
byte-identically to its FlowStore::load, every ArchiveError kind maps to the
same error, and the in-place archive analysis (K2 reading big-endian entries)
equals the oracle on the decoded records."""
import os
import tempfile

import numpy as np
import pytest

import parity
from paper_1108_1785_b200 import ArchiveError, FlowRecords, SiteCatalog, synth


def _archive(ref, rows):
    fd, path = tempfile.mkstemp(suffix=".arc")
    os.close(fd)
    try:
        ref.write_archive(rows, path)
        with open(path, "rb") as f:
            return f.read()
    finally:
        os.unlink(path)


def _rows(n, seed=3):
    w = synth.workload("D2")
    cols = synth.generate(w, n)
    aos = synth.to_aos(cols).reshape(-1, 64).copy()
    rng = np.random.default_rng(seed)
    aos[:, 8:16] = rng.integers(0, 256, (n, 8), dtype=np.uint8)   # next_hop, ifs
    aos[:, 32:48] = rng.integers(0, 256, (n, 16), dtype=np.uint8)  # ports .. pad2
    return w, cols, aos


def _ref_load(ref, data):
    fd, path = tempfile.mkstemp(suffix=".arc")
    os.close(fd)
    try:
        with open(path, "wb") as f:
            f.write(data)
        return ref.load_archive(path)
    finally:
        os.unlink(path)


def test_reference_archive_round_trip(ref):
    _, _, rows = _rows(1000)
    data = _archive(ref, rows)
    assert data[:8] == b"FLOWARC1" and len(data) == 20 + 64 * 1000
    got, kind = _ref_load(ref, data)
    assert kind == -1 and got == rows.tobytes()


@pytest.mark.gpu
@pytest.mark.parametrize("on_device", [False, True])
def test_gpu_decode_archive_matches_reference(engine, ref, on_device):
    _, _, rows = _rows(50_000)
    data = _archive(ref, rows)
    want, _ = _ref_load(ref, data)
    arg = data
    if on_device:
        import torch
        arg = torch.from_numpy(np.frombuffer(data, np.uint8).copy()).cuda()
    got = engine.decode_archive(arg)
    assert got.tobytes() == want


@pytest.mark.gpu
def test_archive_errors_match_reference(engine, ref):
    _, _, rows = _rows(10)
    data = _archive(ref, rows)
    cases = {
        "BadMagic": b"FLOWARC2" + data[8:],
        "BadVersion": data[:8] + b"\x00\x00\x00\x02" + data[12:],
        "TruncatedArchive": data[:-1],
        "trailing": data + b"\x00",
        "header": data[:19],
    }
    kinds = ["BadMagic", "BadVersion", "TruncatedArchive", "IoFailure"]
    for name, bad in cases.items():
        rows_ref, kind = _ref_load(ref, bad)
        assert rows_ref is None
        with pytest.raises(ArchiveError) as e:
            engine.decode_archive(bad)
        assert e.value.kind == kinds[kind], name
    assert len(engine.decode_archive(_archive(ref, rows[:0]))) == 0


@pytest.mark.gpu
@pytest.mark.parametrize("on_device", [False, True])
def test_analyze_archive_in_place(engine, ref, orc, on_device):
    w, cols, rows = _rows(300_001)
    data = _archive(ref, rows)
    cat = SiteCatalog()
    w.sites.register(cat)
    arg = data
    if on_device:
        import torch
        arg = torch.from_numpy(np.frombuffer(data, np.uint8).copy()).cuda()
    got = engine.aggregate_archive(arg, cat, histograms=True)
    parity.assert_matches_oracle(got, parity.oracle_reference(orc, cat, cols))
    same = engine.aggregate(FlowRecords(rows.reshape(-1)), cat, histograms=True)
    np.testing.assert_array_equal(got.table, same.table)


@pytest.mark.gpu
@pytest.mark.parametrize("on_device", [False, True])
def test_analyze_archive_hosts_mode(engine, ref, orc, on_device):
    """Per-host rows from the in-place archive path (K2 layout 4, hosts mode)
    equal the oracle's SiteResult::hosts restatement on the same records."""
    w, cols, rows = _rows(200_003, seed=5)
    data = _archive(ref, rows)
    cat = SiteCatalog()
    w.sites.register(cat)
    arg = data
    if on_device:
        import torch
        arg = torch.from_numpy(np.frombuffer(data, np.uint8).copy()).cuda()
    engine.set_hosts(True)
    try:
        got = engine.aggregate_archive(arg, cat)
    finally:
        engine.reset()
        engine.set_hosts(False)
    p, s = cat.entries_arrays()
    want = orc.host_stats(cols, orc.catalog(p, s))
    t = got.host_table
    for k_got, k_want in (("site", "site"), ("host", "host"), ("flow_count", "count"),
                          ("rate_ubps_lo", "ubps_lo"), ("rate_ubps_hi", "ubps_hi")):
        np.testing.assert_array_equal(t[k_got].astype(np.uint64), want[k_want].astype(np.uint64), err_msg=k_got)
    for k_got, k_want in (("min_bps", "min"), ("max_bps", "max"), ("avg_bps", "avg"), ("median_bps", "median")):
        np.testing.assert_array_equal(t[k_got].view(np.uint64), want[k_want].view(np.uint64), err_msg=k_got)

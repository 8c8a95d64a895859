"""A small pass over every kernel family, for compute-sanitizer
(tools/sanitize.sh): K1/K2/K3 on SoA host and AoS inputs with histograms and
a fused window, hot-slot modes, per-host rows (both median paths: two-round
and sorted), NetFlow decode (golden datagrams), FLOWARC1 decode and in-place
analysis. Host numpy inputs (torch only for the key union of the cross-context path)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import numpy as np

import golden_io
from bench_ingest import make_archive
from paper_1108_1785_b200 import Engine, FlowBatch, FlowRecords, SiteCatalog, synth

w = synth.workload("D1")
cols = synth.generate(w, 200_000)
cat = SiteCatalog()
w.sites.register(cat)
with Engine(0) as eng:
    for mode in ("auto", "force", "off"):
        eng.set_hot_mode(mode)
        eng.aggregate(FlowBatch(*cols), cat, histograms=True)
    eng.set_hot_mode("auto")
    eng.aggregate(FlowRecords(synth.to_aos(cols)), cat)
    lo, hi = int(np.percentile(cols[5], 10)), int(np.percentile(cols[5], 90))
    eng.aggregate_window(FlowBatch(*cols), cat, lo, hi)
    eng.set_hosts(True)
    r = eng.aggregate(FlowBatch(*cols), cat, histograms=True)
    eng.host_histogram_entries()
    # > 100k rows: the sorted median path
    rng = np.random.default_rng(3)
    big = SiteCatalog()
    for i in range(8):
        big.register_site(f"b{i}", [f"10.{i}.0.0/16"])
    n = 400_000
    src = (0x0A000000 + (rng.integers(0, 8, n) << 16) + rng.integers(0, 65536, n)).astype(np.uint32)
    bcols = (src, rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32),
             rng.integers(20, 400, n).astype(np.uint32), rng.integers(20_000, 2**31, n).astype(np.uint32),
             np.full(n, 1_000_000, np.uint64) - rng.integers(100, 100_000, n).astype(np.uint64),
             np.full(n, 1_000_000, np.uint64))
    rb = eng.aggregate(FlowBatch(*bcols), big)
    assert len(rb.host_table) > 100_000, len(rb.host_table)
    eng.host_histogram_entries()
    # > 256 non-empty /16 blocks: hashed host slots instead of dense ids
    many = SiteCatalog()
    for i in range(300):
        many.register_site(f"m{i}", [f"{20 + i // 256}.{i % 256}.1.0/24"])
    msrc = np.array([((20 + i // 256) << 24) | ((i % 256) << 16) | (1 << 8) | (j % 200)
                     for i in range(300) for j in range(50)], np.uint32)
    m = len(msrc)
    mcols = (msrc, np.full(m, 1, np.uint32), np.full(m, 50, np.uint32), np.full(m, 500_000, np.uint32),
             np.full(m, 1_000_000 - 2000, np.uint64), np.full(m, 1_000_000, np.uint64))
    assert len(eng.aggregate(FlowBatch(*mcols), many).host_table) > 0
    # the cross-context union path with one context
    eng.accumulate(FlowBatch(*bcols), big)
    import torch
    keys = eng.hosts_local_keys(big)
    eng.hosts_set_keys(keys.clone())
    eng.hosts_prepare_median()
    eng.finalize(big)
    eng.set_hosts(False)
    # repeated device-batch calls: plain, capture, graph replays
    import torch
    dcols = [torch.from_numpy(c.view(np.int32 if c.dtype.itemsize == 4 else np.int64).copy()).cuda() for c in cols]
    for _ in range(4):
        eng.aggregate(FlowBatch(*dcols), cat)
    z = golden_io.load("netflow")
    eng.decode_netflow(z["datagrams"], z["offsets"])
    arc = make_archive(cols)
    eng.decode_archive(arc)
    eng.aggregate_archive(arc, cat)
    # the archive resident in HBM: k2_arc's 16-byte vector loads (entry - 4 reads the header)
    import torch
    eng.aggregate_archive(torch.from_numpy(np.frombuffer(arc, np.uint8).copy()).cuda(), cat)
# in-library multi-rank combine: a loopback group (sites, per-host union,
# histograms summed) and a world-size-1 NCCL communicator with graph replay
from paper_1108_1785_b200 import Group
with Group([0, 0], kind="loopback") as g:
    g.aggregate(FlowBatch(*cols), cat, histograms=True)
    g.set_hosts(True)
    g.aggregate(FlowRecords(synth.to_aos(cols)), cat)
    g.host_histogram_entries()
with Engine(0) as e1:
    e1.comm_init(1, 0, Engine.comm_unique_id())
    for _ in range(3):
        e1.aggregate(FlowBatch(*dcols), cat)
print("sanitize run ok:", len(r.host_table), "host rows,", len(rb.host_table), "host rows (sorted path)")

"""Where a hosts-mode step goes (run under gpurun): the finalize call's
phases on the host clock -- accumulate (async), gnm_finalize (K3 + the
per-host post-pass + its syncs), and gnm_host_results (D2H of the rows into
the caller's buffer, pageable vs pinned) -- on D3 in HBM."""
import ctypes as C
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_1108_1785_b200 import Engine, FlowBatch, SiteCatalog, synth, _lib

w = synth.workload("D3")
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
cat = SiteCatalog()
w.sites.register(cat)
cols = synth.generate(w, n)
dev = [torch.from_numpy(c.view(np.int32 if c.dtype.itemsize == 4 else np.int64)).cuda() for c in cols]
b = FlowBatch(*dev)
eng = Engine(0)
eng.set_hosts(True)
for _ in range(3):
    eng.aggregate(b, cat)
torch.cuda.synchronize()
L = _lib.lib
ph = {"accumulate": [], "finalize": [], "rows_pageable": [], "rows_pinned": []}
pinned = torch.empty(200_000 * 64, dtype=torch.uint8).pin_memory()
for _ in range(10):
    t0 = time.perf_counter()
    eng.accumulate(b, cat)
    t1 = time.perf_counter()
    r, table, hist, ns = eng._result(cat, 0, 0, 1e6, False)
    _lib.lib.gnm_finalize(eng.handle, cat.handle, C.byref(r))
    t2 = time.perf_counter()
    k = L.gnm_host_count(eng.handle)
    rows = np.empty(k, _lib.HOST_STATS_DTYPE)
    L.gnm_host_results(eng.handle, rows.ctypes.data, k, None)
    t3 = time.perf_counter()
    L.gnm_host_results(eng.handle, pinned.data_ptr(), k, None)
    t4 = time.perf_counter()
    for key, v in zip(ph, (t1 - t0, t2 - t1, t3 - t2, t4 - t3)):
        ph[key].append(v * 1e3)
print({k: round(float(np.median(v)), 3) for k, v in ph.items()}, "host rows", k, flush=True)

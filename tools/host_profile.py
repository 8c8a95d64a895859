"""Where the host time of one bench step goes (run under gpurun): wall time of
Engine.accumulate / Engine.finalize / the whole aggregate, against the device
time of the same step (CUDA events), on the D3 workload in HBM."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_1108_1785_b200 import Engine, FlowBatch, SiteCatalog, synth

w = synth.workload("D3")
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
cat = SiteCatalog()
w.sites.register(cat)
cols = synth.generate(w, n)
dev = [torch.from_numpy(c.view(np.int32 if c.dtype.itemsize == 4 else np.int64)).cuda() for c in cols]
b = FlowBatch(*dev)
for timing in (True, False):
    eng = Engine(0)
    eng.enable_timing(timing)
    for _ in range(3):
        eng.aggregate(b, cat)
    torch.cuda.synchronize()
    acc, fin, tot = [], [], []
    for _ in range(10):
        t0 = time.perf_counter()
        eng.accumulate(b, cat)
        t1 = time.perf_counter()
        r = eng.finalize(cat)
        t2 = time.perf_counter()
        acc.append(t1 - t0)
        fin.append(t2 - t1)
        tot.append(t2 - t0)
    t0 = time.perf_counter()
    for _ in range(10):
        eng.aggregate(b, cat)
    wall = (time.perf_counter() - t0) / 10
    print(f"timing={timing}: accumulate call {np.median(acc)*1e3:.3f} ms (host, async), finalize call "
          f"{np.median(fin)*1e3:.3f} ms (host, includes waiting for K2), step wall {wall*1e3:.3f} ms",
          flush=True)
    eng.close()

"""GPU idle per step with graph replay (run under gpurun): device events
around each Engine.aggregate call on the engine stream; the span of a call
vs its kernels, and host time per call split into the C call and the Python
wrapper."""
import sys
import time

sys.path.insert(0, ".")
import ctypes as C
import numpy as np
import torch

from paper_1108_1785_b200 import Engine, FlowBatch, SiteCatalog, synth
from paper_1108_1785_b200._lib import lib

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
w = synth.workload("D3")
cat = SiteCatalog()
w.sites.register(cat)
cols = synth.generate(w, n)
dev = [torch.from_numpy(c.view(np.int32 if c.dtype.itemsize == 4 else np.int64)).cuda() for c in cols]
b = FlowBatch(*dev)
eng = Engine(0)
stream = torch.cuda.ExternalStream(eng.stream_handle(), device="cuda:0")
for _ in range(5):
    eng.aggregate(b, cat)
torch.cuda.synchronize()
steps = 30
evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
wall = []
for i in range(steps):
    t0 = time.perf_counter()
    evs[i][0].record(stream)
    eng.aggregate(b, cat)
    evs[i][1].record(stream)
    wall.append(time.perf_counter() - t0)
torch.cuda.synchronize()
span = [a.elapsed_time(z) for a, z in evs]
gap = [evs[i][1].elapsed_time(evs[i + 1][0]) for i in range(steps - 1)]
print(f"wall/call {np.median(wall)*1e3:.3f} ms, device span {np.median(span):.3f} ms, "
      f"gap between calls {np.median(gap):.3f} ms")
# Host cost of the Python result wrapper vs the raw C call on a tiny batch.
small = FlowBatch(*[x[:4096] for x in dev])
for _ in range(5):
    eng.aggregate(small, cat)
t0 = time.perf_counter()
for _ in range(200):
    eng.aggregate(small, cat)
print(f"4096-record aggregate (graph replay): {(time.perf_counter() - t0) / 200 * 1e3:.3f} ms per call")

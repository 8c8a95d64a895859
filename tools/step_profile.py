"""Where a bench step's time goes beyond the kernels (run under gpurun):
per step, the wall time of Engine.aggregate, the device span between
events recorded on the engine stream just before and after the call, and
the context's own kernel totals (K1 + K2 + finalize). The difference
between the device span and the kernel sum is GPU idle time inside the call
(host-side launch preparation); wall minus span is host time outside the
GPU's view (result building, the call's prologue before its first launch).

    python tools/step_profile.py [records]
"""
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_1108_1785_b200 import Engine, FlowBatch, SiteCatalog, synth

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
steps = 20
eng.enable_timing(True)
evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
wall = []
t_all = time.perf_counter()
for i in range(steps):
    t0 = time.perf_counter()
    evs[i][0].record(stream)
    eng.aggregate(b, cat)
    evs[i][1].record(stream)
    wall.append(time.perf_counter() - t0)
torch.cuda.synchronize()
t_all = (time.perf_counter() - t_all) / steps
t = eng.timing()
span = [a.elapsed_time(z) for a, z in evs]
between = [evs[i][1].elapsed_time(evs[i + 1][0]) for i in range(steps - 1)]
k = (t["total_plan_ms"] + t["total_accumulate_ms"] + t["total_finalize_ms"]) / steps
print(f"records {n}: wall/step {t_all*1e3:.3f} ms (call {np.median(wall)*1e3:.3f}), device span/step "
      f"{np.median(span):.3f} ms, kernels/step {k:.3f} ms (K1 {t['total_plan_ms']/steps:.3f}, "
      f"K2 {t['total_accumulate_ms']/steps:.3f}, finalize {t['total_finalize_ms']/steps:.3f}), "
      f"idle between calls {np.median(between):.3f} ms")

# Host cost of the call with almost no device work.
small = FlowBatch(*[x[:4096] for x in dev])
for _ in range(5):
    eng.aggregate(small, cat)
t0 = time.perf_counter()
for _ in range(100):
    eng.aggregate(small, cat)
print(f"4096-record aggregate: {(time.perf_counter() - t0) * 10:.3f} ms per call (host + launch floor)")

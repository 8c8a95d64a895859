import sys, time, ctypes as C
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1108_1785_b200 import Engine, FlowBatch, SiteCatalog, synth
from paper_1108_1785_b200 import _lib
w = synth.workload("D3"); cat = SiteCatalog(); w.sites.register(cat)
cols = synth.generate(w, 100_000_000)
dev = [torch.from_numpy(c.view(np.int32 if c.dtype.itemsize == 4 else np.int64)).cuda() for c in cols]
b = FlowBatch(*dev); eng = Engine(0)
stream = torch.cuda.ExternalStream(eng.stream_handle(), device="cuda:0")
for _ in range(5): eng.aggregate(b, cat)
torch.cuda.synchronize()
# raw C call with a persistent table (no numpy allocation per call)
p = Engine._params(None); bb = b._c()
r, table, hist, n = eng._result(cat, 0, 0, 1e6, False)
def raw():
    _lib.lib.gnm_analyze(eng.handle, cat.handle, C.byref(p), C.byref(bb), C.byref(r))
for name, fn in (("python aggregate", lambda: eng.aggregate(b, cat)), ("raw C, reused table", raw)):
    for _ in range(5): fn()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); e0.record(stream)
    for _ in range(50): fn()
    e1.record(stream); torch.cuda.synchronize()
    print(name, "device ms/step", e0.elapsed_time(e1) / 50, "wall", (time.perf_counter() - t0) / 50 * 1e3)

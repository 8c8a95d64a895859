"""One hosts-mode step on the device timeline (run under gpurun): every
kernel, memset and copy of one Engine.aggregate call with set_hosts(True)
on D3 in HBM, from CUPTI via torch.profiler (not serialised, unlike the ncu
launch list), with the idle gap before each, so host syncs and launch
latency show up beside the kernels.

    python tools/hosts_timeline.py [records] [--sites]
"""
import sys

sys.path.insert(0, ".")
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

from paper_1108_1785_b200 import Engine, FlowBatch, SiteCatalog, synth

args = [a for a in sys.argv[1:] if not a.startswith("--")]
n = int(args[0]) if args else 100_000_000
hosts = "--sites" not in sys.argv
w = synth.workload("D3")
cat = SiteCatalog()
w.sites.register(cat)
cols = synth.generate(w, n)
dev = [torch.from_numpy(c.view(np.int32 if c.dtype.itemsize == 4 else np.int64)).cuda() for c in cols]
b = FlowBatch(*dev)
eng = Engine(0)
eng.set_hosts(hosts)
for _ in range(4):
    eng.aggregate(b, cat)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        eng.aggregate(b, cat)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
# split into the three calls at the K1 sampling kernel
starts = [i for i, e in enumerate(ev) if e.name.startswith("void gnm::") and "k_sample" in e.name or
          e.name.startswith("k_sample") or "k_sample<" in e.name]
if len(starts) >= 2:
    ev = ev[starts[-2]:starts[-1]] if len(starts) >= 3 else ev[starts[-1]:]
t0 = ev[0].time_range.start
prev = t0
tot = {}
print(f"{'start_us':>9} {'gap_us':>7} {'dur_us':>8}  name")
for e in ev:
    s, d = e.time_range.start, e.time_range.end - e.time_range.start
    nm = e.name.replace("void ", "").replace("gnm::", "").replace("(anonymous namespace)::", "")[:90]
    print(f"{s - t0:9.1f} {s - prev:7.1f} {d:8.1f}  {nm}")
    prev = max(prev, e.time_range.end)
    k = nm.split("(")[0]
    tot[k] = tot.get(k, 0) + d
span = prev - t0
busy = sum(tot.values())
print(f"step span {span:.1f} us, busy {busy:.1f} us, idle {span - busy:.1f} us")
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:25]:
    print(f"{v:9.1f}  {k}")

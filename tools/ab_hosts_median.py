"""A/B of the per-host median schemes (run under gpurun): the hosts-mode step
at D3 in HBM with GNM_HOSTS_MEDIAN=two|sort, one process per setting
(interleaved), CUDA events on the engine's calls; the row tables of both
schemes must be identical (a digest is printed)."""
import hashlib
import os
import subprocess
import sys

if len(sys.argv) > 1 and sys.argv[1] == "--child":
    sys.path.insert(0, ".")
    import numpy as np
    import torch

    from paper_1108_1785_b200 import Engine, FlowBatch, SiteCatalog, synth

    w = synth.workload("D3")
    n = int(sys.argv[2])
    cat = SiteCatalog()
    w.sites.register(cat)
    cols = synth.generate(w, n)
    dev = [torch.from_numpy(c.view(np.int32 if c.dtype.itemsize == 4 else np.int64)).cuda() for c in cols]
    b = FlowBatch(*dev)
    eng = Engine(0)
    eng.set_hosts(True)
    for _ in range(3):
        res = eng.aggregate(b, cat)
    torch.cuda.synchronize()
    ts = []
    for _ in range(15):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        res = eng.aggregate(b, cat)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    t = res.host_table
    dig = hashlib.sha1(t.tobytes()).hexdigest()[:16]
    print(f"{os.environ.get('GNM_HOSTS_MEDIAN', 'default'):8s} median {np.median(ts):.3f} ms min {min(ts):.3f} rows {len(t)} digest {dig}", flush=True)
    sys.exit(0)

n = sys.argv[1] if len(sys.argv) > 1 else "100000000"
for rep in range(2):
    for mode in ("two", "sort"):
        env = dict(os.environ, GNM_HOSTS_MEDIAN=mode)
        subprocess.run([sys.executable, __file__, "--child", n], env=env, check=True)

# K2 ablation on D3 (100M records): times K2 with parts of the pipeline
# switched off, using the measurement build (make ablation). Run under gpurun.
#   1 stage A only (stream, classify, /16 probes; nothing queued)
#   2 + queue/drain + /24 resolve, no per-flow arithmetic
#   3 + all per-flow arithmetic, no reductions
#   4 + the histogram RED only
#   5 full kernel with an approximate (single-MUFU) rate: the cost of the IEEE division
#   6 full kernel without min/max; 7 full kernel without the sums
#   0 full kernel
set -u
mkdir -p gpurun_out
for m in ${MODES:-1 2 3 4 0}; do
  GNM_K2_ABLATION=$m GNM_LIB=paper_1108_1785_b200/lib/ablation/libgnetmon.so timeout 300 python - <<'PY' 2>&1 | tail -1 | tee -a gpurun_out/ablation.txt
import os, sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_1108_1785_b200 import Engine, FlowBatch, SiteCatalog, synth
w = synth.workload('D3'); n = 100_000_000
cat = SiteCatalog(); w.sites.register(cat)
cols = synth.generate(w, n)
dev = [torch.from_numpy(c.view(np.int32 if c.dtype.itemsize == 4 else np.int64)).cuda() for c in cols]
b = FlowBatch(*dev)
eng = Engine(0); eng.enable_timing(True)
for _ in range(3): eng.aggregate(b, cat)
eng.timing()
ts = []
for _ in range(5):
    eng.aggregate(b, cat); ts.append(eng.timing()['accumulate_ms'])
print(os.environ.get('GNM_K2_VARIANT', 'reg'), 'ablation', os.environ['GNM_K2_ABLATION'], 'k2 ms', [round(t, 3) for t in ts])
PY
done

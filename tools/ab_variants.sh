#!/usr/bin/env bash
# A/B of the in-tree library against variant builds (run under gpurun):
#   VARIANTS="lib/v896 lib/ab_old" bash tools/ab_variants.sh
# Each line: variant, step ms, K2 ms, finalize ms (bench.py, 100 steps).
set -u
mkdir -p gpurun_out
for i in 1 2 3; do
  for v in cur ${VARIANTS}; do
    if [ $v = cur ]; then unset GNM_LIB; else export GNM_LIB=$PWD/paper_1108_1785_b200/$v/libgnetmon.so; fi
    python bench.py --no-cpu-baseline --e2e-steps 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],4), round(d['breakdown_ms']['k2'],4), round(d['breakdown_ms']['k3_finalize'],4))" >> gpurun_out/ab.txt
  done
done

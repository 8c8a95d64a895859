#!/usr/bin/env bash
# tools/bench_ingest.py per library variant, interleaved (run under gpurun):
#   VARIANTS="a b" ROUNDS=2 bash tools/ab_ingest.sh  -> gpurun_out/ab_ingest.txt
set -u
mkdir -p gpurun_out
for i in $(seq 1 ${ROUNDS:-2}); do
  for v in $VARIANTS; do
    GNM_LIB=$PWD/paper_1108_1785_b200/lib/$v/libgnetmon.so python tools/bench_ingest.py --cpu-records 100000 2>/dev/null \
      | python -c "
import json, sys
for l in sys.stdin:
    d = json.loads(l)
    print('$v', d['row'], round(d['ms'], 4))" >> gpurun_out/ab_ingest.txt
  done
done

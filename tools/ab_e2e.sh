#!/usr/bin/env bash
# e2e (pinned and pageable host input) per library variant, interleaved:
#   VARIANTS="a b" ROUNDS=2 [BENCH_ARGS=...] bash tools/ab_e2e.sh
set -u
mkdir -p gpurun_out
for i in $(seq 1 ${ROUNDS:-2}); do
  for v in $VARIANTS; do
    GNM_LIB=$PWD/paper_1108_1785_b200/lib/$v/libgnetmon.so python bench.py --no-cpu-baseline --no-adapter --no-extras \
        ${BENCH_ARGS:-} 2>/dev/null | python -c "
import json, sys
d = json.loads(sys.stdin.read()); e = d['e2e']
print('$v', 'value', round(d['value'] / 1e9, 2), 'e2e', round(e['value'] / 1e9, 3),
      'pageable', round(e['pageable']['value'] / 1e9, 3) if e.get('pageable') else None)" >> gpurun_out/ab_e2e.txt
  done
done

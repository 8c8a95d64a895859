#!/usr/bin/env bash
# Per-variant ncu metrics of one kernel (run under gpurun from the repo root):
#   VARIANTS="a b" KERNEL=h_insert BENCH_ARGS="--hosts" bash tools/ab_ncu_metrics.sh
# One line per variant: duration, L2 RED sectors, warp instructions, DRAM bytes.
set -u
mkdir -p gpurun_out
M=gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_red.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum
for v in $VARIANTS; do
  GNM_LIB=$PWD/paper_1108_1785_b200/lib/$v/libgnetmon.so timeout 900 ncu --metrics $M --clock-control none \
      -k "regex:${KERNEL}" -s 2 -c 1 --csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 \
      --no-pageable --no-adapter --no-extras ${BENCH_ARGS:-} 2>/dev/null \
    | python -c "
import csv, sys
rows = [r for r in csv.reader(sys.stdin)]
i = next(k for k, r in enumerate(rows) if 'Metric Name' in r)
h = rows[i]; out = {}
for r in rows[i + 1:]:
    if len(r) != len(h): continue
    out[r[h.index('Metric Name')]] = r[h.index('Metric Value')]
print('$v', ' '.join(f'{k.split(\"__\")[1][:28]}={v}' for k, v in out.items()))
" >> gpurun_out/ab_ncu.txt
done

set -u
mkdir -p gpurun_out
for i in 1 2 3; do
  for v in old new; do
    if [ $v = old ]; then export GNM_LIB=$PWD/paper_1108_1785_b200/lib/ab_old/libgnetmon.so; else unset GNM_LIB; fi
    python bench.py --no-cpu-baseline --e2e-steps 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],4), round(d['breakdown_ms']['k2'],4), round(d['breakdown_ms']['k3_finalize'],4))" >> gpurun_out/ab.txt
  done
done

# A/B/C over prebuilt libraries: VARIANTS="ab_v32 ab_v16" (dirs under
# paper_1108_1785_b200/lib, each holding a libgnetmon.so), ROUNDS pairs,
# interleaved on one box. Lines: variant ms_per_step k2_ms finalize_ms.
set -u
mkdir -p gpurun_out
for i in $(seq 1 ${ROUNDS:-3}); do
  for v in $VARIANTS; do
    GNM_LIB=$PWD/paper_1108_1785_b200/lib/$v/libgnetmon.so python bench.py --no-cpu-baseline --e2e-steps 3 --no-adapter --no-pageable --no-extras ${BENCH_ARGS:-} 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],4), round(d['breakdown_ms']['k2'],4), round(d['breakdown_ms']['k3_finalize'],4))" >> gpurun_out/ab_multi.txt
  done
done

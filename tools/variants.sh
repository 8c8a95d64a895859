# K2 variant matrix (env knobs read by gnm_ctx_create); results are identical,
# only the time differs. Usage: bash tools/variants.sh [variants...]
V=${*:-"reg l2"}
for v in $V; do
  GNM_K2_VARIANT=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/var_${v}.json 2>gpurun_out/var_${v}.err
  python -c "
import json,sys
d=json.loads(open('gpurun_out/var_${v}.json').read().strip().splitlines()[-1]); print('$v', round(d['value']/1e9,2), 'Grec/s', {k:round(x,3) for k,x in d['breakdown_ms'].items()})
" | tee -a gpurun_out/variants.txt
done

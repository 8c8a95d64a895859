# Variant matrix for K2 (env knobs read by gnm_ctx_create).
for v in direct tma; do for cm in check red; do
  GNM_K2_VARIANT=$v GNM_COLD_MINMAX=$cm timeout 200 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/var_${v}_${cm}.json 2>/dev/null
  python -c "
import json,sys
d=json.loads(open('gpurun_out/var_${v}_${cm}.json').read().strip().splitlines()[-1]); print('$v $cm', round(d['value']/1e9,2), {k:round(x,3) for k,x in d['breakdown_ms'].items()})
"
done; done

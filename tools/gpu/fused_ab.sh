# bench with the separate advect + Laplacian/count kernels (HB_FUSED_FIELD=0) and the fused one (1)
for v in 0 1; do
  HB_FUSED_FIELD=$v python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('fused=$v', round(d['value']/1e9,3), round(d['ms_per_step'],2), {k:v['avg_ms'] for k,v in d['roofline']['per_kernel'].items() if v['avg_ms']>0.1})"
done

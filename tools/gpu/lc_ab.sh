# A/B of the Laplacian + count kernel: bench per-kernel averages for each variant
for v in default "$@"; do
  if [ "$v" != default ]; then export HB_B200_LIB=paper_1504_02687_b200/_lib/var_$v/libhb_b200.so; else unset HB_B200_LIB; fi
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['value']/1e9,3), round(d['ms_per_step'],2), {k:v['avg_ms'] for k,v in d['roofline']['per_kernel'].items() if v['avg_ms']>0.1})"
done

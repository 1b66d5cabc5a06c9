# config-5 bench (tile-record splat) for each built variant
for v in default "$@"; do
  if [ "$v" != default ]; then export HB_B200_LIB=paper_1504_02687_b200/_lib/var_$v/libhb_b200.so; else unset HB_B200_LIB; fi
  python bench.py --config 5 --steps 1 --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['value']/1e9,3), round(d['ms_per_step'],1), {k:round(v['avg_ms'],2) for k,v in d['roofline']['per_kernel'].items() if v['avg_ms']>1})"
done

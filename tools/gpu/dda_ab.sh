# A/B for the rasteriser: config-4 bench (iteration-0 splat, key expansion) and config-5 bench (tile flush)
for v in default "$@"; do
  if [ "$v" != default ]; then export HB_B200_LIB=paper_1504_02687_b200/_lib/var_$v/libhb_b200.so; else unset HB_B200_LIB; fi
  for c in 4 5; do
    python bench.py --config $c --steps 1 --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v cfg$c', round(d['value']/1e9,3), round(d['ms_per_step'],2), {k:v['avg_ms'] for k,v in d['roofline']['per_kernel'].items() if v['avg_ms']>0.1})"
  done
done

# usage: bench_variants.sh name...  -- short bench per library variant (same box)
mkdir -p gpurun_out
for v in default "$@"; do
  if [ "$v" = nodefer ]; then export HB_DEFER_LAP=0; else unset HB_DEFER_LAP; fi
  if [ "$v" != default ] && [ "$v" != nodefer ]; then export HB_B200_LIB=paper_1504_02687_b200/_lib/var_$v/libhb_b200.so; else unset HB_B200_LIB; fi
  timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bv_$v.json 2>/dev/null
  python - "$v" <<'PY'
import json, sys
v = sys.argv[1]
d = json.loads([l for l in open(f'gpurun_out/bv_{v}.json') if l.startswith('{')][-1])
pk = d['roofline']['per_kernel']
print(v, "%.3e" % d['value'], "%.1f ms/step" % d['ms_per_step'], {k: pk[k]['avg_ms'] for k in list(pk)[:4]})
PY
done

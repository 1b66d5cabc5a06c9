# usage: bench_variants.sh name...  -- short bench per library variant (same box)
# BV_ARGS: extra bench.py arguments (e.g. "--scale 0.125")
mkdir -p gpurun_out
for v in default "$@"; do
  # env:NAME=VALUE variants set an environment switch, others pick a library
  unset HB_B200_LIB HB_SYNC_FREE HB_FLAT_ADVECT
  case "$v" in
    default) ;;
    env:*) export "${v#env:}" ;;
    *) export HB_B200_LIB=paper_1504_02687_b200/_lib/var_$v/libhb_b200.so ;;
  esac
  timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline $BV_ARGS > "gpurun_out/bv_${v//[:=]/_}.json" 2>/dev/null
  python - "${v//[:=]/_}" <<'PY'
import json, sys
v = sys.argv[1]
d = json.loads([l for l in open(f'gpurun_out/bv_{v}.json') if l.startswith('{')][-1])
pk = d['roofline']['per_kernel']
print(v, "%.3e" % d['value'], "%.1f ms/step" % d['ms_per_step'], {k: pk[k]['avg_ms'] for k in list(pk)[:4]})
PY
done

# usage: probe_variants.sh keys name...  -- kernel_probe per library variant (same box)
mkdir -p gpurun_out
keys="$1"; shift
for v in default "$@"; do
  if [ "$v" != default ]; then export HB_B200_LIB=paper_1504_02687_b200/_lib/var_$v/libhb_b200.so; else unset HB_B200_LIB; fi
  timeout 300 python tools/kernel_probe.py --config 4 --iters 6 > gpurun_out/probe_$v.json 2>&1
  python - "$v" "$keys" <<'PY'
import json, sys
v, keys = sys.argv[1], sys.argv[2].split(',')
try:
    d = json.load(open(f'gpurun_out/probe_{v}.json'))
    print(v, {k: round(d[k], 3) for k in keys if k in d})
except Exception as ex:
    print(v, 'failed', ex)
PY
done

for q in 4096 0; do
HB_QUAD_LIMIT_MB=$q timeout 900 python bench.py --config 5 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/cfg5_q$q.json 2> gpurun_out/cfg5_q$q.err
python - $q <<'PY'
import json,sys
d=json.loads([l for l in open(f"gpurun_out/cfg5_q{sys.argv[1]}.json") if l.startswith('{')][-1])
print("quad", sys.argv[1], "value %.3e ms/it %.2f" % (d['value'], d['ms_per_iteration']))
print({k:v['avg_ms'] for k,v in d['roofline']['per_kernel'].items()})
PY
done

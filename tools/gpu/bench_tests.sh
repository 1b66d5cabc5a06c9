mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_cur.json 2> gpurun_out/bench_cur.err; echo bench rc=$?
python - <<'PY'
import json
d=json.loads([l for l in open('gpurun_out/bench_cur.json') if l.startswith('{')][-1])
print("value %.3e ms/step %.1f e2e %.3e" % (d['value'], d['ms_per_step'], d['e2e']['value']))
print({k:(v['avg_ms'],v['launches']) for k,v in d['roofline']['per_kernel'].items()})
print("clocks", d['clocks'], "cpu", d['cpu_baseline']['value'])
PY

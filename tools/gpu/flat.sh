mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python tools/kernel_probe.py --config 4 --iters 6 > gpurun_out/probe.json 2>&1; echo probe rc=$?
python -c "
import json; d=json.load(open('gpurun_out/probe.json')); print({k:round(v,3) for k,v in d.items() if k.endswith('_ms')})" || tail -5 gpurun_out/probe.json
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_flat.json 2> gpurun_out/bench_flat.err; echo bench rc=$?
python - <<'PY'
import json
d=json.loads([l for l in open('gpurun_out/bench_flat.json') if l.startswith('{')][-1])
print("value %.3e ms/step %.1f e2e %.3e" % (d['value'], d['ms_per_step'], d['e2e']['value']))
print({k:(v['avg_ms'],v['launches']) for k,v in d['roofline']['per_kernel'].items()})
PY

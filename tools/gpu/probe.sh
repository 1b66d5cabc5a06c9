mkdir -p gpurun_out
timeout 300 python tools/kernel_probe.py --config 4 --iters 6 > gpurun_out/probe.json 2>&1; echo probe rc=$?
python -c "
import json; d=json.load(open('gpurun_out/probe.json')); print({k:round(v,3) for k,v in d.items() if k.endswith('_ms')})"
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2

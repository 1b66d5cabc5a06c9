mkdir -p gpurun_out
timeout 300 python tools/kernel_probe.py --config 4 --iters 6 > gpurun_out/probe.json 2>&1; echo probe rc=$?
python -c "
import json; d=json.load(open('gpurun_out/probe.json')); print({k:round(v,3) for k,v in d.items() if k.endswith('_ms')})"
# count kernel of iteration 5 (6th launch of the COUNT-only variant) on the real state
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base mangled -k regex:ILb0ELb0ELb1ELb0E --launch-skip 5 --launch-count 1 -o gpurun_out/prof_cnt5 -f python tools/kernel_probe.py --config 4 --iters 6 > gpurun_out/prof_cnt5.log 2>&1
tail -2 gpurun_out/prof_cnt5.log

mkdir -p gpurun_out
timeout 300 python tools/kernel_probe.py --config 4 --iters 6 > gpurun_out/probe_base.json 2>&1 || exit 1
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base mangled -k regex:ILb1ELb1ELb0ELb1E --launch-skip 5 --launch-count 1 -o gpurun_out/prof_adv5 -f python tools/kernel_probe.py --config 4 --iters 6 > gpurun_out/prof_adv5.log 2>&1
tail -3 gpurun_out/prof_adv5.log

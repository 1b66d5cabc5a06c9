mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:advect_flat_kernel --launch-skip 5 --launch-count 1 -o gpurun_out/prof_flat5 -f python tools/kernel_probe.py --config 4 --iters 6 > gpurun_out/prof_flat5.log 2>&1
tail -1 gpurun_out/prof_flat5.log
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base mangled -k regex:ILb0ELb1ELb1ELb0E --launch-skip 4 --launch-count 1 -o gpurun_out/prof_lapcnt5 -f python tools/kernel_probe.py --config 4 --iters 6 > gpurun_out/prof_lapcnt5.log 2>&1
tail -1 gpurun_out/prof_lapcnt5.log

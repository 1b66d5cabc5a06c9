mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:segtab_expand --launch-skip 4 --launch-count 1 -o gpurun_out/prof_exp -f python tools/kernel_probe.py --config 4 --iters 6 > gpurun_out/prof_exp.log 2>&1
tail -1 gpurun_out/prof_exp.log

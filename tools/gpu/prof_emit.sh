mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:emit_kernel --launch-skip 4 --launch-count 1 -o gpurun_out/prof_emit5 -f python tools/kernel_probe.py --config 4 --iters 6 > gpurun_out/prof_emit5.log 2>&1
tail -1 gpurun_out/prof_emit5.log

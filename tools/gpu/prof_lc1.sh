mkdir -p gpurun_out
python tools/kernel_probe.py --config 4 --iters 6 > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:lapcount_kernel \
  --launch-skip 4 --launch-count 1 -o gpurun_out/pr_lapcount -f python tools/kernel_probe.py --config 4 --iters 6 \
  > gpurun_out/pr_lapcount.log 2>&1; echo lapcount rc=$?

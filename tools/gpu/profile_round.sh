# Round profile: bench line, ncu launch list, ncu --set full of the top kernels.
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/pr_bench.json 2> gpurun_out/pr_bench.err; echo bench rc=$?
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/pr_launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline \
  > gpurun_out/pr_launches.log 2>&1; echo launches rc=$?
for k in emit_ring_kernel advect_flat_kernel; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k --launch-skip 4 --launch-count 1 \
    -o gpurun_out/pr_$k -f python tools/kernel_probe.py --config 4 --iters 6 > gpurun_out/pr_$k.log 2>&1; echo $k rc=$?
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:lapcount_kernel \
  --launch-skip 4 --launch-count 1 -o gpurun_out/pr_lapcount -f python tools/kernel_probe.py --config 4 --iters 6 \
  > gpurun_out/pr_lapcount.log 2>&1; echo lapcount rc=$?

# bench line + launch list of the final code (no ncu full: kernels unchanged)
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/pr_bench.json 2> gpurun_out/pr_bench.err; echo bench rc=$?
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/pr_launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline \
  > gpurun_out/pr_launches.log 2>&1; echo launches rc=$?

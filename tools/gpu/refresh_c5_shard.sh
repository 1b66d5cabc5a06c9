mkdir -p gpurun_out
timeout 1200 python bench.py --config 5 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/cfg5_bench.json 2> gpurun_out/cfg5_bench.err; echo cfg5 rc=$?
timeout 1200 python tools/shard_probe.py > gpurun_out/shard_probe.json 2> gpurun_out/shard_probe.err; echo shard rc=$?

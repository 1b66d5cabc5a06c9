set -x; mkdir -p gpurun_out
export HB_BENCH_ONE_DEVICE=1 HB_DIST_BACKEND=gloo
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --steps 2 --warmup 3 --config 1 > gpurun_out/mr_c1.log 2>&1; echo rc=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29532 bench.py --gpus 2 --steps 2 --warmup 3 --config 4 --no-cpu-baseline > gpurun_out/mr_c4.log 2>&1; echo rc=$?
unset HB_BENCH_ONE_DEVICE HB_DIST_BACKEND
timeout 900 python bench.py --config 5 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c5.log 2>&1; echo rc=$?
nvidia-smi --query-gpu=memory.used,memory.total --format=csv
tail -3 gpurun_out/mr_c1.log gpurun_out/mr_c4.log gpurun_out/c5.log

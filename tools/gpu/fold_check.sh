# fused fold: parity tests, then timing (CUDA events) and the launch list of one smoothing call
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "smooth" 2>&1 | tail -3
python tools/smooth_probe.py
python tools/smooth_probe.py --nbins 1 --nv 1024 --nu 1024 --sigma 25.6
HB_FOLD=0 python tools/smooth_probe.py --nbins 1 --nv 1024 --nu 1024 --sigma 25.6
bash tools/gpu/smooth_breakdown.sh 2>&1 | grep -v "at::"

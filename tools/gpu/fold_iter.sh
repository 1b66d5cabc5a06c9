mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "smooth" 2>&1 | tail -2
python tools/smooth_probe.py
python tools/smooth_probe.py --nbins 1 --nv 1024 --nu 1024 --sigma 25.6
export HB_B200_LIB=paper_1504_02687_b200/_lib/var_trace/libhb_b200.so
python tools/fold_trace.py | tail -5
python tools/fold_trace.py --nbins 4 --nv 2047 --nu 2048 | tail -9

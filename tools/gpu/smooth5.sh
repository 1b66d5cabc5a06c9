# hb_smooth on the config-5 map (4 x 2047 x 2048) and config 4's (1 x 1024 x 1024):
# CUDA-event time, then the per-kernel launch list (cold, serialised).
mkdir -p gpurun_out
python tools/smooth_probe.py
python tools/smooth_probe.py --nbins 1 --nv 1024 --nu 1024 --sigma 25.6
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  python tools/smooth_probe.py --reps 1 2>/dev/null | grep -v "^==" | grep -v '^{' > gpurun_out/smooth5_ncu.csv

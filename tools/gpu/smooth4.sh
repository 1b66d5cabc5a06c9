mkdir -p gpurun_out
timeout 300 python tools/smooth_probe.py --nbins 1 --nv 1024 --nu 1024 --sigma 25.6
timeout 300 python tools/smooth_probe.py
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv python tools/smooth_probe.py --nbins 1 --nv 1024 --nu 1024 --sigma 25.6 --reps 1 2>/dev/null | grep -v "^==" > gpurun_out/smooth4_ncu.csv

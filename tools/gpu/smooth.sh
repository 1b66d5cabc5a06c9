mkdir -p gpurun_out
timeout 300 python tools/smooth_probe.py
timeout 300 python tools/smooth_probe.py --nbins 1 --nv 1024 --nu 1024 --sigma 25.6
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv python tools/smooth_probe.py --reps 1 2>/dev/null | grep -v "^==" > gpurun_out/smooth_ncu.csv

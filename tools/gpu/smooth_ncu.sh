mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum --clock-control none --csv python tools/smooth_probe.py --nbins 1 --nv 1024 --nu 1024 --sigma 25.6 --reps 1 2>/dev/null | grep -v "^==" > gpurun_out/smooth4_ncu.csv
timeout 600 ncu --set full --clock-control none -k regex:col_fold --launch-count 1 -o gpurun_out/prof_colfold -f python tools/smooth_probe.py --nbins 1 --nv 1024 --nu 1024 --sigma 25.6 --reps 1 > /dev/null 2>&1

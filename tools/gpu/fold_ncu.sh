mkdir -p gpurun_out
python tools/smooth_probe.py --nbins 1 --nv 1024 --nu 1024 --sigma 25.6 --reps 1 > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --set full --warp-sampling-interval 0 --clock-control none --import-source on -k regex:fold_kernel -c 1 -o gpurun_out/prof_fold4 -f python tools/smooth_probe.py --nbins 1 --nv 1024 --nu 1024 --sigma 25.6 --reps 1 > gpurun_out/ncu.log 2>&1
tail -3 gpurun_out/ncu.log

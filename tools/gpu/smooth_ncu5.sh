mkdir -p gpurun_out
python tools/smooth_probe.py --reps 1 > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"hwin|vwin" -c 2 -o gpurun_out/prof_smooth5 -f python tools/smooth_probe.py --reps 1 > gpurun_out/ncu.log 2>&1
tail -2 gpurun_out/ncu.log

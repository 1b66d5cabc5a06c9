# Smoothing evidence for profiles/: CUDA-event times (3 maps), the per-kernel
# launch list (config-5 and config-4 maps), fold event traces, and one
# ncu --set full capture of each smoothing kernel on the config-5 map.
mkdir -p gpurun_out
python tools/smooth_probe.py > gpurun_out/sp5.json
python tools/smooth_probe.py --nbins 1 --nv 1024 --nu 1024 --sigma 25.6 > gpurun_out/sp4.json
python tools/smooth_probe.py --nbins 8 --nv 512 --nu 512 --sigma 24 > gpurun_out/sp3.json
bash tools/gpu/smooth_breakdown.sh > /dev/null 2>&1
HB_B200_LIB=paper_1504_02687_b200/_lib/var_trace/libhb_b200.so python tools/fold_trace.py > gpurun_out/fold_trace4.txt 2>&1
HB_B200_LIB=paper_1504_02687_b200/_lib/var_trace/libhb_b200.so python tools/fold_trace.py --nbins 4 --nv 2047 --nu 2048 > gpurun_out/fold_trace5.txt 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"fold_kernel|box_kernel|hwin|vwin" -s 4 -c 4 \
  -o gpurun_out/prof_smooth5 -f python tools/smooth_probe.py --reps 1 > gpurun_out/ncu_smooth.log 2>&1; echo ncu rc=$?

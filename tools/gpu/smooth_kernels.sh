mkdir -p gpurun_out
for v in default rowscalar; do
  if [ "$v" != default ]; then export HB_B200_LIB=paper_1504_02687_b200/_lib/var_$v/libhb_b200.so; else unset HB_B200_LIB; fi
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/smooth_probe.py --nbins 1 --nv 1024 --nu 1024 --sigma 25.6 --reps 1 2>/dev/null | grep -v "^==" > gpurun_out/sk_$v.csv
done

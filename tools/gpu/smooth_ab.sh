mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for v in default rowscalar; do
  if [ "$v" != default ]; then export HB_B200_LIB=paper_1504_02687_b200/_lib/var_$v/libhb_b200.so; else unset HB_B200_LIB; fi
  echo "== $v"
  timeout 300 python tools/smooth_probe.py --nbins 1 --nv 1024 --nu 1024 --sigma 25.6
  timeout 300 python tools/smooth_probe.py
  timeout 300 python tools/smooth_probe.py --nbins 1 --nv 256 --nu 255 --sigma 16
done

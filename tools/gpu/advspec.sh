mkdir -p gpurun_out
for v in "" var_s2m3 var_s3m2 var_s2m4; do
  if [ -n "$v" ]; then export HB_B200_LIB=paper_1504_02687_b200/_lib/$v/libhb_b200.so; else unset HB_B200_LIB; fi
  echo "== variant ${v:-default}"
  timeout 300 python tools/kernel_probe.py --config 4 --iters 6 2>&1 | tail -1
done
unset HB_B200_LIB
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2

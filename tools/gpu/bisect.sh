for v in default rowlayout ty32 rowty32; do
  if [ "$v" != default ]; then export HB_B200_LIB=paper_1504_02687_b200/_lib/var_$v/libhb_b200.so; else unset HB_B200_LIB; fi
  echo "== $v"; timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "bit_exact or emit_splat" 2>&1 | tail -2
done

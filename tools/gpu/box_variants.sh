# hb_smooth on the config-5 map with box-kernel row-count variants (built by tools/build_variant.py)
for v in default "$@"; do
  if [ "$v" != default ]; then export HB_B200_LIB=paper_1504_02687_b200/_lib/var_$v/libhb_b200.so; else unset HB_B200_LIB; fi
  echo "$v $(python tools/smooth_probe.py)"
done

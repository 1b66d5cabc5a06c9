# hb_smooth on config 4's and config 5's maps for each built variant
for v in default "$@"; do
  if [ "$v" != default ]; then export HB_B200_LIB=paper_1504_02687_b200/_lib/var_$v/libhb_b200.so; else unset HB_B200_LIB; fi
  a=$(python tools/smooth_probe.py --nbins 1 --nv 1024 --nu 1024 --sigma 25.6 | python -c "import json,sys; print(round(json.load(sys.stdin)['ms']*1e3,1))")
  b=$(python tools/smooth_probe.py | python -c "import json,sys; print(round(json.load(sys.stdin)['ms']*1e3,1))")
  echo "$v cfg4_us=$a cfg5_us=$b"
done

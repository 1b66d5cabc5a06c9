# usage: variants.sh name1 name2 ...   (builds under paper_1504_02687_b200/_lib/var_<name>)
mkdir -p gpurun_out
for v in default "$@"; do
  if [ "$v" != default ]; then export HB_B200_LIB=paper_1504_02687_b200/_lib/var_$v/libhb_b200.so; else unset HB_B200_LIB; fi
  timeout 300 python tools/kernel_probe.py --config 4 --iters 6 > gpurun_out/probe_$v.json 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/probe_$v.json')); print('$v', {k:round(v,3) for k,v in d.items() if k.endswith('_ms')})"
done

mkdir -p gpurun_out
for v in on off on; do
  if [ "$v" = off ]; then export HB_STREAM_OUT=0; else unset HB_STREAM_OUT; fi
  timeout 900 python bench.py --steps 4 --warmup 3 --no-cpu-baseline > gpurun_out/e2e_$v.json 2>/dev/null
  python -c "
import json
d=json.loads([l for l in open('gpurun_out/e2e_$v.json') if l.startswith('{')][-1])
print('$v', 'value %.3e' % d['value'], 'e2e %.3e' % d['e2e']['value'], 's/step %.4f' % d['e2e']['s_per_step'])"
done

mkdir -p gpurun_out
for srt in none srcdst; do
  timeout 400 python tools/kernel_probe.py --config 4 --iters 6 --sort-edges $srt > gpurun_out/probe_sort_$srt.json 2>&1
  python - "$srt" <<'PY'
import json, sys
v = sys.argv[1]
try:
    d = json.load(open(f'gpurun_out/probe_sort_{v}.json'))
    print(v, {k: round(d[k], 3) for k in ('emit_only_ms','emit_segtab_ms','expand_ms','gf_flat_adv_ms','lap_count_ms','count_final_ms') if k in d}, d['segtab'])
except Exception as ex:
    print(v, 'failed', ex, open(f'gpurun_out/probe_sort_{v}.json').read()[-500:])
PY
done

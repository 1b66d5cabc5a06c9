mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "smooth" 2>&1 | tail -2
python tools/smooth_probe.py
python tools/smooth_probe.py --nbins 1 --nv 1024 --nu 1024 --sigma 25.6
bash tools/gpu/smooth_breakdown.sh > /dev/null 2>&1
for f in sk5 sk4; do echo "== $f"; python - "$f" <<'PY'
import csv,sys,collections
lines=[l for l in open(f"gpurun_out/{sys.argv[1]}.csv") if l.startswith('"')]
agg=collections.defaultdict(list)
for r in csv.DictReader(lines):
    if r.get("Metric Name")=="gpu__time_duration.sum" and "hb::" in r["Kernel Name"]:
        agg[r["Kernel Name"].split("(")[0].replace("void ","")].append(float(r["Metric Value"])/1000)
for k,v in agg.items(): print("  %-40s n=%2d mean %.1f us" % (k, len(v), sum(v)/len(v)))
PY
done
export HB_B200_LIB=paper_1504_02687_b200/_lib/var_trace/libhb_b200.so
python tools/fold_trace.py 2>&1 | grep -v "^  b" | grep -v "^strip" | tail -5
python tools/fold_trace.py --nbins 4 --nv 2047 --nu 2048 2>&1 | grep -v "^  b" | grep -v "^strip" | tail -5

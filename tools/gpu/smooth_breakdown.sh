# per-kernel launch list of one hb_smooth_counts call on the config-5 and config-4 maps
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/smooth_probe.py --reps 1 2>/dev/null | grep -v "^==" > gpurun_out/sk5.csv
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/smooth_probe.py --nbins 1 --nv 1024 --nu 1024 --sigma 25.6 --reps 1 2>/dev/null | grep -v "^==" > gpurun_out/sk4.csv
for f in sk5 sk4; do echo "== $f"; python - "$f" <<'PY'
import csv,sys
rows=list(csv.DictReader(open(f"gpurun_out/{sys.argv[1]}.csv")))
for r in rows:
    if r.get("Metric Name")=="gpu__time_duration.sum":
        print(r["ID"], r["Kernel Name"][:60], r["Metric Value"], r["Metric Unit"])
PY
done

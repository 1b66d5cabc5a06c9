# one bench line per BASELINE config on one B200 (configs 1-3 are parity/test cases)
mkdir -p gpurun_out
for c in 1 2 3; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/cfg${c}_line.json 2> gpurun_out/cfg${c}_line.err; echo cfg$c rc=$?
done

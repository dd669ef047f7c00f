# every BASELINE config through bench.py (device-resident value leg + live kernel timings)
for c in 0 2 3 4; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c$c.log 2>&1
  echo "config $c rc=$?"
  tail -1 gpurun_out/bench_c$c.log | cut -c1-600
done

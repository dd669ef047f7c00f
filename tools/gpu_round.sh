# Round measurement with the int8 fp64 default: full GPU suite, every config's bench, reference arm,
# parity report, launch list and ncu --set full of the c1 kernels (segmax, K1Q, kind::i8 Gram).
R=${1:-r01}
set -e; make -s -C paper_2401_13185_b200 >/dev/null; make -s -C oracle >/dev/null; set +e
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_${R}_default.log 2>&1; echo "bench default rc=$?"
for c in 0 2 4; do
  python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_${R}_c$c.log 2>&1; echo "bench c$c rc=$?"
done
CVG_FP64_KIND=dmma python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${R}_c1_dmma.log 2>&1; echo "bench c1 dmma rc=$?"
timeout 900 python tests/parity_report.py --out gpurun_out/parity_${R}.json > gpurun_out/parity.log 2>&1; echo "parity rc=$?"
python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${R}.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"segmax|reorder_q|gram_i8" -c 3 -o gpurun_out/prof_c1_i8_${R} \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_c1.log 2>&1; echo "ncu c1 rc=$?"

# Round measurement: every BASELINE config through bench.py, the reference arm, the
# launch list (ncu, cold/serialised), ncu --set full captures of the c1 Gram + K1 and the
# c2 epilogue (plain runs of the same commands exit 0 first), the paper-size P sweep and
# leave-one-out, and the per-config parity report.
# Usage (from the repo root, on the GPU box):  bash tools/gpu_measure.sh r01
R=${1:-r01}
set -e; make -s -C paper_2401_13185_b200 >/dev/null; set +e
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_${R}_default.log 2>&1; echo "bench default rc=$?"
for c in 0 2 3 4; do
  python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench_${R}_c$c.log 2>&1; echo "bench c$c rc=$?"
done
CVG_FP64_KIND=dmma python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${R}_c1_dmma.log 2>&1; echo "bench c1 dmma rc=$?"
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_${R}_ref.log 2>&1; echo "ref rc=$?"
python tools/p_sweep.py --out gpurun_out/p_sweep_${R}.jsonl > gpurun_out/p_sweep.log 2>&1; echo "p sweep rc=$?"
python tools/loo_bench.py --batch 4096 > gpurun_out/loo_${R}.log 2>&1; echo "loo rc=$?"
python tests/parity_report.py --out gpurun_out/parity_${R}.json > gpurun_out/parity.log 2>&1; echo "parity rc=$?"
python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${R}.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"segmax|reorder_q|gram_i8" -c 3 -o gpurun_out/prof_c1_${R} \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_c1.log 2>&1; echo "ncu c1 rc=$?"
python bench.py --config 2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none -k regex:"products_kernel|fold_stats" -c 2 -o gpurun_out/prof_c2_${R} \
  python bench.py --config 2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_c2.log 2>&1; echo "ncu c2 rc=$?"

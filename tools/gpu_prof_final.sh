# ncu of the final c1 path: launch list + --set full of the int8 kernels (plain run first).
R=${1:-r01}
set -e; make -s -C paper_2401_13185_b200 >/dev/null; set +e
python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${R}.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"segmax|reorder_q|gram_i8" -c 3 -o gpurun_out/prof_c1_${R} \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_c1.log 2>&1; echo "ncu c1 rc=$?"

# ncu --set full of the int8-slice fp64 path on configs[1] (segmax, K1Q, kind::i8 Gram) + the launch list.
R=${1:-r01}; S=${2:-7}
set -e; make -s -C paper_2401_13185_b200 >/dev/null; set +e
export CVG_FP64_KIND=i8 CVG_I8_SLICES=$S
python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/plain_i8.log 2>&1; echo "plain rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_i8_${R}.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_i8.log 2>&1; echo "ncu launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"segmax|reorder_q|gram_i8" -c 3 -o gpurun_out/prof_i8_${R} \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_i8.log 2>&1; echo "ncu full rc=$?"

# c1 bench + one ncu --set full capture of the fp64 Gram (plain run first, as the recipe requires)
R=${1:-r01}
set -e; make -s -C paper_2401_13185_b200 >/dev/null; set +e
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "c0 or c1_shape or c4 or edges" 2>&1 | tail -1
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/plain.log 2>&1; echo "plain rc=$?"; tail -1 gpurun_out/plain.log | cut -c1-200
ncu --set full --clock-control none --import-source on -k regex:"gram_f64" -c 1 -o gpurun_out/prof_gram_${R} \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_gram.log 2>&1; echo "ncu rc=$?"

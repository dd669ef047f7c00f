set -e; make -s -C paper_2401_13185_b200 >/dev/null; set +e
python bench.py --config 3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/plain3.log 2>&1; echo "plain rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"gram_f16s" -c 1 -o gpurun_out/prof_c3_f16b \
  python bench.py --config 3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_c3.log 2>&1; echo "ncu rc=$?"

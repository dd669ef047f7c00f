set -e; make -s -C paper_2401_13185_b200 >/dev/null; set +e
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "accumulation_range or nonfinite" 2>&1 | tail -2
python bench.py --config 3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/plain3.log 2>&1; echo "plain rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"reorder_split_h" -c 1 -o gpurun_out/prof_k1h_b \
  python bench.py --config 3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_k1h.log 2>&1; echo "ncu rc=$?"

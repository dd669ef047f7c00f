timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
python bench.py --config 3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"reorder_split|gram_tf32" -c 2 -o gpurun_out/prof_c3 python bench.py --config 3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_c3.log 2>&1; echo ncu rc=$?

python bench.py --config 3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"reorder_split" -c 1 -o gpurun_out/prof_k1t python bench.py --config 3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_k1t.log 2>&1; echo ncu rc=$?

set -e; make -s -C paper_2401_13185_b200 >/dev/null; set +e
python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"gram_f64_fused" -c 1 -o gpurun_out/prof_fused python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_fused.log 2>&1; echo ncu rc=$?
tail -2 gpurun_out/ncu_fused.log

# one ncu --set full capture of the Gram kernel (plain run first, as the recipe requires)
python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"gram_f64" -c 1 -o gpurun_out/prof_gram python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_gram.log 2>&1; echo ncu rc=$?
tail -2 gpurun_out/ncu_gram.log

set -x
nproc
python -m pytest tests/test_cpp_header.py -q -m gpu -s 2>&1 | tail -25 > gpurun_out/cpp_tests.log
python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; echo bench rc=$?
tail -3 gpurun_out/bench.log
python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1; echo ncu1 rc=$?
ncu --set full --clock-control none --import-source on -k regex:"gram_f64|products_kernel|reorder_kernel" -c 3 -o gpurun_out/prof_r01 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1; echo ncu2 rc=$?
tail -5 gpurun_out/ncu_full.log

set -x
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -5 > gpurun_out/gpu_tests.log
cat gpurun_out/gpu_tests.log
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench.log

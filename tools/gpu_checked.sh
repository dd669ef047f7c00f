# Bounds-checked build (CVG_DCHECK device assertions) through the whole GPU suite.
set -e; make -s -C paper_2401_13185_b200 >/dev/null; make -s -C paper_2401_13185_b200 CHECKED=1 >/dev/null; set +e
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "loo_beyond" 2>&1 | grep -E "Error|error|passed|failed|assert" | head -5
CVG_LIB_VARIANT=checked timeout 1800 python -m pytest tests -q -m gpu 2>&1 | tail -15 > gpurun_out/checked_suite.txt
tail -3 gpurun_out/checked_suite.txt
CVG_LIB_VARIANT=checked timeout 900 python bench.py --config 1 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/checked_bench.log 2>&1; echo "checked bench c1 rc=$?"
CVG_LIB_VARIANT=checked timeout 900 python bench.py --config 3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/checked_bench3.log 2>&1; echo "checked bench c3 rc=$?"
CVG_LIB_VARIANT=checked timeout 900 python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/checked_bench4.log 2>&1; echo "checked bench c4 rc=$?"

set -e; make -s -C paper_2401_13185_b200 >/dev/null; set +e
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "row_mapped or sharded or staged" 2>&1 | grep -E "Error|error|passed|failed|assert" | head -8
timeout 600 python bench.py --config 1 --steps 3 --warmup 3 --no-cpu-baseline --e2e-path sharded > gpurun_out/ba.log 2>&1
python -c "
import json; d = json.loads(open('gpurun_out/ba.log').read().strip().splitlines()[-1])
print('c1 sharded e2e', d['e2e']['ms_per_step'])" || tail -5 gpurun_out/ba.log

set -e; make -s -C paper_2401_13185_b200 >/dev/null; set +e
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "tf32 or c3 or fp32 or tile_edges" 2>&1 | grep -E "Error|error|passed|failed|assert" | head -12
for env in "CVG_TF32_PRESPLIT=0" "CVG_TF32_PRESPLIT=1"; do
env $env timeout 300 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bt.log 2>&1
python -c "
import json; d = json.loads(open('gpurun_out/bt.log').read().strip().splitlines()[-1])
print('c3 $env', d['ms_per_step'], d['value'], d['kernels_ms_per_step'])" || tail -5 gpurun_out/bt.log
done

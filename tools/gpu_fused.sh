set -e; make -s -C paper_2401_13185_b200 >/dev/null; set +e
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "fused or small_segments or c1_shape or c4 or c0" 2>&1 | grep -E "Error|error|passed|failed|assert" | head -12
for c in 1 2 4; do
for u in 0 1; do
CVG_UNFUSED=$u timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bf.log 2>&1
python -c "
import json; d = json.loads(open('gpurun_out/bf.log').read().strip().splitlines()[-1])
print('c$c unfused=$u', d['ms_per_step'], d['value'], d['kernels_ms_per_step'])" || tail -5 gpurun_out/bf.log
done; done

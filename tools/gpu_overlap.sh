set -e; make -s -C paper_2401_13185_b200 >/dev/null; set +e
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "overlap or c4 or c1_shape" 2>&1 | grep -E "Error|error|passed|failed|assert" | head -5
for c in 1 2 4; do
for ov in 0 4 0 4 8; do
CVG_OVERLAP=$ov timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bov.log 2>&1
python -c "
import json; d = json.loads(open('gpurun_out/bov.log').read().strip().splitlines()[-1])
print('c$c overlap=$ov', d['ms_per_step'], d['kernels_ms_per_step'])" || tail -5 gpurun_out/bov.log
done; done

set -e; make -s -C paper_2401_13185_b200 >/dev/null; set +e
timeout 1200 python -m pytest tests -q -m gpu -x -k "tile_edges or c0 or c1_shape or c4 or loo or bitwise" 2>&1 | grep -E "Error|error|passed|failed|assert" | head -12
for c in 1 2 4; do
timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bo.log 2>&1
python -c "
import json; d = json.loads(open('gpurun_out/bo.log').read().strip().splitlines()[-1])
print('c$c', d['ms_per_step'], d['kernels_ms_per_step'])" || tail -5 gpurun_out/bo.log
done

set -e; make -s -C paper_2401_13185_b200 >/dev/null; set +e
timeout 1200 python -m pytest tests -q -m gpu 2>&1 | grep -E "^E|FAILED|passed|failed" | head -6
for c in 1 2 3 4; do
timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bt.log 2>&1
python -c "
import json; d = json.loads(open('gpurun_out/bt.log').read().strip().splitlines()[-1])
k=d['kernels_ms_per_step']; print('c$c', d['ms_per_step'], 'tree', k['tree_sum'], 'gram', k['gram'])" || tail -5 gpurun_out/bt.log
done

set -e; make -s -C paper_2401_13185_b200 >/dev/null; set +e
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | grep -E "^E |FAILED|passed|failed" | head -5
for c in 1 2 4; do
timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bd.log 2>&1
python -c "
import json; d = json.loads(open('gpurun_out/bd.log').read().strip().splitlines()[-1])
k=d['kernels_ms_per_step']; print('c$c', d['ms_per_step'], 'gram', k['gram'], d['roofline']['executed_frac'])" || tail -5 gpurun_out/bd.log
done

set -e; make -s -C paper_2401_13185_b200 >/dev/null; set +e
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | grep -E "Error|error|passed|failed|assert" | head -12
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bc3.log 2>&1
python -c "
import json; d = json.loads(open('gpurun_out/bc3.log').read().strip().splitlines()[-1])
print('c3', d['ms_per_step'], d['kernels_ms_per_step'], d['e2e']['ms_per_step'])" || tail -5 gpurun_out/bc3.log

set -e; make -s -C paper_2401_13185_b200 >/dev/null; set +e
for ch in 32768 16384 12288 8192; do
CVG_CHUNK_ROWS=$ch timeout 900 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bc.log 2>&1
python -c "
import json; d = json.loads(open('gpurun_out/bc.log').read().strip().splitlines()[-1])
print('c3 chunk $ch', d['ms_per_step'], d['kernels_ms_per_step'])" || tail -5 gpurun_out/bc.log
done

set -e; make -s -C paper_2401_13185_b200 >/dev/null; set +e
for ch in 32768 8192 4096 2048; do
CVG_CHUNK_ROWS=$ch python bench.py --config 1 --steps 5 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bch.log 2>&1
python -c "
import json; d = json.loads(open('gpurun_out/bch.log').read().strip().splitlines()[-1])
print('chunk $ch', d['ms_per_step'], d['kernels_ms_per_step'])"
done
for ch in 32768 8192 2048; do
CVG_CHUNK_ROWS=$ch python bench.py --config 3 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/bch.log 2>&1
python -c "
import json; d = json.loads(open('gpurun_out/bch.log').read().strip().splitlines()[-1])
print('c3 chunk $ch', d['ms_per_step'], d['kernels_ms_per_step'])"
done

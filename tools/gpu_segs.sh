set -e; make -s -C paper_2401_13185_b200 >/dev/null; set +e
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "shared_folds or c4 or multi_seg or small_segments or staged or c3 or c1_shape" 2>&1 | grep -E "Error|error|passed|failed|assert" | head -5
for c in 1 4; do
for ch in 32768 16384 8192 5120; do
CVG_CHUNK_ROWS=$ch timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bs.log 2>&1
python -c "
import json; d = json.loads(open('gpurun_out/bs.log').read().strip().splitlines()[-1])
k=d['kernels_ms_per_step']; print('c$c chunk $ch', d['ms_per_step'], 'gram', k['gram'], 'tree', k['tree_sum'])" || tail -5 gpurun_out/bs.log
done; done
for ch in 12288 8192 6144; do
CVG_CHUNK_ROWS=$ch timeout 600 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bs.log 2>&1
python -c "
import json; d = json.loads(open('gpurun_out/bs.log').read().strip().splitlines()[-1])
k=d['kernels_ms_per_step']; print('c3 chunk $ch', d['ms_per_step'], 'gram', k['gram'], 'tree', k['tree_sum'])" || tail -5 gpurun_out/bs.log
done

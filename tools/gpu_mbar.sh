set -e; make -s -C paper_2401_13185_b200 >/dev/null; set +e
CVG_GRAM_STAGES=6 timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "c0 or c1_shape or c4 or tile_edges or loo" 2>&1 | grep -E "Error|error|passed|failed|assert" | head -5
for c in 1 2 4; do
for mb in 3 6 3 6; do
CVG_GRAM_STAGES=$mb timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bm.log 2>&1
python -c "
import json; d = json.loads(open('gpurun_out/bm.log').read().strip().splitlines()[-1])
print('c$c stages=$mb', d['ms_per_step'], d['kernels_ms_per_step']['gram'])" || tail -5 gpurun_out/bm.log
done; done

set -e; make -s -C paper_2401_13185_b200 >/dev/null; set +e
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "c3 or fp32 or f32" 2>&1 | tail -1
for i in 1 2; do
timeout 600 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bk.log 2>&1
python -c "
import json; d = json.loads(open('gpurun_out/bk.log').read().strip().splitlines()[-1])
print('c3', d['ms_per_step'], d['kernels_ms_per_step'], d['hbm_rooflines']['reorder'])" || tail -5 gpurun_out/bk.log
done

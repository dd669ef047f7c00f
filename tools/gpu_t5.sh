set -e; make -s -C paper_2401_13185_b200 >/dev/null
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "f32 or c3 or fp32" 2>&1 | grep -E "AssertionError|passed|failed" | head -5
python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bq_c3.log 2>&1; echo bench c3 rc=$?
python -c "
import json; d = json.loads(open('gpurun_out/bq_c3.log').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['kernels_ms_per_step'], 'exec_frac', d['roofline']['executed_frac'], 'reorder', d['hbm_rooflines']['reorder']['achieved_gbs'])"

timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "c0 or c1_shape or tile_edges or c3 or fp32 or staged" 2>&1 | tail -2
for c in 1 3; do
python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bq_c$c.log 2>&1; echo bench c$c rc=$?
python -c "
import json; d = json.loads(open('gpurun_out/bq_c$c.log').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['kernels_ms_per_step'], 'exec_frac', d['roofline']['executed_frac'], 'reorder', d['hbm_rooflines']['reorder']['achieved_gbs'])"
done

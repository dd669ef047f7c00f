set -e; make -s -C paper_2401_13185_b200 >/dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_reference_kats.py -q -x -m gpu 2>&1 | grep -E "Error|passed|failed" | head -5
for c in 1 4; do
python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bq_c$c.log 2>&1; echo bench c$c rc=$?
python -c "
import json; d = json.loads(open('gpurun_out/bq_c$c.log').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['kernels_ms_per_step'], 'exec_frac', d['roofline']['executed_frac'], 'alg frac', d['roofline']['frac'])"
done

# quick check: parity subset + bench line
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "c0 or c1_shape or tile_edges or staged or nonfinite" 2>&1 | tail -2
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_quick.log 2>&1; echo bench rc=$?
python -c "
import json; d = json.loads(open('gpurun_out/bench_quick.log').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['kernels_ms_per_step'], 'gram_exec_frac', d['roofline']['executed_frac'])"

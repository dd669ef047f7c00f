set -e; make -s -C paper_2401_13185_b200 >/dev/null; set +e
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | grep -E "^E |FAILED|passed|failed" | head -5
for c in 1 2; do
timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/be.log 2>&1
python -c "
import json; d = json.loads(open('gpurun_out/be.log').read().strip().splitlines()[-1])
k=d['kernels_ms_per_step']; print('c$c', d['ms_per_step'], 'products', k['products'], d['hbm_rooflines']['epilogue']['achieved_gbs'])" || tail -5 gpurun_out/be.log
done
timeout 900 python tools/loo_bench.py --batch 4096 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('loo', d['ms'], d['output_write_gbs'], d['worst_rel_err_vs_numpy_direct'])"

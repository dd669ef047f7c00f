# fp32 path A/B: scaled-fp16 kind::f16 (default) vs 3xTF32 kind::tf32 -- parity and c3 timing
set -e; make -s -C paper_2401_13185_b200 >/dev/null; set +e
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "c3 or fp32 or tile_edges or small_segments or mapped or rank_plans or staged or fuzz" 2>&1 | tail -3
timeout 300 python tests/parity_report.py --cases 3 2>&1 | tail -4
CVG_FP32_KIND=tf32 timeout 300 python tests/parity_report.py --cases 3 2>&1 | tail -4
python bench.py --config 3 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/f16_c3.log 2>&1; echo "f16 rc=$?"
CVG_FP32_KIND=tf32 python bench.py --config 3 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/tf32_c3.log 2>&1; echo "tf32 rc=$?"
for f in f16_c3 tf32_c3; do tail -1 gpurun_out/$f.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f', d['ms_per_step'], d.get('kernels_ms_per_step'))"; done

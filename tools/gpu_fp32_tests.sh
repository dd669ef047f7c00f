# fp32 path: all fp32-relevant GPU tests + c3 bench
set -e; make -s -C paper_2401_13185_b200 >/dev/null; set +e
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "fp32 or c3 or tile_edges or fuzz or tf32 or small_segments or mapped or rank_plans or staged or nonfinite" 2>&1 | tail -3
python bench.py --config 3 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/f16_c3.log 2>&1; echo "f16 rc=$?"
tail -1 gpurun_out/f16_c3.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['executed_tflops'], d['roofline']['frac'], d.get('kernels_ms_per_step'), d['hbm_rooflines']['reorder'])"

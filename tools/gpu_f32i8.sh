set -e; make -s -C paper_2401_13185_b200 >/dev/null; make -s -C oracle >/dev/null; set +e
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -s -k "fp32_i8_kind" 2>&1 | grep -E "worst|passed|failed|^E " | tail -8
for kd in "i8 4" "i8 3" "f16 4"; do set -- $kd
  CVG_FP32_KIND=$1 CVG_I8_SLICES_F32=$2 python bench.py --config 3 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/f32.log 2>&1
  tail -1 gpurun_out/f32.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2', d['ms_per_step'], d['kernels_ms_per_step'])"
done

# int8-slice fp64 Gram (CVG_FP64_KIND=i8): parity subset against the truth, then c1/c2/c4 timing A/B vs DMMA.
set -e; make -s -C paper_2401_13185_b200 >/dev/null; make -s -C oracle >/dev/null; set +e
export CVG_FP64_KIND=i8
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -s -k "c1_shape or c0_full or tile_edges" 2>&1 | grep -E "worst|passed|failed|Error|error" | head -30
for S in 7 6; do
  CVG_I8_SLICES=$S python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/i8_c1_s$S.log 2>&1; echo "i8 S=$S c1 rc=$?"
  tail -1 gpurun_out/i8_c1_s$S.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d.get('kernels_ms_per_step'))"
done
CVG_FP64_KIND=dmma python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/dmma_c1.log 2>&1
tail -1 gpurun_out/dmma_c1.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('dmma', d['ms_per_step'], d.get('kernels_ms_per_step'))"
python tools/fp64_peaks.py int8 2>&1 | tail -1

set -e; make -s -C paper_2401_13185_b200 OUT=_build_sq >/dev/null; make -s -C oracle >/dev/null; set +e
echo "tests: $(CVG_LIB_VARIANT=sq timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k 'c1_full_size or c1_shape or c0_full or c4_contig or extreme or staged or fuzz' 2>&1 | tail -1)"
for v in sq; do for c in 1 4; do
  CVG_LIB_VARIANT=$v python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sq.log 2>&1
  tail -1 gpurun_out/sq.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('[$v] c$c', d['ms_per_step'], d['kernels_ms_per_step']['gram'])"
done; done

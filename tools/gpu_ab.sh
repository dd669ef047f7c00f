# Quick A/B of the current tree: parity subset + c1/c4 benches (S=7 and S=6).
set -e; make -s -C paper_2401_13185_b200 >/dev/null; make -s -C oracle >/dev/null; set +e
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "c1_shape or c0_full or c4_contig or tile_edges or extreme or staged or fuzz" 2>&1 | tail -1
for S in 7 6; do for c in 1 4; do
  CVG_I8_SLICES=$S python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab.log 2>&1
  tail -1 gpurun_out/ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('S $S c$c', d['ms_per_step'], d['kernels_ms_per_step']['gram'], d['kernels_ms_per_step']['reorder'])"
done; done

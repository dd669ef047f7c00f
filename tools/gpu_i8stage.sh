set -e; make -s -C paper_2401_13185_b200 >/dev/null; make -s -C oracle >/dev/null; set +e
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "c1_shape or c0_full or c4_contig or tile_edges or extreme or staged or fuzz" 2>&1 | tail -1
for ks in 32 64; do for S in 7 6; do for c in 1 4; do
  CVG_I8_STAGE_ROWS=$ks CVG_I8_SLICES=$S python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/st.log 2>&1
  tail -1 gpurun_out/st.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ks $ks S $S c$c', d['ms_per_step'], d['kernels_ms_per_step']['gram'], d['kernels_ms_per_step']['reorder'])"
done; done; done

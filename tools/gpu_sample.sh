set -e; make -s -C paper_2401_13185_b200 >/dev/null; make -s -C oracle >/dev/null; set +e
K="c1_shape or c0_full or c2_shape or c4_contig or tile_edges or extreme or staged or fuzz or rank_plans or mapped or minimum or nonfinite"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "$K" 2>&1 | tail -1
CVG_I8_SAMPLE=4096 timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "c1_shape or c0_full or c4_contig or extreme or staged or fuzz or nonfinite" 2>&1 | tail -1
for c in 1 2 4; do
  python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/smp.log 2>&1
  tail -1 gpurun_out/smp.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c$c', d['ms_per_step'], d['kernels_ms_per_step'])"
done

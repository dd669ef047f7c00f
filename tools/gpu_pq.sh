set -e; make -s -C paper_2401_13185_b200 >/dev/null; make -s -C paper_2401_13185_b200 OUT=_build_pq2 EXTRA=-DCVG_K1Q_PQ=2 >/dev/null; set +e
CVG_LIB_VARIANT=pq2 timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "c1_shape or c4_contig or staged or fuzz or extreme" 2>&1 | tail -1
for v in "" pq2; do for c in 1 4; do
  CVG_LIB_VARIANT=$v python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/pq.log 2>&1
  tail -1 gpurun_out/pq.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('[$v] c$c', d['ms_per_step'], d['kernels_ms_per_step']['reorder'], d['kernels_ms_per_step']['gram'])"
done; done

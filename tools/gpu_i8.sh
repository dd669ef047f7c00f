# int8-slice fp64 Gram (CVG_FP64_KIND=i8): parity subset against the truth, then c1/c2/c4 timing A/B vs DMMA.
set -e; make -s -C paper_2401_13185_b200 >/dev/null; make -s -C oracle >/dev/null; set +e
export CVG_FP64_KIND=i8
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -s -k "c1_shape or c0_full or c2_shape or c4_contig or tile_edges or staged or rank_plans or row_sharded_host_entry_single or mapped or fuzz or minimum" 2>&1 | grep -E "worst|passed|failed|Error|error" | tail -12
for c in 1 2 4; do
  python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/i8_c$c.log 2>&1; echo "i8 c$c rc=$?"
  tail -1 gpurun_out/i8_c$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d.get('kernels_ms_per_step'))"
done
CVG_I8_SLICES=6 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/i8_c1_s6.log 2>&1
tail -1 gpurun_out/i8_c1_s6.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('S6', d['ms_per_step'], d.get('kernels_ms_per_step'))"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"segmax|reorder_q|gram_i8" -c 3 \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e 2>&1 | grep -E "segmax|reorder_q|gram_i8|duration|bytes" | head -20

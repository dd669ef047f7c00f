set -e; make -s -C paper_2401_13185_b200 >/dev/null; set +e
export CVG_FP64_KIND=i8
python tools/i8_debug.py 20000 500 10 100 | tail -1
python tools/i8_debug.py 3000 130 3 3 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "c1_shape or c0_full or c2_shape or c4_contig or tile_edges or staged or rank_plans or mapped or fuzz" 2>&1 | tail -1
for c in 1 4; do python bench.py --config $c --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/i8_c$c.log 2>&1
tail -1 gpurun_out/i8_c$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c$c', d['ms_per_step'], d.get('kernels_ms_per_step'))"; done
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"segmax|reorder_q" -c 2 \
  python bench.py --config 4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e 2>&1 | grep -E "duration|bytes" | head -20

set -e; make -s -C paper_2401_13185_b200 >/dev/null; make -s -C oracle >/dev/null; set +e
echo "A: $(timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k 'c1_full_size or c1_shape or c0_full or c2_shape or c4_contig or extreme or staged or fuzz' 2>&1 | tail -1)"
timeout 600 python tests/parity_report.py --out gpurun_out/parity_q.json > gpurun_out/parity_q.log 2>&1; grep -E "normalized" gpurun_out/parity_q.log | grep -v fp32 | awk '{print $0}' | sort -g -k7 | tail -3
for c in 1 4; do python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/q.log 2>&1
tail -1 gpurun_out/q.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c$c', d['ms_per_step'], d['kernels_ms_per_step'])"; done

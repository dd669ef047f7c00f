set -e; make -s -C paper_2401_13185_b200 >/dev/null; set +e
for cr in 24576 32768 49152 65536; do
  CVG_CHUNK_ROWS=$cr python bench.py --config 3 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/cr_$cr.log 2>&1
  tail -1 gpurun_out/cr_$cr.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('[$cr]', d['ms_per_step'], d.get('kernels_ms_per_step'))"
done

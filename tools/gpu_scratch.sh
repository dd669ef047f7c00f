set -e; make -s -C paper_2401_13185_b200 >/dev/null; set +e
for v in "" nodrain; do
  CVG_LIB_VARIANT=$v python bench.py --config 3 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/exp_$v.log 2>&1; echo "$v rc=$?"
  tail -1 gpurun_out/exp_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('[$v]', d['ms_per_step'], d.get('kernels_ms_per_step'))"
done

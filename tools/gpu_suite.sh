# Full GPU suite + c0/c1 benches (current tree).
set -e; make -s -C paper_2401_13185_b200 >/dev/null; make -s -C oracle >/dev/null; set +e
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log; grep -E "^FAILED" gpurun_out/pytest_gpu.log | head
for c in 0 1; do python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/suite_c$c.log 2>&1
tail -1 gpurun_out/suite_c$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c$c', d['ms_per_step'], d['kernels_ms_per_step'], d['e2e']['ms_per_step'])"; done
python -c "import __graft_entry__ as g; g.smoke()"

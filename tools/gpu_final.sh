# Final round record: full GPU suite, the bench lines (current bench.py), smoke, checked build.
set -e; make -s -C paper_2401_13185_b200 >/dev/null; make -s -C oracle >/dev/null; set +e
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log; grep -E "^FAILED" gpurun_out/pytest_gpu.log | head
python bench.py --steps 10 --warmup 3 > gpurun_out/final_c1.log 2>&1; echo "bench c1 rc=$?"
for c in 2 4; do python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/final_c$c.log 2>&1; echo "bench c$c rc=$?"; done
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
bash tools/gpu_checked.sh

set -e; make -s -C paper_2401_13185_b200 >/dev/null; set +e
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_plain.log 2>&1 && \
timeout 600 compute-sanitizer --tool memcheck --leak-check no --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -k "c0_full or loo or tile_edges or staged or rank_plans" > gpurun_out/memcheck.log 2>&1; echo memcheck rc=$?
grep -E "ERROR SUMMARY|passed|failed|Invalid|out of bounds" gpurun_out/memcheck.log | head -20

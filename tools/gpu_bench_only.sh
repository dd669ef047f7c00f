set -e; make -s -C paper_2401_13185_b200 >/dev/null; set +e
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r01_full.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench_r01_full.log

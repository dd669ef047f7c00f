set -e; make -s -C paper_2401_13185_b200 >/dev/null; set +e
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r01_full.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench_r01_full.log | cut -c1-300
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_r01_ref.log 2>&1; echo ref rc=$?
tail -1 gpurun_out/bench_r01_ref.log | cut -c1-300
python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01b.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1; echo ncu1 rc=$?
python bench.py --config 3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"gram_tf32|reorder_split" -c 2 -o gpurun_out/prof_c3_r01 python bench.py --config 3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_c3.log 2>&1; echo ncu2 rc=$?

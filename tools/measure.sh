#!/bin/bash
# One measurement pass on a B200 (run under gpurun): bench lines of every BASELINE config and the reference
# arm, the c1 launch list, and ncu --set full captures of the int8 Gram (lean) and the direct-store cut.
# Outputs under gpurun_out/m/ (copied into profiles/ by hand after reading).
set -u
O=gpurun_out/m
mkdir -p $O
python bench.py --steps 20 --warmup 5 > $O/bench_c1.jsonl 2> $O/bench_c1.err
for c in 0 2 3 4; do
  python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c$c.jsonl 2> $O/bench_c$c.err
done
CVG_I8_OVERLAP=0 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/bench_c1_serial.jsonl 2> $O/bench_c1_serial.err
CVG_I8_OVERLAP=0 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_c4_serial.jsonl 2> $O/bench_c4_serial.err
python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference_arm.jsonl 2> $O/bench_reference_arm.err
# launch list (serialised, cold cache: shares only), then the full captures
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/plain.log 2>&1 &&
  ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'gram_i8_kernel|reorder_q_kernel' -s 2 -c 2 -f \
  -o $O/c1_cut_gram python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_full.log 2>&1
ls -la $O

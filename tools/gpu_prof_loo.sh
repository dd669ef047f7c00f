set -e; make -s -C paper_2401_13185_b200 >/dev/null; set +e
python tools/loo_bench.py --batch 4096 --reps 1 > gpurun_out/loo_plain.log 2>&1; echo "plain rc=$?"
ncu --set full --clock-control none -k regex:"products_kernel" -c 1 -s 20 -o gpurun_out/prof_loo python tools/loo_bench.py --batch 4096 --reps 1 > gpurun_out/ncu_loo.log 2>&1; echo "ncu rc=$?"

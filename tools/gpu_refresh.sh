# Refresh after the fp16 Gram landed: full GPU suite, default + c3 benches, parity report,
# and an ncu --set full capture of the c3 kernels (K1H + kind::f16 Gram).
R=${1:-r01}
set -e; make -s -C paper_2401_13185_b200 >/dev/null; make -s -C oracle >/dev/null; set +e
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_${R}_default.log 2>&1; echo "bench default rc=$?"
python bench.py --config 3 --steps 5 --warmup 3 > gpurun_out/bench_${R}_c3.log 2>&1; echo "bench c3 rc=$?"
timeout 900 python tests/parity_report.py --out gpurun_out/parity_${R}.json > gpurun_out/parity.log 2>&1; echo "parity rc=$?"
bash tools/gpu_prof_c3.sh $R

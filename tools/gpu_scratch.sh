set -e; make -s -C paper_2401_13185_b200 >/dev/null; set +e
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "accumulation_range" 2>&1 | grep -v "^$" | tail -30
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "(fp32 or c3 or tile_edges or fuzz or tf32 or small_segments or mapped or rank_plans or staged or nonfinite) and not accumulation_range" 2>&1 | tail -3

timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "c2_shape" 2>&1 | grep -E "^E " | head -12

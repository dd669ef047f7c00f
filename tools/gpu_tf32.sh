timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -s -k "f32 or c3 or fp32" 2>&1 | tail -30

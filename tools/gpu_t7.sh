set -e; make -s -C paper_2401_13185_b200 >/dev/null
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | grep -E "Error|error|passed|failed|assert" | head -12

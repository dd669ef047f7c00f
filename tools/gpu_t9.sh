set -e; make -s -C paper_2401_13185_b200 >/dev/null; set +e
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | grep -E "Error|error|passed|failed|assert" | head -8
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1

export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | grep -E "^E|passed|failed" | head -12
echo "== config 1"; timeout 300 python tools/mv_time.py 1 2>&1 | tail -2

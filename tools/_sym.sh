export PYTHONUNBUFFERED=1
timeout 900 python -m pytest tests/test_gpu_matvec.py tests/test_gpu_symmetric.py tests/test_gpu_properties.py -x -q 2>&1 | grep -E "^E|passed|failed" | head -12
timeout 800 python tools/e2e_probe.py 2>&1 | tail -6

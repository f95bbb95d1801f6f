cd $GRAFT_REPO_ROOT
timeout 120 python -m pytest tests/test_gpu_matvec.py -q -x 2>&1 | tail -2
H2B_DIAG_FWD_ONLY=1 timeout 120 python tools/mv_trace.py 2>&1 | grep -E "forward|climb" | head -14
timeout 120 python tools/mv_time.py 2>&1 | tail -1

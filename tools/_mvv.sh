cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_matvec.py -q -x 2>&1 | tail -2
for i in 1 2; do timeout 300 python tools/mv_time.py 2>&1 | tail -1; done
timeout 300 python tools/mv_trace.py 2>&1 | grep -v "^\s*$" | grep -v Warn | grep -v "print(f" | grep -v climb | head -8

cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_matvec.py -q -x 2>&1 | tail -2
for v in "0.2 0.5" "0.1 0.5" "0.3 0.5" "0.2 0.6" "0.2 0.4" "0.1 0.7"; do set -- $v; echo -n "A1=$1 A2=$2: "; H2B_NEAR_A1=$1 H2B_NEAR_A2=$2 timeout 300 python tools/mv_time.py 2>&1 | tail -1; done
timeout 300 python tools/mv_trace.py 2>&1 | grep -v "^\s*$" | grep -v Warn | grep -v "print(f" | grep -v "ph = "

cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_matvec.py -q -x 2>&1 | tail -2
for v in 0.7 0.8 0.6; do echo -n "split=$v: "; H2B_NEAR_SPLIT=$v timeout 300 python tools/mv_time.py 2>&1 | tail -1; done

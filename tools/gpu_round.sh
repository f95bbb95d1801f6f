set -x
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r02w_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02w_pytest.log
tail -n 3 gpurun_out/r02w_pytest.log
for c in 1 2s 3; do for m in 0 0.2 0.4; do echo "== $c mix $m"; H2B_FWD_MIX=$m timeout 400 python tools/mv_time.py $c 2>&1 | grep -E "^matvec"; done; done > gpurun_out/r02w_mv.txt 2>&1
grep -E "^== |^matvec" gpurun_out/r02w_mv.txt

# Session check on one B200 (run under gpurun): matvec tests, task trace, timings.
R=${1:-r02af}
OUT=gpurun_out
mkdir -p $OUT
set -x
timeout 1500 python -m pytest tests/test_gpu_matvec.py tests/test_gpu_sharded.py tests/test_gpu_parity_large.py tests/test_gpu_symmetric.py tests/test_gpu_dropin.py -m gpu -q -x > $OUT/${R}_pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/${R}_pytest.log
timeout 900 python tools/mv_trace.py 3 > $OUT/${R}_trace.txt 2>&1
for c in 1 2 3; do timeout 900 python tools/mv_time.py $c 2>&1 | grep -v "^plan" >> $OUT/${R}_mvtime.txt; done
tail -n 3 $OUT/${R}_pytest.log; head -8 $OUT/${R}_trace.txt; tail -5 $OUT/${R}_mvtime.txt

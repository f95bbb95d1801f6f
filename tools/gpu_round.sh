R=${1:-r02bb}
OUT=gpurun_out
mkdir -p $OUT
set -x
V=$PWD/paper_2001_05523_b200/_lib/variants
for c in 1 3; do H2B_LIB_PATH=$V/dbg_cur.so timeout 300 python tools/ll_debug.py $c 2>&1 | grep "stuck\|launch" > $OUT/${R}_lldebug_$c.txt; done
cat $OUT/${R}_lldebug_*.txt
if grep -q "stuck addr 0x0 .*abandoned 0" $OUT/${R}_lldebug_1.txt && grep -q "stuck addr 0x0 .*abandoned 0" $OUT/${R}_lldebug_3.txt; then
timeout 1500 python -m pytest tests/test_gpu_matvec.py tests/test_gpu_sharded.py tests/test_gpu_parity_large.py tests/test_gpu_symmetric.py tests/test_gpu_dropin.py tests/test_hyp.py -m gpu -q -x > $OUT/${R}_pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/${R}_pytest.log
for c in 1 2s 3; do
  for v in prev main; do
    if [ $v = main ]; then L=$PWD/paper_2001_05523_b200/_lib/libh2b.so; else L=$V/$v.so; fi
    echo "config $c $v: $(H2B_LIB_PATH=$L timeout 900 python tools/mv_time.py $c 2>&1 | grep '^matvec')" >> $OUT/${R}_mvtime.txt
  done
done
timeout 900 python tools/mv_trace.py 3 > $OUT/${R}_trace.txt 2>&1
fi
tail -n 5 $OUT/${R}_pytest.log; cat $OUT/${R}_mvtime.txt; head -8 $OUT/${R}_trace.txt

R=${1:-r02au}
OUT=gpurun_out
mkdir -p $OUT
set -x
V=$PWD/paper_2001_05523_b200/_lib/variants
H2B_LIB_PATH=$V/xel_pef.so timeout 900 python -m pytest -k "not zzz" tests/test_gpu_matvec.py tests/test_gpu_symmetric.py -m gpu -q -x > $OUT/${R}_pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/${R}_pytest.log
H2B_LIB_PATH=$V/leaf4_fa4k.so timeout 900 python -m pytest tests/test_gpu_matvec.py tests/test_gpu_sharded.py -m gpu -q -x > $OUT/${R}_pytest2.log 2>&1; echo "pytest2 rc=$?" >> $OUT/${R}_pytest2.log
for c in 1 2s 3; do
  for v in main xel xel_pef leaf4 fa2k leaf4_fa4k; do
    if [ $v = main ]; then L=$PWD/paper_2001_05523_b200/_lib/libh2b.so; else L=$V/$v.so; fi
    echo "config $c $v: $(H2B_LIB_PATH=$L timeout 900 python tools/mv_time.py $c 2>&1 | grep '^matvec')" >> $OUT/${R}_mvtime.txt
  done
done
tail -3 $OUT/${R}_pytest.log; cat $OUT/${R}_mvtime.txt

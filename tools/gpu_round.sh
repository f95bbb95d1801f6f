R=${1:-r02az}
OUT=gpurun_out
mkdir -p $OUT
set -x
V=$PWD/paper_2001_05523_b200/_lib/variants
for c in 1 2s 3; do
  for v in prev p0s32 p0s128 p0s512 p1s128 p1s512; do
    echo "config $c $v: $(H2B_LIB_PATH=$V/$v.so timeout 900 python tools/mv_time.py $c 2>&1 | grep '^matvec')" >> $OUT/${R}_mvtime.txt
  done
done
cat $OUT/${R}_mvtime.txt

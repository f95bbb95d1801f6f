R=${1:-r02be}
OUT=gpurun_out
mkdir -p $OUT
set -x
for c in 2s 3; do
  for kb in 24 20 28 32; do
    echo "config $c stage ${kb} KB: $(H2B_STAGE_KB=$kb timeout 900 python tools/mv_time.py $c 2>&1 | grep '^matvec\|^plan' | tr '\n' ' ' | cut -c1-330)" >> $OUT/${R}_stage.txt
  done
done
cat $OUT/${R}_stage.txt

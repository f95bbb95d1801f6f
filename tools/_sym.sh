L=paper_2001_05523_b200/_lib
for rep in 1 2; do
for v in base r16 r4; do
  if [ $v = base ]; then lp=$L/libh2b.so; else lp=$L/variants/$v.so; fi
  echo "== cfg1 $v"; H2B_LIB_PATH=$lp timeout 600 python tools/mv_time.py 1 2>&1 | tail -2 | head -1
done; done
echo "== cfg1 EARLY_INNER"; H2B_EARLY_INNER=1 timeout 600 python tools/mv_time.py 1 2>&1 | tail -2 | head -1
for a in "0.1 0.5" "0.3 0.5" "0.2 0.3" "0.2 0.7"; do set -- $a; echo "== cfg1 A1=$1 A2=$2"; H2B_NEAR_A1=$1 H2B_NEAR_A2=$2 timeout 600 python tools/mv_time.py 1 2>&1 | tail -2 | head -1; done
for v in base r16; do
  if [ $v = base ]; then lp=$L/libh2b.so; else lp=$L/variants/$v.so; fi
  echo "== L8 $v"; H2B_LIB_PATH=$lp timeout 600 python tools/mv_time.py sphere 8 4 2 2>&1 | tail -2 | head -1
done

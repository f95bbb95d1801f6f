for v in d_par d_all; do
echo "$v full $(H2B_LIB_PATH=paper_2001_05523_b200/_lib/variants/$v.so timeout 100 python tools/mv_time.py 1 2>&1 | tail -1)"
done

cd $GRAFT_REPO_ROOT
for v in ${VARS:-a b d e f}; do
  echo -n "$v "; H2B_LIB_PATH=paper_2001_05523_b200/_lib/variants/$v.so python bench.py --steps 300 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['frac'])"
done
for v in ${TRACE:-a}; do
H2B_LIB_PATH=paper_2001_05523_b200/_lib/variants/$v.so python tools/mv_trace.py 2>&1 | grep -E "span|forward|bands |marks"
done

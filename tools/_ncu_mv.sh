cd $GRAFT_REPO_ROOT
python tools/mv_run.py --nearfield 0 > gpurun_out/mvrun_plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"k_matvec" -s 2 -c 1 -o gpurun_out/mv_orig python tools/mv_run.py --nearfield 0 --matvecs 3 > gpurun_out/ncu_orig.log 2>&1
H2B_LIB_PATH=paper_2001_05523_b200/_lib/variants/d.so ncu --set full --clock-control none --import-source on -k regex:"k_matvec" -s 2 -c 1 -o gpurun_out/mv_d python tools/mv_run.py --nearfield 0 --matvecs 3 > gpurun_out/ncu_d.log 2>&1
tail -2 gpurun_out/ncu_orig.log gpurun_out/ncu_d.log

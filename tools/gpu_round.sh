set -x
H2B_PERSIST=2 H2B_STAGE_KB=12 timeout 300 ncu --set full --clock-control none -k regex:k_matvec -c 1 -s 2 -o gpurun_out/r02q_persist python tools/persist_one.py 1 > gpurun_out/r02q_ncu.log 2>&1
H2B_PERSIST=0 timeout 300 ncu --set full --clock-control none -k regex:k_matvec -c 1 -s 2 -o gpurun_out/r02q_onetask python tools/persist_one.py 1 >> gpurun_out/r02q_ncu.log 2>&1
tail -n 4 gpurun_out/r02q_ncu.log

#!/bin/bash
# Round profiling on one B200 (run under gpurun).  Plain runs first (must exit 0),
# then the launch list and one full ncu capture per hot kernel.
set -e
R=${1:-r01}
OUT=gpurun_out
python bench.py --steps 20 --warmup 3 --no-cpu-baseline > $OUT/${R}_bench_plain.json 2> $OUT/${R}_bench_plain.log
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $OUT/${R}_launches.csv \
    python bench.py --steps 20 --warmup 3 --no-cpu-baseline > /dev/null 2>&1 || true
python tools/mv_run.py > $OUT/${R}_mvrun_plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_gca_columns|k_gca_aca|k_step" -c 3 -o $OUT/${R}_full_gca_cg python tools/config3.py 6 4 2.0 > $OUT/${R}_ncu_gca.log 2>&1 || true
ncu --set full --clock-control none --import-source on -k regex:"k_matvec|k_blocks_slp|k_singular" -c 4 \
    -o $OUT/${R}_full python tools/mv_run.py --matvecs 2 > $OUT/${R}_ncu_full.log 2>&1 || true
tail -3 $OUT/${R}_ncu_full.log

#!/bin/bash
# Round profiling on one B200 (run under gpurun).  Plain runs first (each must
# exit 0), then the launch list and one full ncu capture per hot kernel.
#   bash tools/profile_round.sh r02
R=${1:-r02}
OUT=gpurun_out
mkdir -p $OUT
set -x
python bench.py > $OUT/${R}_bench.json 2> $OUT/${R}_bench.log; echo "bench rc=$?" >> $OUT/${R}_bench.log
python bench.py --impl reference --steps 3 --warmup 3 > $OUT/${R}_ref.json 2> $OUT/${R}_ref.log; echo "ref rc=$?" >> $OUT/${R}_ref.log
python tools/mv_run.py --config 3 --matvecs 2 > $OUT/${R}_mvrun_plain.log 2>&1 || exit 1
python tools/dlp_nearfield.py 8 3 5 > $OUT/${R}_config2_dlp_nearfield.json 2> $OUT/${R}_dlp_nf.log
python tools/big_config_dlp.py > $OUT/${R}_config2_dlp_single_gpu.json 2> $OUT/${R}_big_dlp.log
python tools/config4.py 64 > $OUT/${R}_config4_n64_single_gpu.json 2> $OUT/${R}_config4.log
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $OUT/${R}_launches.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_matvec|k_blocks_slp|k_singular" -c 4 \
    -o $OUT/${R}_full python tools/mv_run.py --config 3 --matvecs 2 > $OUT/${R}_ncu_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_blocks_dlp" -c 1 \
    -o $OUT/${R}_full_dlp python tools/dlp_nearfield.py 8 3 5 > $OUT/${R}_ncu_dlp.log 2>&1
tail -3 $OUT/${R}_ncu_full.log

#!/bin/bash
# Round profiling on one B200 (run under gpurun).  Plain runs first (each must
# exit 0), then the launch list and one full ncu capture per hot kernel.
#   bash tools/profile_round.sh r02f
R=${1:-r02bd}
OUT=gpurun_out
mkdir -p $OUT
set -x
timeout 1500 python -m pytest tests -m gpu -q > $OUT/${R}_pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/${R}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/${R}_smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/${R}_smoke.log
timeout 1200 python bench.py > $OUT/${R}_bench.json 2> $OUT/${R}_bench.log; echo "bench rc=$?" >> $OUT/${R}_bench.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/${R}_ref.json 2> $OUT/${R}_ref.log; echo "ref rc=$?" >> $OUT/${R}_ref.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_|k_matvec|k_blocks|k_singular|k_touch|k_gca" -c 3000 --csv --log-file $OUT/${R}_launches.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_matvec|k_blocks_slp|k_singular" -c 4 \
    -o $OUT/${R}_full python tools/mv_run.py --config 3 --matvecs 2 > $OUT/${R}_ncu_full.log 2>&1
tail -n 3 $OUT/${R}_pytest.log; cat $OUT/${R}_smoke.log; tail -n 2 $OUT/${R}_bench.log $OUT/${R}_ref.log

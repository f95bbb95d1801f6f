set -e
R=r01s5
OUT=gpurun_out
python bench.py > $OUT/${R}_bench_default.json 2> $OUT/${R}_bench_default.log
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $OUT/${R}_launches.csv \
    python bench.py --steps 20 --warmup 3 --no-cpu-baseline > /dev/null 2>&1 || true
ncu --set full --clock-control none --import-source on -k regex:"k_matvec|k_blocks_slp|k_singular" -c 4 \
    -o $OUT/${R}_full python tools/mv_run.py --matvecs 2 > $OUT/${R}_ncu_full.log 2>&1 || true
tail -3 $OUT/${R}_ncu_full.log
cat $OUT/${R}_bench_default.json

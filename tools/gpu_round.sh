# scratch GPU script (session r02e)
set -x
mkdir -p gpurun_out
NF_LEVEL=8 NF_DLP=0 timeout 900 python tools/nf_variants.py prev r3b s3u3 s3u9 s3u1 s3u3t256 s3u1t256 s9u9 s9u9t256 > gpurun_out/r02e_nfv.txt 2>&1
timeout 600 python tools/mv_run.py --config 3 --matvecs 2 > gpurun_out/r02e_mvrun_plain.log 2>&1; echo "mvrun rc=$?" >> gpurun_out/r02e_mvrun_plain.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_matvec" -c 1 -o gpurun_out/r02e_mv3 python tools/mv_run.py --config 3 --matvecs 2 > gpurun_out/r02e_ncu_mv3.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/r02e_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
cat gpurun_out/r02e_nfv.txt; tail -2 gpurun_out/r02e_mvrun_plain.log; tail -3 gpurun_out/r02e_ncu_mv3.log; wc -l gpurun_out/r02e_launches.csv

# scratch GPU script (session r02h): runtime stage + chunked wide rows
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02h_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02h_pytest.log
for c in 1 2s 3; do echo "== $c"; timeout 600 python tools/mv_time.py $c 2>&1 | grep -E "^matvec|^plan"; done > gpurun_out/r02h_mv.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02h_bench.json 2> gpurun_out/r02h_bench.err; echo "bench rc=$?" >> gpurun_out/r02h_bench.err
tail -3 gpurun_out/r02h_pytest.log; cat gpurun_out/r02h_mv.txt; tail -2 gpurun_out/r02h_bench.err

R=${1:-r02aw}
OUT=gpurun_out
mkdir -p $OUT
set -x
timeout 1500 python -m pytest tests/test_gpu_quadrature.py tests/test_gpu_scale.py tests/test_gpu_symmetric.py tests/test_hyp.py -m gpu -q -x > $OUT/${R}_pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/${R}_pytest.log
timeout 1200 python bench.py --no-cpu-baseline > $OUT/${R}_bench.json 2> $OUT/${R}_bench.log; echo "bench rc=$?" >> $OUT/${R}_bench.log
tail -n 3 $OUT/${R}_pytest.log; tail -n 2 $OUT/${R}_bench.log

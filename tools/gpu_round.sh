# scratch GPU script (session r02i): HYP operator
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_hyp.py tests/test_gpu_dropin.py -m gpu -q -x > gpurun_out/r02i_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02i_pytest.log
tail -30 gpurun_out/r02i_pytest.log

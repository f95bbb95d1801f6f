# scratch GPU script (session r02l): one test
set -x
timeout 600 python -m pytest tests/test_gpu_quadrature.py -m gpu -q -k require_disjoint > gpurun_out/r02l2_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02l2_pytest.log
tail -3 gpurun_out/r02l2_pytest.log

set -x
timeout 1200 python -m pytest tests/test_gpu_tree_device.py -m gpu -q -x -s > gpurun_out/r02s_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02s_pytest.log
tail -n 25 gpurun_out/r02s_pytest.log

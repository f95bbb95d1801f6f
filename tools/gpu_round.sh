set -x
timeout 900 python -m pytest tests/test_gpu_sharded.py -m gpu -q -x > gpurun_out/r02ab_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02ab_pytest.log
timeout 2400 python tools/shard_time.py 3 1 2 4 8 > gpurun_out/r02ab_shard_time.txt 2>&1
tail -n 3 gpurun_out/r02ab_pytest.log; tail -n 6 gpurun_out/r02ab_shard_time.txt

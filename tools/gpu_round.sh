set -x
timeout 600 python -m pytest tests/test_gpu_sharded.py -m gpu -q -x -k xhat > gpurun_out/r02ad_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02ad_pytest.log
H2B_XHAT_ORDER=0 timeout 1800 python tools/shard_time.py 3 2 8 > gpurun_out/r02ad_old.txt 2>&1
timeout 1800 python tools/shard_time.py 3 2 8 > gpurun_out/r02ad_new.txt 2>&1
tail -n 2 gpurun_out/r02ad_pytest.log; head -n 2 gpurun_out/r02ad_old.txt; head -n 2 gpurun_out/r02ad_new.txt

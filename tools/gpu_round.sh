set -x
H2B_DIST_BACKEND=gloo timeout 1200 python bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02z2_gpus2.json 2> gpurun_out/r02z2_gpus2.err; echo "rc=$?" >> gpurun_out/r02z2_gpus2.err
tail -n 3 gpurun_out/r02z2_gpus2.err

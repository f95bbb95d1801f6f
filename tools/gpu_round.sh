# scratch GPU script (session r02b): touch table rewrite + SLP variants
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "touch or singular or quadrature or sharded or nearfield" > gpurun_out/r02b_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02b_pytest.log
./tools/_bin/mufu_probe > gpurun_out/r02b_mufu.txt 2>&1
NF_LEVEL=8 NF_DLP=0 timeout 900 python tools/nf_variants.py old base r3 j3r3 t256j3r3 r1 > gpurun_out/r02b_nfv.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02b_bench.json 2> gpurun_out/r02b_bench.err; echo "bench rc=$?" >> gpurun_out/r02b_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02b_ref.json 2> gpurun_out/r02b_ref.err; echo "ref rc=$?" >> gpurun_out/r02b_ref.err
tail -3 gpurun_out/r02b_pytest.log; cat gpurun_out/r02b_mufu.txt gpurun_out/r02b_nfv.txt; tail -3 gpurun_out/r02b_bench.err; tail -3 gpurun_out/r02b_ref.err

set -x
timeout 900 python -m pytest tests -m gpu -q -x -k "singular or quadrature or nearfield or cfg or hyp or touch" > gpurun_out/r02u_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02u_pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02u_bench.json 2> gpurun_out/r02u_bench.err
tail -n 3 gpurun_out/r02u_pytest.log
python -c "import json;d=json.load(open('gpurun_out/r02u_bench.json'));nf=d['nearfield'];print(d['ms_per_step'], nf['singular'], nf['regular']['ms'], nf['roofline']['frac'])"

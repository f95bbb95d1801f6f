# scratch GPU script (session r02j): DLP kernel variants at sphere L8
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "dlp or DLP" > gpurun_out/r02j_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02j_pytest.log
NF_LEVEL=8 timeout 1500 python tools/nf_variants.py dold dnew dui3 dj9 > gpurun_out/r02j_nfv.txt 2>&1
tail -3 gpurun_out/r02j_pytest.log; cat gpurun_out/r02j_nfv.txt

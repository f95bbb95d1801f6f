R=${1:-r02av}
OUT=gpurun_out
mkdir -p $OUT
set -x
timeout 1200 python tools/big_config_dlp.py > $OUT/${R}_config2_dlp.txt 2>&1
timeout 1200 python tools/config4.py 64 > $OUT/${R}_config4_n64.txt 2>&1
tail -5 $OUT/${R}_config2_dlp.txt $OUT/${R}_config4_n64.txt

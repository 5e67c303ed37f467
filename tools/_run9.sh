set -x
MACKO_TIMING=1 REPS=4 timeout 300 python tools/compress_time.py > gpurun_out/r9_compress.log 2>&1
MACKO_NO_BLOCK_CACHE=1 MACKO_TIMING=1 REPS=4 timeout 300 python tools/compress_time.py >> gpurun_out/r9_compress.log 2>&1
bash tools/round_measure.sh r03 > gpurun_out/r9_measure.log 2>&1
tail -c 2500 gpurun_out/bench_r03_full.json; tail -c 600 gpurun_out/bench_r03_reference.json; grep -v Warn gpurun_out/r9_compress.log

timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_full_size.py -m gpu -x -q 2>&1 | tail -3 > gpurun_out/r11_test.log
cat gpurun_out/r11_test.log
for A in 32 28 25 24 20 16; do
  MACKO_ACTIVE_WARPS=$A timeout 300 python tools/spmv_time.py --shapes 11008x4096@0.5,12288x4096@0.5,22016x4096@0.5,4096x11008@0.5,4096x4096@0.5,36864x12288@0.5 --soak 0 --tag A$A 2>&1 | grep -v Warn >> gpurun_out/r11_var.log
done
timeout 300 python tools/spmm_time.py --modes 8 >> gpurun_out/r11_var.log 2>&1
MACKO_TIMING=1 REPS=4 timeout 300 python tools/compress_time.py >> gpurun_out/r11_var.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"count_rows|emit_rows" --csv --log-file gpurun_out/r11_compress_ncu.csv python tools/compress_time.py > /dev/null 2>&1
grep -h "emit\|count" gpurun_out/r11_compress_ncu.csv | awk -F'","' '{print $5, $(NF)}' | tail -4
cat gpurun_out/r11_var.log

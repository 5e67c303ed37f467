timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -3 > gpurun_out/r10_test.log
cat gpurun_out/r10_test.log
for A in 32 28 25 24 20 16; do
  MACKO_ACTIVE_WARPS=$A timeout 300 python tools/spmv_time.py --shapes 11008x4096@0.5,12288x4096@0.5,22016x4096@0.5,4096x11008@0.5,4096x4096@0.5,36864x12288@0.5 --soak 0 --tag A$A 2>&1 | grep -v Warn >> gpurun_out/r10_var.log
done
timeout 300 python tools/spmm_time.py >> gpurun_out/r10_var.log 2>&1
for v in default rec0; do
  if [ $v = default ]; then L=""; else L="MACKO_LIB=build/variants/libmacko_cuda_$v.so"; fi
  env $L timeout 300 python tools/chain_time.py --tag $v 2>&1 | grep -v Warn >> gpurun_out/r10_var.log
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"count_rows|emit_rows" --csv --log-file gpurun_out/r10_compress_ncu.csv python tools/compress_time.py > /dev/null 2>&1
grep -h "emit\|count" gpurun_out/r10_compress_ncu.csv | cut -c1-200 | tail -4
cat gpurun_out/r10_var.log

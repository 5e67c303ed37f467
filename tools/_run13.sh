for RW in 128 1024 2048 3072 4096; do
  MACKO_ROW_WEIGHT=$RW timeout 300 python tools/spmv_time.py --shapes 36864x12288@0.5,36864x12288@0.3,36864x12288@0.7,11008x4096@0.5,4096x11008@0.5,4096x4096@0.5,22016x4096@0.5 --soak 0 --tag RW$RW 2>&1 | grep -v Warn >> gpurun_out/r13_var.log
  MACKO_ROW_WEIGHT=$RW timeout 300 python tools/chain_time.py --tag RW$RW 2>&1 | grep -v Warn >> gpurun_out/r13_var.log
done
cat gpurun_out/r13_var.log

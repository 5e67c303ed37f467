timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/r15_test.log
cat gpurun_out/r15_test.log
for rep in 1 2; do
for F in 0 1; do
  if [ $F = 1 ]; then E="MACKO_NO_FILL_TABLE=1"; T=nofill; else E="X=1"; T=fill; fi
  env $E timeout 300 python tools/spmv_time.py --shapes 36864x12288@0.5,36864x12288@0.3,36864x12288@0.9,11008x4096@0.5,4096x11008@0.5,4096x4096@0.5,22016x4096@0.5,12288x4096@0.5 --soak 0 --tag $T 2>&1 | grep -v Warn >> gpurun_out/r15_var.log
  env $E timeout 300 python tools/chain_time.py --tag $T 2>&1 | grep -v Warn >> gpurun_out/r15_var.log
done
done
cat gpurun_out/r15_var.log

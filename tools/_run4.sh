timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_chain.py -m gpu -x -q 2>&1 | tail -3 > gpurun_out/r4_test.log
cat gpurun_out/r4_test.log
VARIANTS="default old u4 default old u4" SHAPES="36864x12288@0.5,11008x4096@0.5,4096x4096@0.5,4096x11008@0.5,12288x4096@0.5,22016x4096@0.5,36864x12288@0.9" SOAK=0 timeout 900 bash tools/var_run.sh > gpurun_out/r4_var.log 2>&1
for v in default old; do
  if [ $v = default ]; then L=""; else L="MACKO_LIB=build/variants/libmacko_cuda_$v.so"; fi
  env $L timeout 300 python tools/chain_time.py --tag $v 2>&1 | grep -v Warn >> gpurun_out/r4_var.log
done
cat gpurun_out/r4_var.log

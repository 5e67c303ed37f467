timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/r6_test.log
cat gpurun_out/r6_test.log
VARIANTS="default noedge default noedge" SHAPES="36864x12288@0.5,11008x4096@0.5,4096x4096@0.5,4096x11008@0.5,12288x4096@0.5,22016x4096@0.5" SOAK=0 timeout 900 bash tools/var_run.sh > gpurun_out/r6_var.log 2>&1
for v in default noedge; do
  if [ $v = default ]; then L=""; else L="MACKO_LIB=build/variants/libmacko_cuda_$v.so"; fi
  env $L timeout 300 python tools/chain_time.py --tag $v 2>&1 | grep -v Warn >> gpurun_out/r6_var.log
done
cat gpurun_out/r6_var.log

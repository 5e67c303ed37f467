set -x
VARIANTS="default pf1 pf2 default pf1 pf2" SHAPES="36864x12288@0.5,36864x12288@0.3,36864x12288@0.7,11008x4096@0.5,4096x4096@0.5,4096x11008@0.5" SOAK=0 timeout 600 bash tools/var_run.sh > gpurun_out/r2_var.log 2>&1
for v in default pf1; do
  if [ $v = default ]; then L=""; else L="MACKO_LIB=build/variants/libmacko_cuda_$v.so"; fi
  env $L python tools/spmv_time.py --shapes 5120x12288@0.5,36864x12288@0.5 --no-flush --soak 0 --tag l2res_$v 2>&1 | grep -v Warn >> gpurun_out/r2_var.log
done
for s in "11008 4096" "36864 12288" "4096 4096"; do
  set -- $s
  timeout 120 python tools/trace_spmv.py --rows $1 --cols $2 >> gpurun_out/r2_trace.log 2>&1
done
tail -50 gpurun_out/r2_var.log; cat gpurun_out/r2_trace.log

VARIANTS="default chainall default chainall" SHAPES="36864x12288@0.5,36864x12288@0.3,11008x4096@0.5,4096x11008@0.5,4096x4096@0.5,22016x4096@0.5,12288x4096@0.5" SOAK=0 timeout 900 bash tools/var_run.sh > gpurun_out/r14_var.log 2>&1
timeout 300 python tools/chain_time.py --tag default 2>&1 | grep -v Warn >> gpurun_out/r14_var.log
cat gpurun_out/r14_var.log

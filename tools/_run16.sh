VARIANTS="default esall default esall" SHAPES="36864x12288@0.1,36864x12288@0.2,36864x12288@0.3,36864x12288@0.5,11008x4096@0.5,4096x11008@0.5,4096x4096@0.5,131072x32768@0.1" SOAK=0 timeout 1200 bash tools/var_run.sh > gpurun_out/r16_var.log 2>&1
cat gpurun_out/r16_var.log

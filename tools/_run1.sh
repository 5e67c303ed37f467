set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/r1_gputest.log
cat gpurun_out/r1_gputest.log
VARIANTS="default old cs hint default old cs hint" SHAPES="36864x12288@0.5,36864x12288@0.3,36864x12288@0.7,11008x4096@0.5,4096x4096@0.5,4096x11008@0.5" SOAK=0 timeout 900 bash tools/var_run.sh > gpurun_out/r1_var.log 2>&1
tail -60 gpurun_out/r1_var.log

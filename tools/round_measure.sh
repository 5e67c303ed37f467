#!/bin/bash
# Full measurement pass (run under gpurun): bench lines, launch list and one ncu --set full capture.
# tools/round_measure.sh TAG
tag=${1:-v16}
o=gpurun_out
timeout 600 python bench.py > $o/bench_${tag}_full.json 2> $o/bench_${tag}_full.err; tail -1 $o/bench_${tag}_full.json
timeout 900 python bench.py --sweep --chain --no-cpu-baseline > $o/bench_${tag}_sweep_chain.json 2> $o/bench_${tag}_sweep.err; tail -c 600 $o/bench_${tag}_sweep_chain.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $o/bench_${tag}_reference.json 2>&1; tail -1 $o/bench_${tag}_reference.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $o/${tag}_launches.csv \
  python bench.py --steps 20 --warmup 3 --no-cpu-baseline > $o/ncu_launch_${tag}.log 2>&1; tail -2 $o/ncu_launch_${tag}.log
bash tools/prof.sh ${tag}_spmv_36864x12288

#!/bin/bash
# Full measurement pass (run under gpurun): bench lines, launch list and one ncu --set full capture.
# tools/round_measure.sh TAG [skip_sweep]
tag=${1:-r02}
o=gpurun_out
timeout 900 python bench.py > $o/bench_${tag}_full.json 2> $o/bench_${tag}_full.err; tail -c 1500 $o/bench_${tag}_full.json
timeout 600 python bench.py --impl reference > $o/bench_${tag}_reference.json 2>&1; tail -c 400 $o/bench_${tag}_reference.json
if [ -z "$2" ]; then
timeout 1200 python bench.py --sweep --chain --strong --no-cpu-baseline --no-decode > $o/bench_${tag}_sweep_chain.json 2> $o/bench_${tag}_sweep.err; tail -c 600 $o/bench_${tag}_sweep_chain.json
fi
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $o/${tag}_launches.csv \
  python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-decode --soak-s 0 > $o/ncu_launch_${tag}.log 2>&1; tail -2 $o/ncu_launch_${tag}.log
bash tools/prof.sh ${tag}_spmv_36864x12288

#!/bin/bash
# tools/prof.sh TAG [spmv_once args...]: ncu --set full capture of one macko_spmv launch
# (second launch, warm TLB/x) into gpurun_out/TAG.ncu-rep.  Run under gpurun.
tag=$1; shift
timeout 300 ncu --set full --import-source on --clock-control none -k regex:macko_spmv -s 1 -c 1 \
  -o gpurun_out/$tag python tools/spmv_once.py "$@" > gpurun_out/ncu_$tag.log 2>&1
tail -1 gpurun_out/ncu_$tag.log

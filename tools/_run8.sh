timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_full_size.py -m gpu -x -q 2>&1 | tail -5 > gpurun_out/r8_test.log
cat gpurun_out/r8_test.log
MACKO_TIMING=1 timeout 300 python tools/compress_time.py > gpurun_out/r8_compress.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"count_rows|emit_rows|scan_counts" --csv --log-file gpurun_out/r8_compress_ncu.csv python tools/compress_time.py > /dev/null 2>&1
VARIANTS="default default" SHAPES="36864x12288@0.5,11008x4096@0.5,4096x4096@0.5,4096x11008@0.5,12288x4096@0.5,22016x4096@0.5" SOAK=0 timeout 900 bash tools/var_run.sh > gpurun_out/r8_var.log 2>&1
timeout 300 python tools/chain_time.py --tag default 2>&1 | grep -v Warn >> gpurun_out/r8_var.log
cat gpurun_out/r8_var.log gpurun_out/r8_compress.log
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/r8_compress_ncu.csv')) if len(r)>10]
h=rows[0]
for r in rows[1:]:
    d=dict(zip(h,r))
    print(d.get('Kernel Name','')[:40], d.get('Metric Name'), d.get('Metric Value'))
PY

for v in default e5 e6; do
  if [ $v = default ]; then L=""; else L="MACKO_LIB=build/variants/libmacko_cuda_$v.so"; fi
  env $L timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"emit_rows" --csv --log-file gpurun_out/r17_$v.csv python tools/compress_time.py > /dev/null 2>&1
  echo $v; grep -h "emit" gpurun_out/r17_$v.csv | awk -F'","' '{print $(NF)}' | tail -3
done

# A/B timing of SpMV variants (tools/build_variant.sh) on the same box, interleaved.
S=${SHAPES:-"36864x12288@0.5,36864x12288@0.3,36864x12288@0.1,11008x4096@0.5,4096x4096@0.5"}
for v in ${VARIANTS:-default old default old}; do
  if [ "$v" = default ]; then L=""; else L="MACKO_LIB=build/variants/libmacko_cuda_$v.so"; fi
  env $L python tools/spmv_time.py --shapes $S --soak ${SOAK:-0.5} --tag $v 2>&1 | grep -v Warning
done

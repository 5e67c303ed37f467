#!/bin/bash
# Build an experimental variant of libmacko_cuda.so with extra -D knobs (never the product .so):
#   tools/build_variant.sh NAME "-DMACKO_CHUNK=2048 ..."  ->  build/variants/libmacko_cuda_NAME.so
# Time it with MACKO_LIB=build/variants/libmacko_cuda_NAME.so python tools/spmv_time.py ...
set -e
cd "$(dirname "$0")/.."
NAME=$1
FLAGS=$2
NVCC=${NVCC:-/usr/local/cuda/bin/nvcc}
ARCH="-gencode arch=compute_100a,code=sm_100a"
OUT=build/variants/$NAME
mkdir -p "$OUT"
for f in capi spmv compress generate convert plan; do
  $NVCC $ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr $FLAGS \
    -c paper_2511_13061_b200/csrc/$f.cu -o "$OUT/$f.o" 2> "$OUT/$f.ptxas.log" &
done
wait
$NVCC $ARCH -shared -o build/variants/libmacko_cuda_$NAME.so "$OUT"/*.o -cudart static
grep -A2 "macko_spmvILi7ELi4" "$OUT/spmv.ptxas.log" | grep -o "Used [0-9]* registers" | head -1
echo "built build/variants/libmacko_cuda_$NAME.so"

#!/bin/bash
# Build an A/B variant of libvf.so with extra nvcc defines: tools/build_variant.sh NAME -DFOO=1 ...
set -e
cd "$(dirname "$0")/.."
name=$1; shift
out=build/variant_$name
mkdir -p $out
for f in format build trace capi; do
  nvcc -O3 -std=c++17 --extended-lambda -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC \
    -Xcompiler -fvisibility=hidden -I include "$@" -c paper_2410_14128_b200/csrc/$f.cu -o $out/$f.o &
done
wait
nvcc -shared -gencode arch=compute_100a,code=sm_100a -o $out/libvf.so $out/*.o
echo $out/libvf.so

#!/bin/bash
# Build an A/B variant of libvf.so with extra nvcc defines: tools/build_variant.sh NAME -DFOO=1 ...
# Only trace.cu and format.cu are recompiled; the other objects come from the in-tree build (paper_2410_14128_b200/build).
set -e
cd "$(dirname "$0")/.."
name=$1; shift
out=build/variant_$name
mkdir -p $out
[ -f paper_2410_14128_b200/build/capi.o ] || python -c "from paper_2410_14128_b200 import _build; _build.build()" > /dev/null
nvcc -O3 -std=c++17 --extended-lambda -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC \
  -Xcompiler -fvisibility=hidden -I include "$@" -c ${TRACE_SRC:-paper_2410_14128_b200/csrc/trace.cu} -o $out/trace.o
nvcc -O3 -std=c++17 --extended-lambda -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC \
  -Xcompiler -fvisibility=hidden -I include "$@" -c paper_2410_14128_b200/csrc/format.cu -o $out/format.o
nvcc -shared -gencode arch=compute_100a,code=sm_100a -o $out/libvf.so $out/trace.o $out/format.o \
  paper_2410_14128_b200/build/{build,capi}.o
echo $out/libvf.so

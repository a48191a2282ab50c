#!/bin/bash
# Build libvf.so from a git revision's csrc (A/B baseline): tools/build_ref_variant.sh NAME REV [nvcc defines]
set -e
cd "$(dirname "$0")/.."
name=$1; rev=$2; shift 2
src=build/src_$name
out=build/variant_$name
rm -rf $src; mkdir -p $src/pkg/csrc $src/include $out
for f in $(git ls-tree --name-only $rev paper_2410_14128_b200/csrc/); do git show $rev:$f > $src/pkg/csrc/$(basename $f); done
git show $rev:include/vf.h > $src/include/vf.h
for f in format build trace capi; do
  nvcc -O3 -std=c++17 --extended-lambda -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC \
    -Xcompiler -fvisibility=hidden -I $src/include "$@" -c $src/pkg/csrc/$f.cu -o $out/$f.o &
done
wait
nvcc -shared -gencode arch=compute_100a,code=sm_100a -o $out/libvf.so $out/*.o
echo $out/libvf.so

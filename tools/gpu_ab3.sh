#!/bin/bash
cd "$(dirname "$0")/.."
for spec in cfg5: cfg4: t512:; do
  timeout 900 python tools/ab_env.py "$spec" "cur=VF_LIB=build/variant_k5cur/libvf.so" "sel=VF_LIB=build/variant_k5sel/libvf.so" 2>&1
done
for spec in cfg2: cfg3: cfg5:; do
  timeout 900 python tools/ab_env.py "$spec" "b128=" "b64=VF_BLOCK=64" "b96=VF_BLOCK=96" \
    "c32=VF_LIB=build/variant_chunk5/libvf.so,VF_CHUNKED=1,VF_CHUNK=32,VF_CREFILL=32" \
    "c64=VF_LIB=build/variant_chunk5/libvf.so,VF_CHUNKED=1,VF_CHUNK=64,VF_CREFILL=32" 2>&1
done

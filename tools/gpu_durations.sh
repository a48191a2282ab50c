#!/bin/bash
# per-block durations (natural order) of each config's frame and of its moved-camera frames
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/dur
for c in cfg2 cfg3 cfg4 cfg5 t512; do
  for m in 0 0.005 0.02 0.05; do
    VF_LIB=build/variant_clkall/libvf.so timeout 300 python tools/block_timeline.py --config $c --moved $m \
      --save gpurun_out/dur/${c}_$m.npy > gpurun_out/dur/${c}_$m.txt 2>&1
    echo "$c $m rc=$?"
  done
done

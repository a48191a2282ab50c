#!/bin/bash
# Session check after a container restore: block timelines (tail analysis), the exact driver bench
# command, and the full GPU test suite.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/c_smi.txt 2>&1
for c in cfg2 cfg4 cfg5; do
  VF_LIB=build/variant_clk/libvf.so timeout 300 python tools/block_timeline.py --config $c > gpurun_out/c_blk_$c.txt 2>&1
  echo "blk $c rc=$?"
done
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/c_bench.json 2> gpurun_out/c_bench.err
echo "bench rc=$? bytes=$(wc -c < gpurun_out/c_bench.json)"
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/c_tests.log 2>&1
echo "tests rc=$? $(tail -1 gpurun_out/c_tests.log)"; grep -E "^FAILED|Error" gpurun_out/c_tests.log | head -10

#!/bin/bash
# One bench.py run per config (JSON lines into gpurun_out/bench_<cfg>.json).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for c in ${@:-cfg4 cfg2 cfg3 cfg5 cfg4i t512 cfg1}; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  echo "$c rc=$? $(head -c 200 gpurun_out/bench_$c.json)"
done

#!/bin/bash
# bench.py --sweep for every config: JSON line -> gpurun_out/bench_<cfg>.json, rows -> gpurun_out/sweep_<cfg>.json
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for c in ${CFGS:-cfg5 cfg4 cfg2 cfg3 t512 cfg1 cfg4i cfg4s}; do
  timeout 1500 python bench.py --config $c --sweep --sweep-out gpurun_out/sweep_$c.json --no-side > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  echo "$c rc=$? $(head -c 160 gpurun_out/bench_$c.json)"
done

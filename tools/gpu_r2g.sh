#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_schedule.py tests/test_bench_contract.py -x -q -p no:cacheprovider > gpurun_out/g_tests.log 2>&1
echo "tests rc=$? $(tail -1 gpurun_out/g_tests.log)"; grep -E "^FAILED|Error|assert" gpurun_out/g_tests.log | head -8
for c in cfg1 cfg4s; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-side > gpurun_out/g_bench_$c.json 2> gpurun_out/g_bench_$c.err
  echo "bench $c rc=$?"; cut -c 1-120 gpurun_out/g_bench_$c.json
done
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/g_bench.json 2> gpurun_out/g_bench.err
echo "bench rc=$?"; cat gpurun_out/g_bench.json

#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/h_tests.log 2>&1
echo "tests rc=$? $(tail -1 gpurun_out/h_tests.log)"; grep -E "^FAILED|Error|assert" gpurun_out/h_tests.log | head -8
for c in cfg1 cfg2 cfg3 t512 cfg4s cfg4i cfg4; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-side > gpurun_out/h_bench_$c.json 2> gpurun_out/h_bench_$c.err
  echo "bench $c rc=$?"
done
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/h_bench.json 2> gpurun_out/h_bench.err
echo "bench rc=$?"; cat gpurun_out/h_bench.json
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/h_smoke.log 2>&1; echo "smoke rc=$? $(tail -1 gpurun_out/h_smoke.log)"

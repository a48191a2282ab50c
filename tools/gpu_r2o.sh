#!/bin/bash
# final-ish verification: all GPU tests, smoke, bench default; then sweeps with the scheduled column
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/o_tests.log 2>&1
echo "tests rc=$? $(tail -1 gpurun_out/o_tests.log)"; grep -E "^FAILED|Error|assert" gpurun_out/o_tests.log | head -8
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/o_smoke.log 2>&1; echo "smoke rc=$? $(tail -1 gpurun_out/o_smoke.log)"
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/o_bench.json 2> gpurun_out/o_bench.err
echo "bench rc=$?"; cat gpurun_out/o_bench.json
CFGS="cfg5 cfg4 t512 cfg3 cfg2" bash tools/gpu_sweeps.sh

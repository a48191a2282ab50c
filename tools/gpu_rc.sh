#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/rc_tests.log 2>&1
echo "tests rc=$? $(tail -1 gpurun_out/rc_tests.log)"; grep -E "^FAILED|Error" gpurun_out/rc_tests.log | head -20
for spec in "cfg4:R(4, 4, 4) R(3, 3, 3) G(4)" "cfg4:R(4, 4, 4) R(4, 4, 4) R(3, 3, 3)" "cfg5:R(4, 4, 4) R(4, 4, 4) R(4, 4, 4)" \
    "t512:R(3, 3, 3) R(3, 3, 3) G(3)" "t512:R(4, 4, 4) R(1, 1, 1) R(4, 4, 4)" "t512:D(5, 5, 5, 6) D(4, 4, 4, 6)" \
    "t512:R(5, 5, 5) R(4, 4, 4)" "t512:R(3, 3, 3) R(3, 3, 3) R(3, 3, 3)" "cfg4:D(4, 4, 4, 6) D(3, 3, 3, 6) G(4)"; do
  timeout 600 python tools/ab_env.py "$spec" "spec=" "generic=VF_NO_SPEC=1" 2>&1
done
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
echo "bench rc=$?"; cat gpurun_out/bench_default.json

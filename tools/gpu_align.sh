#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/al_tests.log 2>&1
echo "tests rc=$? $(tail -1 gpurun_out/al_tests.log)"; grep -E "^FAILED|Error|assert" gpurun_out/al_tests.log | head -20
for spec in cfg5: cfg4: "cfg5:G(12)" "cfg5:R(3, 3, 3) G(9)" "cfg4:R(3, 3, 3) G(8)"; do
  timeout 600 python tools/ab_env.py "$spec" "packed=" "aligned=VF_AB_ALIGN=1" 2>&1
done

#!/bin/bash
# gpu tests (optional) + A/B of the in-tree lib against build/variant_$OLD on the headline configs
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
if [ -n "$TESTS" ]; then
  timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider $TESTS > gpurun_out/ab_tests.log 2>&1
  echo "tests rc=$? $(tail -1 gpurun_out/ab_tests.log)"; grep -E "FAILED|Error" gpurun_out/ab_tests.log | head -20
fi
L=build/variant_${OLD:-old}/libvf.so
for spec in ${SPECS:-cfg5: cfg4: cfg2: cfg3:}; do
  timeout 900 python tools/ab_env.py $spec "new=" "old=VF_LIB=$L" 2>&1
done

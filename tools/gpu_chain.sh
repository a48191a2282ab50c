#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/chain_tests.log 2>&1
echo "tests rc=$? $(tail -1 gpurun_out/chain_tests.log)"; grep -E "^FAILED|Error" gpurun_out/chain_tests.log | head -20
for spec in "cfg4:R(4, 4, 4) R(3, 3, 3) G(4)" "cfg4:D(4, 4, 4, 6) D(3, 3, 3, 6) G(4)" "cfg4:D(4, 4, 4, 6) R(3, 3, 3) G(4)" \
    "cfg4:R(4, 4, 4) R(4, 4, 4) R(3, 3, 3)" "cfg5:R(4, 4, 4) R(4, 4, 4) R(4, 4, 4)" "t512:R(3, 3, 3) R(3, 3, 3) G(3)" \
    "t512:D(3, 3, 3, 6) D(3, 3, 3, 6) G(3)" "t512:R(4, 4, 4) R(1, 1, 1) R(4, 4, 4)" "t512:D(5, 5, 5, 6) D(4, 4, 4, 6)" \
    "t512:R(5, 5, 5) R(4, 4, 4)" "t512:R(3, 3, 3) R(3, 3, 3) R(3, 3, 3)"; do
  timeout 600 python tools/ab_env.py "$spec" "spec=" "generic=VF_NO_SPEC=1" 2>&1
done
timeout 600 python tools/counters_report.py cfg5: cfg4: cfg2: cfg3: > gpurun_out/counters.txt 2>&1
ncu --set full --import-source on --clock-control none -k regex:trace_kernel -s 1 -c 1 -o gpurun_out/r2b_full_cfg5 \
    python tools/prof_trace.py --config cfg5 --reps 2 > gpurun_out/r2b_full_cfg5.log 2>&1
echo "ncu rc=$?"
bash tools/gpu_pack.sh

#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python tools/e2e_alloc_probe.py cfg5 2>&1 | tail -4
timeout 600 python tools/pcie_probe.py cfg5 2>&1 | tail -8
for spec in "cfg5:R(4, 4, 4) R(4, 4, 4) R(4, 4, 4)" "t512:R(5, 5, 5) R(4, 4, 4)" "cfg5:" "cfg4:"; do
  timeout 600 python tools/ab_env.py "$spec" "spec=" "generic=VF_NO_SPEC=1" 2>&1
done

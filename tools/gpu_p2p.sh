#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_multigpu.py tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "p2p or scatter" > gpurun_out/p2p_tests.log 2>&1
echo "p2p tests rc=$? $(tail -1 gpurun_out/p2p_tests.log)"; grep -E "^FAILED|Error|error" gpurun_out/p2p_tests.log | head -20
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/all_tests.log 2>&1
echo "all tests rc=$? $(tail -1 gpurun_out/all_tests.log)"; grep -E "^FAILED|Error" gpurun_out/all_tests.log | head -20
for g in p2p nccl; do
  timeout 600 python bench.py --force-dist --gather $g --steps 10 --warmup 3 --no-cpu-baseline --no-side > gpurun_out/fd_$g.json 2> gpurun_out/fd_$g.err
  echo "force-dist $g rc=$?"; head -c 700 gpurun_out/fd_$g.json; echo
done

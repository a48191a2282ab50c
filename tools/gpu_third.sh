#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_build_api.py tests/test_full_frame.py -k "build_api or cfg4s or overflow or allocator or single_raw" -x -q -p no:cacheprovider > gpurun_out/t3_tests.log 2>&1
echo "tests rc=$?"; tail -30 gpurun_out/t3_tests.log
timeout 2400 bash tools/ab_chunked.sh > gpurun_out/ab_chunked.log 2>&1
echo "ab rc=$?"; cat gpurun_out/ab_chunked.log

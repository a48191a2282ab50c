#!/bin/bash
# compute-sanitizer (memcheck, initcheck) over the small-volume parity tests.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for tool in memcheck initcheck; do
  compute-sanitizer --tool $tool --error-exitcode 99 --print-limit 20 \
    python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider \
    -k "small_formats and 0.03 or noncubic or payload or empty_volume or query or compiled_in" > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool exit=$?"; tail -3 gpurun_out/sanitize_$tool.log
done

#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
echo "bench rc=$?"; cat gpurun_out/bench_default.json
timeout 3000 bash tools/profile_r2.sh > gpurun_out/profile_r2.log 2>&1
echo "profile rc=$?"; tail -40 gpurun_out/profile_r2.log
bash tools/gpu_pack.sh

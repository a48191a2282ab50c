#!/bin/bash
# Round-2 first GPU call: gpu tests, the driver's exact bench command (both arms), then profile_r2.sh.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=25 > gpurun_out/gputests.log 2>&1
echo "gpu tests rc=$? $(tail -1 gpurun_out/gputests.log)"
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
echo "bench rc=$? bytes=$(wc -c < gpurun_out/bench_default.json)"
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
echo "ref rc=$? $(head -c 300 gpurun_out/bench_ref.json)"
timeout 3000 bash tools/profile_r2.sh > gpurun_out/profile_r2.log 2>&1
echo "profile rc=$?"

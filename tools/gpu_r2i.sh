#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_schedule.py tests/test_bench_contract.py tests/test_multigpu.py -x -q -p no:cacheprovider > gpurun_out/i_tests.log 2>&1
echo "tests rc=$? $(tail -1 gpurun_out/i_tests.log)"; grep -E "^FAILED|Error|assert" gpurun_out/i_tests.log | head -8
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/i_bench.json 2> gpurun_out/i_bench.err
echo "bench rc=$?"; python -c "import json;d=json.load(open('gpurun_out/i_bench.json'));print(d['value'],d['index_order'],d['cfg4_2048']['value'],d['gpu_launches'],d['config']['schedule'][:20])"
timeout 600 python bench.py --config cfg1 --steps 20 --warmup 5 --no-side > gpurun_out/i_bench_cfg1.json 2>/dev/null; cut -c 1-100 gpurun_out/i_bench_cfg1.json

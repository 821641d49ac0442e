#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_fused_update.py tests/test_gpu_conv.py -q -x -p no:cacheprovider --timeout=600 > gpurun_out/r2w_tests.log 2>&1
timeout 900 python tools/bench_configs.py --only C1 --out gpurun_out/r2w_c1.json > gpurun_out/r2w_c1.log 2>&1
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-v 2>/dev/null | tail -1 > gpurun_out/r2w_bench.json

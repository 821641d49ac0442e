#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_fused_update.py tests/test_gpu_pipeline.py tests/test_gpu_gemm.py tests/test_gpu_fullsize.py -q -x -p no:cacheprovider --timeout=900 > gpurun_out/r2aa_tests.log 2>&1
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-v 2>/dev/null | tail -1 > gpurun_out/r2aa_bench.json

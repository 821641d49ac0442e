#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_fused_update.py tests/test_gpu_conv.py -q -x -p no:cacheprovider --timeout=600 > gpurun_out/r2q_tests.log 2>&1
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-v 2>/dev/null | tail -1 > gpurun_out/r2q_bench.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:bias_grad -s 100 -c 20 --csv --log-file gpurun_out/r2q_bias.csv python bench.py --steps 1 --warmup 1 --epoch-mb 4 --no-cpu-baseline --no-e2e --no-v > /dev/null 2>&1
bash tools/cmd_r2p.sh

#!/bin/bash
# split weight-gradient stream (TPS_SPLIT_W=1): parity + A/B
mkdir -p gpurun_out
TPS_SPLIT_W=1 timeout 1500 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_fused_update.py tests/test_gpu_conv.py tests/test_gpu_fullsize.py -q -x -p no:cacheprovider --timeout=900 > gpurun_out/r2x_tests_split.log 2>&1
: > gpurun_out/r2x_ab.log
for v in 1 0 1 0; do
  TPS_SPLIT_W=$v timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-v 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('split=$v', round(d['value']), d['ms_per_step'], d['clocks']['sm_mhz'], d['losses_first_last'])" >> gpurun_out/r2x_ab.log 2>&1
done
timeout 600 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_fused_update.py -q -x -p no:cacheprovider --timeout=600 > gpurun_out/r2x_tests_default.log 2>&1

#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/sgdbn.log
for v in 0 128; do
  TPS_SGD_BN=$v timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-v 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value']), d['roofline']['per_kind'], d['clocks']['sm_mhz'])" >> gpurun_out/sgdbn.log 2>&1
done
TPS_SGD_BN=128 timeout 300 python -m pytest tests/test_gpu_fused_update.py -q 2>&1 | tail -2 >> gpurun_out/sgdbn.log

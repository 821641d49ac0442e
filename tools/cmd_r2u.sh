#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/r2u_ab.log
for v in 0 128 0 128; do
  TPS_SGD_BN=$v timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-v 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('sgd_bn=$v', round(d['value']), d['ms_per_step'], {k:v['ms'] for k,v in d['roofline']['per_kind'].items()}, d['clocks']['sm_mhz'])" >> gpurun_out/r2u_ab.log 2>&1
done

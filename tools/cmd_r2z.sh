#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/r2z_ab.log
for v in 0 1 2 0 1 2; do
  TPS_SW_PRIO=$v timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-v 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('prio=$v', round(d['value']), d['ms_per_step'], d['clocks']['sm_mhz'])" >> gpurun_out/r2z_ab.log 2>&1
done

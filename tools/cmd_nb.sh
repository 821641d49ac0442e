#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/nb.log
for v in "" lib_variants/libtps_nb3.so lib_variants/libtps_nb4.so; do
  TPS_LIB=$v timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-v 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value']), d['roofline']['per_kind'], d['clocks']['sm_mhz'])" >> gpurun_out/nb.log 2>&1
done

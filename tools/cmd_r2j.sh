#!/bin/bash
# timing diagnostic: chunk-blocked w / v layout in the fused update (results not meaningful)
mkdir -p gpurun_out
: > gpurun_out/r2j_ab.log
for v in default blk default blk; do
  E=""; if [ $v = blk ]; then E="TPS_DIAG_BLK=1"; fi
  env $E timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-v 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value']), d['roofline']['per_kind']['wgrad+update'], d['clocks']['sm_mhz'])" >> gpurun_out/r2j_ab.log 2>&1
done

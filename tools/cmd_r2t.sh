#!/bin/bash
# programmatic dependent launch of the stage GEMMs: parity + A/B
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -x -m gpu -p no:cacheprovider --timeout=900 -k "not full_size and not fullsize" > gpurun_out/r2t_tests.log 2>&1
: > gpurun_out/r2t_ab.log
for v in 1 0 1 0; do
  TPS_PDL=$v timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-v 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('pdl=$v', round(d['value']), d['ms_per_step'], {k:v['ms'] for k,v in d['roofline']['per_kind'].items()}, d['clocks']['sm_mhz'])" >> gpurun_out/r2t_ab.log 2>&1
done
for v in 1 0; do TPS_PDL=$v timeout 300 python tools/profile_resnet.py --mb 6 --pool 2 | cut -c1-80 >> gpurun_out/r2t_ab.log 2>&1; done

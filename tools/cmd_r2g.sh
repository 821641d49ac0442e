#!/bin/bash
# shared-space epilogue accesses + CTA-scope TMEM hand-back: parity + microbench + A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_conv.py tests/test_gpu_fused_update.py tests/test_gpu_pipeline.py -q -x -p no:cacheprovider --timeout=600 > gpurun_out/r2g_tests.log 2>&1
timeout 300 python tools/gemm_bench.py --modes 0,1,2,3 > gpurun_out/r2g_gemm.log 2>&1
: > gpurun_out/r2g_ab.log
for v in default stg0 nb3; do
  L=""; if [ $v != default ]; then L="lib_variants/libtps_$v.so"; fi
  TPS_LIB=$L timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-v 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value']), d['roofline']['per_kind'], d['clocks']['sm_mhz'])" >> gpurun_out/r2g_ab.log 2>&1
done

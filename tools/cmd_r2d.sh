#!/bin/bash
# chunk-distance L2 prefetch A/B, parity subset, ncu source capture of the fused wgrad+update kernel
mkdir -p gpurun_out
: > gpurun_out/r2d_ab.log
for v in default pf2 pf4 pf8 default; do
  L=""; if [ $v != default ]; then L="lib_variants/libtps_$v.so"; fi
  TPS_LIB=$L timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-v 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value']), d['roofline']['per_kind']['wgrad+update'], d['clocks']['sm_mhz'])" >> gpurun_out/r2d_ab.log 2>&1
done
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_conv.py tests/test_gpu_fused_update.py tests/test_gpu_pipeline.py -q -x -p no:cacheprovider --timeout=600 > gpurun_out/r2d_tests.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"gemm_kernel<256, 1, 1, 0, 1" -s 40 -c 1 -o gpurun_out/prof_r2d -f python bench.py --steps 1 --warmup 1 --epoch-mb 4 --no-cpu-baseline --no-e2e --no-v > gpurun_out/ncu_r2d.log 2>&1

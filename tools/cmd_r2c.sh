#!/bin/bash
# L2 hints in the fused update: A/B + parity + one ncu source-level capture of the fused kernel
mkdir -p gpurun_out
: > gpurun_out/r2c_ab.log
for v in default hint0 nb3 bn128; do
  L=""; E=""
  if [ $v = hint0 ] || [ $v = nb3 ]; then L="lib_variants/libtps_$v.so"; fi
  if [ $v = bn128 ]; then E="TPS_SGD_BN=128"; fi
  env $E TPS_LIB=$L timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-v 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value']), d['roofline']['per_kind'], d['clocks']['sm_mhz'])" >> gpurun_out/r2c_ab.log 2>&1
done
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_conv.py tests/test_gpu_fused_update.py tests/test_gpu_pipeline.py -q -x -p no:cacheprovider --timeout=600 > gpurun_out/r2c_tests.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gemm_kernel" -s 121 -c 1 -o gpurun_out/prof_r2c -f python bench.py --steps 1 --warmup 1 --epoch-mb 4 --no-cpu-baseline --no-e2e --no-v > gpurun_out/ncu_r2c.log 2>&1

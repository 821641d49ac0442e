#!/bin/bash
# diagnostics: blend arithmetic removed; fused-update traffic removed; ncu of the blend kernel
mkdir -p gpurun_out
: > gpurun_out/r2h.log
for v in default dbgxf; do
  L=""; if [ $v != default ]; then L="lib_variants/libtps_$v.so"; fi
  echo "== $v" >> gpurun_out/r2h.log
  TPS_LIB=$L timeout 120 python tools/gemm_bench.py --modes 1,3 >> gpurun_out/r2h.log 2>&1
  TPS_GEMM_CG=1 TPS_LIB=$L timeout 120 python tools/gemm_bench.py --modes 3 >> gpurun_out/r2h.log 2>&1
done
for v in default dbgsgd; do
  L=""; if [ $v != default ]; then L="lib_variants/libtps_$v.so"; fi
  TPS_LIB=$L timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-v 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value']), d['roofline']['per_kind']['wgrad+update'], d['clocks']['sm_mhz'])" >> gpurun_out/r2h.log 2>&1
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -c 1 -o gpurun_out/prof_r2h_blend -f python tools/gemm_bench.py --modes 3 --iters 1 > gpurun_out/ncu_r2h.log 2>&1

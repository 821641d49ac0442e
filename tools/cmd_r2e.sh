#!/bin/bash
# CTA-pair blend-on-load: parity, microbench, C2 configs; ncu source capture of the fused wgrad+update
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_conv.py tests/test_gpu_pipeline.py tests/test_gpu_resnet.py -q -x -p no:cacheprovider --timeout=600 -k "not full_size" > gpurun_out/r2e_tests.log 2>&1
timeout 300 python tools/gemm_bench.py --modes 1,3 > gpurun_out/r2e_gemm.log 2>&1
timeout 600 python tools/bench_configs.py --only C2 --out gpurun_out/r2e_c2.json > gpurun_out/r2e_c2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:\(int\)1, \(int\)2, \(int\)0>' -s 20 -c 1 -o gpurun_out/prof_r2e -f python bench.py --steps 1 --warmup 1 --epoch-mb 4 --no-cpu-baseline --no-e2e --no-v > gpurun_out/ncu_r2e.log 2>&1

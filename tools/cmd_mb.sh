#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/gemm_bench.py --modes 0,1,2,3 > gpurun_out/mb_cg2.txt 2>&1
TPS_GEMM_CG=1 timeout 300 python tools/gemm_bench.py --modes 0,1,2,3 > gpurun_out/mb_cg1.txt 2>&1

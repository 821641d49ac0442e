#!/bin/bash
mkdir -p gpurun_out
(for s in "64 576 802816" "64 64 802816" "256 64 802816" "512 4608 25088" "1024 512 2048"; do
  set -- $s; timeout 120 python tools/gemm_bench.py --M $1 --N $2 --K $3 --modes 2 --iters 10; done) > gpurun_out/wg.log 2>&1
timeout 300 ncu --set full --clock-control none -k regex:gemm_kernel -c 1 --launch-skip 3 -o gpurun_out/wg_full -f \
  python tools/gemm_bench.py --M 64 --N 64 --K 802816 --modes 2 --iters 1 > gpurun_out/wg_ncu.log 2>&1

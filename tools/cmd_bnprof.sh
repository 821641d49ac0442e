#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_resnet_ops.py -x -q 2>&1 | tail -3 > gpurun_out/bn_tests.log
timeout 300 python tools/profile_resnet.py --mb 4 > gpurun_out/r50_s1.json 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"bn_bwd_apply_vec|bn_partial_vec|bn_apply_vec" --launch-skip 300 -c 6 -o gpurun_out/bn_full -f \
  python tools/profile_resnet.py --mb 1 > gpurun_out/bn_ncu.log 2>&1

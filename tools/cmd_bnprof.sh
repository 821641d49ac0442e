#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none -k regex:"bn_bwd_apply_vec|bn_partial_vec" --launch-skip 200 -c 4 -o gpurun_out/bn_full -f \
  python tools/profile_resnet.py --mb 1 > gpurun_out/bn_ncu.log 2>&1

#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"bn_bwd_apply_vec" --launch-skip 40 -c 2 -o gpurun_out/bnb_full -f \
  python tools/profile_resnet.py --mb 1 > gpurun_out/bnb_ncu.log 2>&1

#!/bin/bash
mkdir -p gpurun_out
for k in bn_bwd_apply_rows bn_partial_vec bn_apply_rows; do
timeout 300 ncu --set full --clock-control none -k regex:$k -s 30 -c 1 -o gpurun_out/r2s_$k -f python tools/profile_resnet.py --mb 1 --pool 2 > /dev/null 2>&1
done

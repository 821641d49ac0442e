#!/bin/bash
mkdir -p gpurun_out
timeout 120 python tools/profile_resnet.py --mb 4 --stages 8 --variant V > gpurun_out/s8v_a.json 2>&1; echo "rc=$?" >> gpurun_out/s8v_a.json
timeout 120 python tools/profile_resnet.py --mb 16 --stages 8 --variant I --pool 4 > gpurun_out/s8v_b.json 2>&1; echo "rc=$?" >> gpurun_out/s8v_b.json
timeout 120 python tools/profile_resnet.py --mb 16 --stages 8 --variant V --pool 4 > gpurun_out/s8v_c.json 2>&1; echo "rc=$?" >> gpurun_out/s8v_c.json

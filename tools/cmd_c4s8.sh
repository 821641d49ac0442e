#!/bin/bash
mkdir -p gpurun_out
timeout 120 python tools/profile_resnet.py --mb 16 --stages 8 --variant V --pool 4 > gpurun_out/c4s8_V.json 2>&1
timeout 120 python tools/profile_resnet.py --mb 16 --stages 8 --variant I --pool 4 > gpurun_out/c4s8_I.json 2>&1
timeout 120 python tools/profile_resnet.py --mb 16 --stages 1 --variant I --pool 4 > gpurun_out/c4s1_I.json 2>&1

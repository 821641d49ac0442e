#!/bin/bash
mkdir -p gpurun_out
run() { timeout 90 python tools/profile_resnet.py "$@" > /tmp/o.txt 2>&1; echo "rc=$? args=$*" >> gpurun_out/s8i.log; head -c 150 /tmp/o.txt >> gpurun_out/s8i.log; echo >> gpurun_out/s8i.log; }
: > gpurun_out/s8i.log
run --mb 16 --stages 8 --variant I --pool 2
run --mb 8 --stages 8 --variant I --pool 4
run --mb 6 --stages 8 --variant I --pool 2
TPS_NO_SPLITK=1 run --mb 16 --stages 8 --variant I --pool 2
CUDA_LAUNCH_BLOCKING=1 run --mb 16 --stages 8 --variant I --pool 2

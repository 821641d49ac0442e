#!/bin/bash
mkdir -p gpurun_out
run() { timeout 90 python tools/profile_resnet.py "$@" > /tmp/o.txt 2>&1; echo "rc=$? args=$*" >> gpurun_out/s8i2.log; head -c 150 /tmp/o.txt >> gpurun_out/s8i2.log; echo >> gpurun_out/s8i2.log; }
: > gpurun_out/s8i2.log
run --mb 16 --stages 8 --variant I --pool 4
run --mb 16 --stages 8 --variant I --pool 4
run --mb 16 --stages 8 --variant V --pool 4
run --mb 16 --stages 8 --variant I --pool 4
nvidia-smi --query-gpu=memory.used,memory.total --format=csv >> gpurun_out/s8i2.log

#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_resnet_ops.py tests/test_gpu_resnet.py -q -x -p no:cacheprovider --timeout=600 -k "not full_size" > gpurun_out/r2r_tests.log 2>&1
for i in 1 2; do timeout 300 python tools/profile_resnet.py --mb 6 --pool 2 | cut -c1-90 >> gpurun_out/r2r_r50.log 2>&1; done
timeout 300 python tools/profile_resnet.py --mb 16 --stages 8 --pool 4 | cut -c1-90 >> gpurun_out/r2r_r50.log 2>&1

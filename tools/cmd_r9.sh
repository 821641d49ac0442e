#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_resnet.py tests/test_gpu_resnet_ops.py -q 2>&1 | tail -5 > gpurun_out/r9_tests.log
timeout 1500 python -m pytest tests -q -m gpu --ignore=tests/test_gpu_resnet.py --ignore=tests/test_gpu_resnet_ops.py 2>&1 | tail -5 >> gpurun_out/r9_tests.log
timeout 300 python tools/profile_resnet.py --mb 4 > gpurun_out/r50_s1.json 2>&1
timeout 300 python tools/profile_resnet.py --mb 4 --stages 8 > gpurun_out/r50_s8.json 2>&1

#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_resnet_ops.py -x -q 2>&1 | tail -30 > gpurun_out/resnet2.log
timeout 900 python -m pytest tests/test_gpu_resnet.py -q 2>&1 | tail -40 >> gpurun_out/resnet2.log

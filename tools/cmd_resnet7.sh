#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_resnet.py tests/test_gpu_conv.py tests/test_gpu_pipeline.py -x -q 2>&1 | tail -15 > gpurun_out/r7_tests.log

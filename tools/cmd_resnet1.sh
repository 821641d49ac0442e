#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_resnet.py -x -q 2>&1 | tail -40 > gpurun_out/resnet1.log
timeout 900 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_conv.py tests/test_gpu_gemm.py -x -q 2>&1 | tail -5 >> gpurun_out/resnet1.log

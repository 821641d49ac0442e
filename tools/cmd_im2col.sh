#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_conv.py -x -q -k im2col 2>&1 | tail -30 > gpurun_out/im2col.log

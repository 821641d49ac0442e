#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/debug_race.py > gpurun_out/race.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_resnet.py -x -q 2>&1 | tail -5 > gpurun_out/r8_tests.log

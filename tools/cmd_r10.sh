#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_resnet_ops.py -x -q 2>&1 | tail -25 > gpurun_out/r10_tests.log
timeout 1500 python -m pytest tests/test_gpu_resnet.py -x -q 2>&1 | tail -5 >> gpurun_out/r10_tests.log
timeout 300 python tools/profile_resnet.py --mb 4 > gpurun_out/r50_s1.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 1400 -c 1000 --csv \
  --log-file gpurun_out/r50_launches.csv python tools/profile_resnet.py --mb 1 > gpurun_out/r50_ncu.log 2>&1
python tools/launches_summary.py gpurun_out/r50_launches.csv gpurun_out/r50_launches_summary.json "ResNet-50 S=1 B=256 one mini-batch" >> gpurun_out/r50_ncu.log 2>&1

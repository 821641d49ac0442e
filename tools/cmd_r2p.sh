#!/bin/bash
# ResNet-50 (C4) S=1 launch list: where a mini-batch's time goes, per kernel family
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 600 -c 2500 --csv --log-file gpurun_out/r50_launches.csv python tools/profile_resnet.py --mb 3 --pool 2 > /dev/null 2>&1
python tools/launches_summary.py gpurun_out/r50_launches.csv gpurun_out/r50_launches_summary.json "profile_resnet.py ResNet-50 S=1 B=256" > /dev/null 2>&1

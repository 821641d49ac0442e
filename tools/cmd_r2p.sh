#!/bin/bash
# ResNet-50 (C4) S=1 launch list: where a mini-batch's time goes, per kernel family
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 3000 --csv --log-file gpurun_out/r50_launches.csv python tools/profile_resnet.py --mb 2 --pool 2 > /dev/null 2>&1
python tools/launches_summary.py gpurun_out/r50_launches.csv gpurun_out/r50_launches_summary.json "profile_resnet.py ResNet-50 S=1 B=256" > /dev/null 2>&1
timeout 300 python tools/profile_resnet.py --mb 6 --pool 2 > gpurun_out/r50_s1.json 2>&1
timeout 300 python tools/profile_resnet.py --mb 16 --stages 8 --pool 4 > gpurun_out/r50_s8.json 2>&1

#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/debug_race.py > gpurun_out/race.log 2>&1
TPS_NO_SPLITK=1 timeout 300 python tools/debug_race.py >> gpurun_out/race.log 2>&1
TPS_GEMM_CG=1 timeout 300 python tools/debug_race.py >> gpurun_out/race.log 2>&1
CUDA_LAUNCH_BLOCKING=1 timeout 300 python tools/debug_race.py >> gpurun_out/race.log 2>&1

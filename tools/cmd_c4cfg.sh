#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python tools/bench_configs.py --only C4 --out gpurun_out/configs_c4.json > gpurun_out/configs_c4.log 2>&1

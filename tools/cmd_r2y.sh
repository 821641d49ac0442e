#!/bin/bash
mkdir -p gpurun_out
timeout 900 python bench.py --steps 5 --warmup 3 2>gpurun_out/r2y_bench.err | tail -1 > gpurun_out/r2y_bench.json

#!/bin/bash
mkdir -p gpurun_out
timeout 400 python tools/debug_resnet.py s1 > gpurun_out/dbg_r50.log 2>&1

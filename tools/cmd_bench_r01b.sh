#!/bin/bash
mkdir -p gpurun_out
# 1) bench line (all legs) with clocks
timeout 900 python bench.py --steps 5 --warmup 3 2>gpurun_out/bench_full.err | tail -1 > gpurun_out/bench_full.json
# 2) reference arm (oracle) line
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 2>/dev/null | tail -1 > gpurun_out/bench_ref.json
# 3) launch list of one epoch (cold, serialised): shares per kernel family
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 2500 -c 600 --csv --log-file gpurun_out/launches_r01b.csv python bench.py --steps 1 --warmup 1 --epoch-mb 16 --no-cpu-baseline --no-e2e --no-v > /dev/null 2>&1
python tools/launches_summary.py gpurun_out/launches_r01b.csv gpurun_out/launches_r01b_summary.json "bench.py C5 S=1 fused update, one epoch window" > /dev/null 2>&1
# 4) full ncu capture of the GEMMs (fused wgrad+update, fwd, dgrad)
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"gemm_kernel" -s 120 -c 4 -o gpurun_out/prof_r01b -f python bench.py --steps 1 --warmup 1 --epoch-mb 4 --no-cpu-baseline --no-e2e --no-v > gpurun_out/ncu_r01b.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_r01b.ncu-rep > gpurun_out/prof_r01b_summary.txt 2>&1
# 5) per-config one-GPU numbers incl. ResNet-50
timeout 1200 python tools/bench_configs.py --out gpurun_out/configs_one_gpu.json > gpurun_out/configs.log 2>&1

#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/f2_build.log 2>&1
timeout 2400 python -m pytest tests -q -m gpu --timeout=1500 -p no:cacheprovider --durations=8 > gpurun_out/f2_tests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f2_smoke.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 2>gpurun_out/f2_bench.err | tail -1 > gpurun_out/f2_bench.json
timeout 1200 python tools/bench_configs.py --out gpurun_out/f2_configs.json > gpurun_out/f2_c4.log 2>&1
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 2>/dev/null | tail -1 > gpurun_out/f2_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 2500 -c 600 --csv --log-file gpurun_out/f2_launches.csv python bench.py --steps 1 --warmup 1 --epoch-mb 16 --no-cpu-baseline --no-e2e --no-v > /dev/null 2>&1
python tools/launches_summary.py gpurun_out/f2_launches.csv gpurun_out/f2_launches_summary.json "bench.py C5 S=1 fused update, one epoch window" > /dev/null 2>&1

#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/f2_build.log 2>&1
timeout 2400 python -m pytest tests -q -m gpu --timeout=1500 -p no:cacheprovider --durations=8 > gpurun_out/f2_tests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f2_smoke.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 2>gpurun_out/f2_bench.err | tail -1 > gpurun_out/f2_bench.json
timeout 1200 python tools/bench_configs.py --only C4 --out gpurun_out/f2_c4.json > gpurun_out/f2_c4.log 2>&1

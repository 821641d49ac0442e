#!/bin/bash
# HEAD check on a fresh box: full GPU suite, smoke, bench line
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2a_build.log 2>&1
timeout 2400 python -m pytest tests -q -m gpu --timeout=1500 -p no:cacheprovider --durations=15 > gpurun_out/r2a_tests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a_smoke.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 2>gpurun_out/r2a_bench.err | tail -1 > gpurun_out/r2a_bench.json

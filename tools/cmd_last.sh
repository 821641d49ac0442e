#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/last_build.log 2>&1
timeout 2400 python -m pytest tests -q -m gpu --timeout=1500 -p no:cacheprovider > gpurun_out/last_tests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/last_smoke.log 2>&1

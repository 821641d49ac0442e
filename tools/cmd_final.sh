#!/bin/bash
# round-1 evidence refresh: bench line, reference line, launch list, ncu --set full of the three
# stage-GEMM kinds, per-config numbers, full GPU suite + smoke
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/fin_build.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 2>gpurun_out/fin_bench.err | tail -1 > gpurun_out/fin_bench.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 2>/dev/null | tail -1 > gpurun_out/fin_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 2500 -c 600 --csv --log-file gpurun_out/fin_launches.csv python bench.py --steps 1 --warmup 1 --epoch-mb 16 --no-cpu-baseline --no-e2e --no-v > /dev/null 2>&1
python tools/launches_summary.py gpurun_out/fin_launches.csv gpurun_out/fin_launches_summary.json "bench.py C5 S=1 fused update, one epoch window" > /dev/null 2>&1
for k in "upd:\(int\)1, \(int\)2, \(int\)0>" "fwd:\(int\)256, \(int\)0, \(int\)0, \(int\)0, \(int\)0, \(int\)2, \(int\)0>" "dgrad:\(int\)256, \(int\)0, \(int\)1, \(int\)0, \(int\)0, \(int\)2, \(int\)0>"; do
  n=${k%%:*}; re=${k#*:}
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$re" -s 20 -c 1 -o gpurun_out/fin_prof_$n -f python bench.py --steps 1 --warmup 1 --epoch-mb 4 --no-cpu-baseline --no-e2e --no-v > gpurun_out/fin_ncu_$n.log 2>&1
done
timeout 1200 python tools/bench_configs.py --out gpurun_out/fin_configs.json > gpurun_out/fin_configs.log 2>&1
timeout 2400 python -m pytest tests -q -m gpu --timeout=1500 -p no:cacheprovider > gpurun_out/fin_tests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.log 2>&1

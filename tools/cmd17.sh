# 1) bench line (all legs) with clocks
timeout 600 python bench.py --steps 5 --warmup 3 2>&1 | tail -1 | tee gpurun_out/bench_full.json
# 2) launch list of one epoch (cold, serialised): shares per kernel family
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 2500 -c 600 --csv --log-file gpurun_out/launches_r01.csv python bench.py --steps 1 --warmup 1 --epoch-mb 16 --no-cpu-baseline --no-e2e --no-v > /dev/null 2>&1
# 3) full ncu capture of the three stage GEMMs + the update kernel at the bench shapes
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"gemm_kernel|sgd_update_kernel<\(bool\)1, \(bool\)1>" -s 120 -c 6 -o gpurun_out/prof_r01 python bench.py --steps 1 --warmup 1 --epoch-mb 4 --no-cpu-baseline --no-e2e --no-v > gpurun_out/ncu_r01.log 2>&1
tail -n 2 gpurun_out/ncu_r01.log

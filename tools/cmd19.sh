timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"gemm_kernel<\(int\)256, \(int\)1, \(int\)1, \(int\)0, \(int\)1" -s 20 -c 1 -o gpurun_out/prof_fused2 python bench.py --steps 1 --warmup 1 --epoch-mb 4 --no-cpu-baseline --no-e2e --no-v --fuse-update 1 > gpurun_out/ncu_fused2.log 2>&1
tail -n 2 gpurun_out/ncu_fused2.log

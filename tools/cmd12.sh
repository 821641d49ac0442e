timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_kernel<256, 1, 1, 0, 1" -s 40 -c 2 -o gpurun_out/prof_fused python bench.py --steps 1 --warmup 1 --epoch-mb 4 --no-cpu-baseline --no-e2e --no-v --fuse-update 1 > gpurun_out/ncu_fused.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sgd_update|gemm_kernel" -s 150 -c 8 -o gpurun_out/prof_sep python bench.py --steps 1 --warmup 1 --epoch-mb 4 --no-cpu-baseline --no-e2e --no-v --fuse-update 0 > gpurun_out/ncu_sep.log 2>&1
tail -2 gpurun_out/ncu_fused.log gpurun_out/ncu_sep.log

timeout 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_pipeline.py -q -p no:cacheprovider --timeout=300 -x 2>&1 | tail -15 | tee gpurun_out/gpu_tests.log
python tools/gemm_bench.py 2>&1 | tee gpurun_out/gemm_bench.log
timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-v --fuse-update 0 2>&1 | tail -1 | tee gpurun_out/bench_f0.log
timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-v --fuse-update 1 2>&1 | tail -1 | tee gpurun_out/bench_f1.log

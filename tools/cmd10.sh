timeout 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_pipeline.py -q -p no:cacheprovider --timeout=300 -x 2>&1 | tail -15 | tee gpurun_out/gpu_tests.log
python tools/gemm_bench.py 2>&1 | tee gpurun_out/gemm_bench_cg2.log
TPS_GEMM_CG=1 python tools/gemm_bench.py --modes 0,1,2 2>&1 | tee gpurun_out/gemm_bench_cg1.log
timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-v 2>&1 | tail -1 | tee gpurun_out/bench_cg2.log

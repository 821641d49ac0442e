timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -p no:cacheprovider --timeout=900 -k c3 2>&1 | tail -5 | tee gpurun_out/c3_test.log
timeout 900 python tools/bench_configs.py --out gpurun_out/r01_configs.json 2>&1 | tail -20

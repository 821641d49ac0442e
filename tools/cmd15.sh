timeout 900 python -m pytest tests/test_gpu_conv.py -q -p no:cacheprovider --timeout=300 2>&1 | tail -30 | tee gpurun_out/conv_tests.log

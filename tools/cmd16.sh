nproc; free -g | head -2
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -p no:cacheprovider --timeout=900 --durations=5 2>&1 | tail -30 | tee gpurun_out/fullsize_tests.log

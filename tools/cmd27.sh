timeout 900 python -m pytest tests/test_gpu_pipeline.py -q -p no:cacheprovider --timeout=300 -k "device_init" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -p no:cacheprovider --timeout=900 -k c3 2>&1 | tail -2

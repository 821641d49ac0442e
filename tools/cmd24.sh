timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -p no:cacheprovider --timeout=900 -k c3 2>&1 | grep -E "^E " | head -5 | cut -c1-300

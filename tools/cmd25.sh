timeout 900 python -m pytest tests/test_gpu_fused_update.py -q -p no:cacheprovider --timeout=300 2>&1 | grep -E "^E  |passed|failed" | head -30 | cut -c1-300

timeout 900 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_conv.py -q -p no:cacheprovider --timeout=300 -x 2>&1 | tail -4 | tee gpurun_out/gpu_tests.log
for f in 0 1; do
timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-v --fuse-update $f 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fuse', $f, round(d['value']), d['roofline']['per_kind'], d['roofline']['update_kernel']['ms'], d['clocks']['sm_mhz'])"
done

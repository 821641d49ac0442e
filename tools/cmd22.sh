for lib in lib_nb1 lib_nb2 lib; do
TPS_LIB=$PWD/paper_2509_23241_b200/$lib/libtps.so timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-v --fuse-update 1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['value']), d['roofline']['per_kind'], d['clocks']['sm_mhz'])"
done

for bps in 1 2 4 8; do
  TPS_UPD_BPS=$bps timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-v 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bps', $bps, round(d['value']), d['roofline']['per_kind'], d['roofline']['update_kernel']['ms'], d['clocks']['sm_mhz'])"
done

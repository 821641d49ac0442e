#!/bin/bash
# fused vs separate (optimizer-stream) update; blocked-layout timing diagnostic with all kinds
mkdir -p gpurun_out
: > gpurun_out/r2l_ab.log
run() {  # name, env..., -- bench args
  name=$1; shift
  env "$@" timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-v $BARGS 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$name', round(d['value']), {k:(v['ms'],v['tflops']) for k,v in r['per_kind'].items()}, r.get('update_kernel'), d['clocks']['sm_mhz'], d.get('losses_first_last'))" >> gpurun_out/r2l_ab.log 2>&1
}
BARGS="" run fused X=1
BARGS="" run blkdiag TPS_LIB=lib_variants/libtps_blk.so
BARGS="--fuse-update 0" run sep_bps1 TPS_UPD_BPS=1
BARGS="--fuse-update 0" run sep_bps2 TPS_UPD_BPS=2
BARGS="--fuse-update 0" run sep_bps4 TPS_UPD_BPS=4
BARGS="" run fused X=1

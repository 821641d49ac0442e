"""Run ResNet-50 (C4) mini-batches on one GPU for ncu launch lists / per-kind timing.
Usage: python tools/profile_resnet.py [--mb 2] [--stages 1] [--profile]"""
import argparse
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2509_23241_b200 import tps  # noqa: E402
from tools.bench_configs import R50, R50_BOUNDS  # noqa: E402


def main():
    import faulthandler
    faulthandler.dump_traceback_later(int(os.environ.get("TPS_DUMP_AFTER", "0")) or 10 ** 6, exit=False)
    ap = argparse.ArgumentParser()
    ap.add_argument("--mb", type=int, default=2)
    ap.add_argument("--stages", type=int, default=1)
    ap.add_argument("--m", type=int, default=4)
    ap.add_argument("--b", type=int, default=64)
    ap.add_argument("--profile", action="store_true")
    ap.add_argument("--variant", default="I", choices=["V", "I"])
    ap.add_argument("--pool", type=int, default=2)
    a = ap.parse_args()
    bounds = R50_BOUNDS if a.stages == 8 else [0, len(R50)]
    S = len(bounds) - 1
    B = a.m * a.b
    feat = 224 * 224 * 3
    stages = []
    for s in range(S):
        spec = tps.StageSpec(dims=[feat, 1000], stage_bounds=bounds, stage_id=s, micro_batches=a.m,
                             micro_batch_size=a.b, variant=tps.TPS_V if a.variant == "V" else tps.TPS_I, blend=tps.TPS_BLEND_EQ1, lam=0.05, lr=0.01,
                             momentum=0.9, transport=tps.TPS_TRANSPORT_LOCAL if S > 1 else tps.TPS_TRANSPORT_NONE,
                             layers=R50)
        st = tps.Pipeline(spec)
        st.init_weights_synthetic()
        stages.append(st)
    if S > 1:
        tps.local_link(stages)
    pool = a.pool
    xp = torch.empty(pool, B, feat, dtype=torch.bfloat16, device="cuda")
    yp = torch.empty(pool, B, dtype=torch.int32, device="cuda")
    for j in range(pool):
        tps.fill_synthetic(1, 0, 0x10000 + j, B, feat, 0, xp[j])
        tps.fill_synthetic(2, 0, 0x20000 + j, B, 1, 1000, yp[j])
    torch.cuda.synchronize()

    import ctypes
    import threading

    def watchdog(after):
        import time as _t
        _t.sleep(after)
        for s_, st in enumerate(stages):
            pos, n, busy = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int32()
            tps.lib().tps_debug_progress(st.h, ctypes.byref(pos), ctypes.byref(n), None)
            print(f"[watchdog] stage {s_} pos {pos.value}/{n.value}", file=sys.stderr, flush=True)
        for s_, st in enumerate(stages):
            pos, n, busy = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int32()
            tps.lib().tps_debug_progress(st.h, ctypes.byref(pos), ctypes.byref(n), ctypes.byref(busy))
            print(f"[watchdog] stage {s_} busy streams {busy.value:06b}", file=sys.stderr, flush=True)

    if os.environ.get("TPS_WATCHDOG"):
        threading.Thread(target=watchdog, args=(int(os.environ["TPS_WATCHDOG"]),), daemon=True).start()

    def run(first, n):
        if S > 1:
            tps.run_schedule_local(stages, first, n, xp, yp, pool)
        else:
            stages[0].run_schedule(first, n, xp, yp, pool)
        for st in stages:
            st.synchronize()

    run(0, 2)
    if a.profile:
        for st in stages:
            st.set_profiling(True)
    t = time.perf_counter()
    run(2, a.mb)
    dt = time.perf_counter() - t
    out = {"samples_per_s": a.mb * B / dt, "ms_per_mb": dt / a.mb * 1e3, "losses": stages[-1].losses().tolist()[-3:],
           "mem": [st.memory_stats() for st in stages]}
    if a.profile:
        out["kinds"] = {k: [st.kernel_stats(i) for st in stages] for i, k in enumerate(["fwd", "dgrad", "wgrad", "all", "update"])}
    print(json.dumps(out))


if __name__ == "__main__":
    main()

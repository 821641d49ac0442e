"""Chrome-trace (chrome://tracing, Perfetto) export of a pipeline run's per-event device timeline.

Builds an S-stage LOCAL pipeline on one GPU (default: the C2 shape, 4 stages of a 10 × 1024
MLP, I-EQ1), enables tps_set_timeline on every stage with one shared origin event, walks
`--mb` mini-batches and writes one complete event ("ph": "X") per schedule event: one track
per stage, named F<j> / B<j> / U<j>, with the trace record (versions, δ, α, β) as args.

  python tools/chrome_trace.py --out gpurun_out/trace.json [--stages 4 --mb 12 --variant I]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synthgen  # noqa: E402
from paper_2509_23241_b200 import tps  # noqa: E402


def to_chrome(recs_per_stage, names=("F", "B", "U")) -> dict:
    ev = []
    for s, recs in enumerate(recs_per_stage):
        ev.append({"ph": "M", "name": "process_name", "pid": s, "args": {"name": f"stage {s}"}})
        for r in recs:
            e = r.ev
            ev.append({"ph": "X", "pid": s, "tid": 0, "name": f"{names[e.kind]}{e.mb}",
                       "ts": r.t0_ms * 1e3, "dur": max(0.0, (r.t1_ms - r.t0_ms) * 1e3),
                       "args": {"mb": e.mb, "micro": e.micro, "micro_count": e.micro_count, "v_used": e.v_used,
                                "v_latest": e.v_latest, "delta": e.delta, "alpha": e.alpha, "beta": e.beta}})
    return {"traceEvents": ev, "displayTimeUnit": "ms"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/trace.json")
    ap.add_argument("--stages", type=int, default=4)
    ap.add_argument("--layers", type=int, default=10)
    ap.add_argument("--width", type=int, default=1024)
    ap.add_argument("--m", type=int, default=4)
    ap.add_argument("--b", type=int, default=64)
    ap.add_argument("--mb", type=int, default=12)
    ap.add_argument("--variant", default="I", choices=["V", "I"])
    a = ap.parse_args()
    dims = [a.width] * a.layers + [10]
    L, S = a.layers, a.stages
    bounds = [round(i * L / S) for i in range(S)] + [L]
    B = a.m * a.b
    pool = 4
    x = torch.from_numpy(np.stack([synthgen.inputs(1, j, B, dims[0]) for j in range(pool)])).to(torch.bfloat16).cuda()
    y = torch.from_numpy(np.stack([synthgen.labels(1, j, B, dims[-1]) for j in range(pool)])).cuda()
    st = [tps.Pipeline(tps.StageSpec(dims=dims, stage_bounds=bounds, stage_id=s, micro_batches=a.m, micro_batch_size=a.b,
                                     variant=tps.TPS_V if a.variant == "V" else tps.TPS_I, blend=tps.TPS_BLEND_EQ1,
                                     lam=0.3, lr=0.01, seed=1,
                                     transport=tps.TPS_TRANSPORT_LOCAL if S > 1 else tps.TPS_TRANSPORT_NONE))
          for s in range(S)]
    for h in st:
        h.init_weights_synthetic()
    if S > 1:
        tps.local_link(st)
    tps.run_schedule_local(st, 0, 4, x, y, pool)          # warm-up
    for h in st:
        h.synchronize()
    origin = torch.cuda.Event(enable_timing=True)
    origin.record()
    for h in st:
        h.set_timeline(True, origin.cuda_event)
    tps.run_schedule_local(st, 4, a.mb, x, y, pool)
    recs = [h.timeline() for h in st]
    os.makedirs(os.path.dirname(os.path.abspath(a.out)), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(to_chrome(recs), f)
    for s, r in enumerate(recs):
        busy = sum(x.t1_ms - x.t0_ms for x in r)
        span = r[-1].t1_ms - r[0].t0_ms if r else 0.0
        print(f"stage {s}: {len(r)} events, span {span:.3f} ms, compute-stream busy {busy / max(span, 1e-9):.2f}")
    for h in st:
        h.close()


if __name__ == "__main__":
    main()

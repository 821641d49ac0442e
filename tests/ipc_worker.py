"""One pipeline stage in its own process, IPC transport (tests/test_gpu_ipc.py and
bench-style multi-process runs on one GPU).

    python tests/ipc_worker.py --rank R --world S --store DIR --case JSON --out DIR

Every rank: init its stage (cuda:0 unless --device), export its IPC descriptor, all-gather
the descriptors over a gloo process group, connect to its neighbours, run the static order
(one run of M mini-batches; a second run that restarts the numbering must be refused), synchronize, and pickle its trace,
losses and final parameters for the parent to compare.
"""
from __future__ import annotations

import argparse
import json
import os
import pickle
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rank", type=int, required=True)
    ap.add_argument("--world", type=int, required=True)
    ap.add_argument("--store", required=True)
    ap.add_argument("--case", required=True)
    ap.add_argument("--out", required=True)
    ap.add_argument("--device", type=int, default=0)
    ap.add_argument("--dp", type=int, default=1, help="data-parallel replicas (rank = replica * S + stage)")
    a = ap.parse_args()
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2509_23241_b200 import tps
    from pipeline_helpers import graph_workload, is_graph, workload

    case = json.loads(a.case)
    torch.cuda.set_device(a.device)
    dist.init_process_group("gloo", init_method=f"file://{a.store}/pg", rank=a.rank, world_size=a.world)
    dims, bounds, m, b, M = case["dims"], case["bounds"], case["m"], case["b"], case["M"]
    S = len(bounds) - 1
    rep_id, stage = divmod(a.rank, S)
    layers = case.get("layers")
    if is_graph(layers):
        xs, ys, params = graph_workload(layers, m, b, M, case.get("seed", 0), case["kind"])
        w0 = [p[0] for p in params]
        b0 = [p[1] if p[1] is not None else (np.zeros(p[0].shape[0], np.float32) if p[0] is not None else None)
              for p in params]
    else:
        # data parallel: the pool holds the merged mini-batch of dp·m micro-batches (replica r's
        # rows are [r·B, (r+1)·B)), i.e. exactly the oracle's workload with m' = dp·m
        xs, ys, w0, b0 = workload(dims, a.dp * m, b, M, case.get("seed", 0), case["kind"])
    spec = tps.StageSpec(dims=dims, stage_bounds=bounds, stage_id=stage, micro_batches=m, micro_batch_size=b,
                         variant=case["variant"], blend=case["blend"], lam=case["lam"], lr=case["lr"],
                         momentum=case["mu"], transport=tps.TPS_TRANSPORT_IPC, device=a.device,
                         fuse_update=case.get("fuse", 1), layers=layers, dp_size=a.dp, dp_rank=rep_id,
                         dtype=case.get("dtype", 0))
    p = tps.Pipeline(spec)
    for k, l in enumerate(p.layers):
        if w0[l] is not None:
            p.set_weights(k, np.asarray(w0[l]).reshape(w0[l].shape[0], -1), b0[l])
    blob = p.ipc_export() if S > 1 else b""
    blobs = [None] * a.world
    dist.all_gather_object(blobs, blob)
    if S > 1:
        p.ipc_connect(blobs[a.rank - 1] if stage > 0 else None, blobs[a.rank + 1] if stage < S - 1 else None)
    if a.dp > 1:
        dblobs = [None] * a.world
        dist.all_gather_object(dblobs, p.dp_export())
        p.dp_connect([dblobs[r * S + stage] for r in range(a.dp)])
    dist.barrier()
    xdt = torch.float32 if case.get("dtype", 0) == tps.TPS_TF32 else torch.bfloat16   # tf32: fp32 containers
    x_pool = torch.from_numpy(np.stack(xs)).to(xdt).cuda() if stage == 0 else None
    y_pool = torch.from_numpy(np.stack(ys)).cuda() if stage == S - 1 else None
    torch.cuda.synchronize()
    p.run_schedule(0, M, x_pool, y_pool, M)
    p.synchronize()
    try:                       # IPC runs number mini-batches contiguously: a restart at 0 is refused
        p.run_schedule(0, 1, x_pool, y_pool, M)
        contiguity = "accepted"
    except tps.TpsError as e:
        contiguity = e.status
    res = {
        "trace": [(e.stage, e.kind, e.micro, e.micro_count, e.mb, e.v_used, e.v_latest, e.delta, e.alpha, e.beta)
                  for e in p.trace()],
        "losses": p.losses(),
        "weights": [p.get_weights(k) if w0[l] is not None else None for k, l in enumerate(p.layers)],
        "layers": p.layers,
        "contiguity": contiguity,
    }
    res["replica"], res["stage"] = rep_id, stage
    with open(os.path.join(a.out, f"stage{a.rank}.pkl"), "wb") as fh:
        pickle.dump(res, fh)
    dist.barrier()
    p.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

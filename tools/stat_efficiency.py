"""NEXT-3 — statistical-efficiency harness ("number of epochs needed to achieve a particular
accuracy"; "I-TiMePReSt outperforms V-TiMePReSt ... in terms of convergence speed").

A learnable synthetic task (no dataset): inputs from synthgen, labels = argmax of a fixed random
teacher MLP.  The B200 pipeline (all stages on one GPU, LOCAL transport) trains a student MLP for
E epochs with V, I-EQ1 and I-CONVEX at several λ; we report the loss curve and the number of
epochs to reach a loss threshold.  This measures the method's convergence behaviour on our GPU
path; it is not a parity claim and not a reproduction of the paper's (stripped) plots.
Usage: python tools/stat_efficiency.py [--stages 4] [--epochs 12] [--out profiles/...json]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synthgen  # noqa: E402
from paper_2509_23241_b200 import tps  # noqa: E402


def teacher_labels(xs, d, classes, seed=123):
    rng = np.random.default_rng(seed)
    W1 = rng.standard_normal((d, 256)) / np.sqrt(d)
    W2 = rng.standard_normal((256, classes)) / np.sqrt(256)
    return [np.argmax(np.maximum(x.astype(np.float64) @ W1, 0) @ W2, axis=1).astype(np.int32) for x in xs]


def train(variant, blend, lam, args, xpool, ypool, n_mb):
    S = args.stages
    dims = [args.width] * (args.depth + 1) + [args.classes]
    per = args.depth // S
    bounds = [s * per for s in range(S)] + [args.depth + 1]
    stages = []
    for s in range(S):
        spec = tps.StageSpec(dims=dims, stage_bounds=bounds, stage_id=s, micro_batches=args.m,
                             micro_batch_size=args.b, variant=variant, blend=blend, lam=lam, lr=args.lr,
                             momentum=args.mu, transport=tps.TPS_TRANSPORT_LOCAL if S > 1 else 0, seed=7)
        st = tps.Pipeline(spec)
        st.init_weights_synthetic()
        stages.append(st)
    if S > 1:
        tps.local_link(stages)
    curve = []
    for e in range(args.epochs):
        tps.run_schedule_local(stages, e * n_mb, n_mb, xpool, ypool, n_mb)
        for st in stages:
            st.synchronize()
        losses = stages[-1].losses()
        curve.append(float(np.mean(losses[-n_mb:])))
    for st in stages:
        st.close()
    return curve


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--stages", type=int, default=4)
    ap.add_argument("--epochs", type=int, default=12)
    ap.add_argument("--width", type=int, default=512)
    ap.add_argument("--depth", type=int, default=8)
    ap.add_argument("--classes", type=int, default=10)
    ap.add_argument("--m", type=int, default=4)
    ap.add_argument("--b", type=int, default=64)
    ap.add_argument("--batches", type=int, default=32)
    ap.add_argument("--lr", type=float, default=0.05)
    ap.add_argument("--mu", type=float, default=0.9)
    ap.add_argument("--threshold", type=float, default=1.0)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    B = args.m * args.b
    xs = [synthgen.inputs(0, j, B, args.width, synthgen.X_SIGNED) for j in range(args.batches)]
    ys = teacher_labels(xs, args.width, args.classes)
    xpool = torch.from_numpy(np.stack(xs)).to(torch.bfloat16).cuda()
    ypool = torch.from_numpy(np.stack(ys)).cuda()
    runs = [("V", tps.TPS_V, tps.TPS_BLEND_EQ1, 0.05)]
    for lam in (0.02, 0.05, 0.2):
        runs.append((f"I-EQ1 λ={lam}", tps.TPS_I, tps.TPS_BLEND_EQ1, lam))
    for lam in (0.05, 0.5, 2.0):
        runs.append((f"I-CONVEX λ={lam}", tps.TPS_I, tps.TPS_BLEND_CONVEX, lam))
    out = {}
    for name, v, bl, lam in runs:
        curve = train(v, bl, lam, args, xpool, ypool, args.batches)
        hit = next((e + 1 for e, l in enumerate(curve) if l <= args.threshold), None)
        out[name] = {"epoch_mean_loss": [round(c, 5) for c in curve], "epochs_to_threshold": hit}
        print(json.dumps({name: out[name]}), flush=True)
    if args.out:
        json.dump({"task": "teacher-student MLP, synthetic inputs", "config": vars(args), "results": out},
                  open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()

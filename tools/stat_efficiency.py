"""NEXT-3 — statistical-efficiency harness ("number of epochs needed to achieve a particular
accuracy"; "I-TiMePReSt outperforms V-TiMePReSt ... in terms of convergence speed").

A learnable synthetic task (no dataset): inputs from synthgen, labels = argmax of a fixed random
teacher MLP.  The B200 pipeline (all stages on one GPU, LOCAL transport) trains a student MLP for
E epochs with V, I-EQ1 and I-CONVEX at several λ; we report the loss curve and the number of
epochs to reach a loss threshold.  This measures the method's convergence behaviour on our GPU
path; it is not a parity claim and not a reproduction of the paper's (stripped) plots.
Every configuration runs for several seeds (data, teacher and student initialisation all change
with the seed); the report gives, per variant, the mean and standard deviation over seeds of the
final epoch loss, of the area under the epoch-loss curve and of the epochs to the threshold.
Usage: python tools/stat_efficiency.py [--stages 4] [--epochs 12] [--seeds 0,1,2] [--out ...json]
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


def train(variant, blend, lam, args, xpool, ypool, n_mb, seed=7):
    S = args.stages
    dims = [args.width] * (args.depth + 1) + [args.classes]
    per = args.depth // S
    bounds = [s * per for s in range(S)] + [args.depth + 1]
    stages = []
    for s in range(S):
        spec = tps.StageSpec(dims=dims, stage_bounds=bounds, stage_id=s, micro_batches=args.m,
                             micro_batch_size=args.b, variant=variant, blend=blend, lam=lam, lr=args.lr,
                             momentum=args.mu, transport=tps.TPS_TRANSPORT_LOCAL if S > 1 else 0, seed=seed)
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
    ap.add_argument("--epochs", type=int, default=20)
    ap.add_argument("--width", type=int, default=256)
    ap.add_argument("--depth", type=int, default=4)
    ap.add_argument("--classes", type=int, default=10)
    ap.add_argument("--m", type=int, default=4)
    ap.add_argument("--b", type=int, default=64)
    ap.add_argument("--batches", type=int, default=32)
    ap.add_argument("--lr", type=float, default=0.1)
    ap.add_argument("--mu", type=float, default=0.9)
    ap.add_argument("--threshold", type=float, default=1.2)
    ap.add_argument("--out", default=None)
    ap.add_argument("--seeds", default="0,1,2")
    ap.add_argument("--quick", action="store_true", help="V, I-EQ1 and I-CONVEX at the default lambda only")
    args = ap.parse_args()
    B = args.m * args.b
    seeds = [int(x) for x in args.seeds.split(",")]
    runs = [("V", tps.TPS_V, tps.TPS_BLEND_EQ1, 0.05)]
    lams_eq1, lams_cvx = ((0.05,), (0.5,)) if args.quick else ((0.02, 0.05, 0.2), (0.05, 0.5, 2.0))
    for lam in lams_eq1:
        runs.append((f"I-EQ1 λ={lam}", tps.TPS_I, tps.TPS_BLEND_EQ1, lam))
    for lam in lams_cvx:
        runs.append((f"I-CONVEX λ={lam}", tps.TPS_I, tps.TPS_BLEND_CONVEX, lam))
    curves = {name: [] for name, *_ in runs}
    for seed in seeds:
        xs = [synthgen.inputs(seed, j, B, args.width, synthgen.X_SIGNED) for j in range(args.batches)]
        ys = teacher_labels(xs, args.width, args.classes, seed=123 + seed)
        xpool = torch.from_numpy(np.stack(xs)).to(torch.bfloat16).cuda()
        ypool = torch.from_numpy(np.stack(ys)).cuda()
        for name, v, bl, lam in runs:
            curves[name].append(train(v, bl, lam, args, xpool, ypool, args.batches, seed=7 + seed))
            print(json.dumps({"seed": seed, name: [round(c, 4) for c in curves[name][-1]]}), flush=True)
    out = {}
    for name, cs in curves.items():
        c = np.array(cs)
        hits = [next((e + 1 for e, l in enumerate(cv) if l <= args.threshold), None) for cv in cs]
        reached = [h for h in hits if h is not None]
        out[name] = {
            "final_loss_mean": float(c[:, -1].mean()), "final_loss_std": float(c[:, -1].std()),
            "auc_mean": float(c.mean(axis=1).mean()), "auc_std": float(c.mean(axis=1).std()),
            "epochs_to_threshold": hits,
            "epochs_to_threshold_mean_of_reached": float(np.mean(reached)) if reached else None,
            "epoch_mean_loss_per_seed": [[round(x, 5) for x in cv] for cv in cs],
        }
    report = {"task": "teacher-student MLP, synthetic inputs (labels = argmax of a fixed random teacher)",
              "config": vars(args), "seeds": seeds, "results": out}
    print(json.dumps({k: {kk: vv for kk, vv in v.items() if kk != "epoch_mean_loss_per_seed"}
                      for k, v in out.items()}, indent=1))
    if args.out:
        json.dump(report, open(args.out, "w"), indent=1)
    return report


if __name__ == "__main__":
    main()

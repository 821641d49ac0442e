"""Per-config throughput on ONE GPU (context numbers, not the bench.py headline).

Multi-stage configs run all S stages as LOCAL-transport handles on the same GPU, so their
samples/s is the single-GPU cost of the whole pipeline, not the S-GPU throughput.
Usage: python tools/bench_configs.py [--out profiles/r01_configs.json]
"""
import argparse
import math
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_2509_23241_b200 import tps  # noqa: E402


def vgg16_cifar(classes=10):
    layers, H, C = [], 32, 3
    for width, n in [(64, 2), (128, 2), (256, 3), (512, 3), (512, 3)]:
        for _ in range(n):
            layers.append({"kind": "conv3", "cin": C, "cout": width, "h": H, "w": H})
            C = width
        layers.append({"kind": "pool2", "c": C, "h": H, "w": H})
        H //= 2
    layers += [{"kind": "linear", "in": 512, "out": 4096}, {"kind": "linear", "in": 4096, "out": 4096},
               {"kind": "linear", "in": 4096, "out": classes}]
    return layers


def conv_flops_per_sample(layers):
    f = 0.0
    for l, sp in enumerate(layers):
        if sp["kind"] == "conv3":
            g = 2.0 * sp["h"] * sp["w"] * 9 * sp["cin"] * sp["cout"]
        elif sp["kind"] == "conv":
            ho = (sp["h"] + 2 * sp["p"] - sp["k"]) // sp["s"] + 1
            wo = (sp["w"] + 2 * sp["p"] - sp["k"]) // sp["s"] + 1
            g = 2.0 * ho * wo * sp["k"] * sp["k"] * sp["cin"] * sp["cout"]
        elif sp["kind"] == "linear":
            g = 2.0 * sp["in"] * sp["out"]
        else:
            continue
        f += g * (3 if l > 0 else 2)
    return f


from oracle import graph as _graph  # noqa: E402  (layer-graph builder only; no oracle arithmetic runs)

R50, R50_STARTS = _graph.resnet_layers()
R50_BOUNDS = [0, R50_STARTS[3], R50_STARTS[5], R50_STARTS[7], R50_STARTS[9], R50_STARTS[11], R50_STARTS[14],
              R50_STARTS[15], len(R50)]

CONFIGS = {
    "C1 MLP 784-256-10 S=2 m=4 b=8": dict(dims=[784, 256, 10], bounds=[0, 1, 2], m=4, b=8, kind=1),
    "C2 MLP 8x4096 S=4 m=8 b=64 (delta 3/2/1/0)": dict(dims=[4096] * 9 + [10], bounds=[0, 2, 4, 6, 9], m=8, b=64,
                                                         kind=0),
    "C3 VGG-16 CIFAR S=1 B=128": dict(layers=vgg16_cifar(), bounds=[0, 21], m=2, b=64, kind=1),
    "C3 VGG-16 CIFAR S=4 B=128 (4 stages on 1 GPU)": dict(layers=vgg16_cifar(), bounds=[0, 6, 10, 14, 21], m=2,
                                                            b=64, kind=1),
    "C5 deep MLP S=1 B=2048": dict(dims=[4096] * 17 + [10], bounds=[0, 17], m=32, b=64, kind=0),
    "C4 ResNet-50 S=1 B=256": dict(layers=R50, bounds=[0, len(R50)], m=4, b=64, kind=1),
    "C4 ResNet-50 S=8 B=256 (8 stages on 1 GPU)": dict(layers=R50, bounds=R50_BOUNDS, m=4, b=64, kind=1),
}


def schedule_period(S, variant, pool):
    """Mini-batches after which every slot index of the static order repeats (tps_graph_capture)."""
    per = math.lcm(2, pool)
    for s in range(S):
        K = S - s
        per = math.lcm(per, K + 1, K, K if variant == tps.TPS_I else 1)
    return per


def run(name, c, variant, blend, epochs=3, epoch_mb=16, pool=4, graph=False):
    S = len(c["bounds"]) - 1
    if graph:
        per = schedule_period(S, variant, pool)
        if per > 64:            # e.g. 8 stages: lcm(9, 8, 7, ...) mini-batches per replayable run
            graph = False
        else:
            epoch_mb = -(-epoch_mb // per) * per
    layers = c.get("layers")
    dims = c.get("dims") or [layers[0]["h"] * layers[0]["w"] * layers[0]["cin"], layers[-1]["out"]]
    B = c["m"] * c["b"]
    feat = dims[0]
    classes = layers[-1]["out"] if layers else dims[-1]
    stages = []
    for s in range(S):
        spec = tps.StageSpec(dims=dims, stage_bounds=c["bounds"], stage_id=s, micro_batches=c["m"],
                             micro_batch_size=c["b"], variant=variant, blend=blend, lam=0.05, lr=0.01, momentum=0.9,
                             transport=tps.TPS_TRANSPORT_LOCAL if S > 1 else tps.TPS_TRANSPORT_NONE, layers=layers)
        st = tps.Pipeline(spec)
        st.init_weights_synthetic()
        stages.append(st)
    if S > 1:
        tps.local_link(stages)
    xp = torch.empty(pool, B, feat, dtype=torch.bfloat16, device="cuda")
    yp = torch.empty(pool, B, dtype=torch.int32, device="cuda")
    for j in range(pool):
        tps.fill_synthetic(c["kind"], 0, 0x10000 + j, B, feat, 0, xp[j])
        tps.fill_synthetic(2, 0, 0x20000 + j, B, 1, classes, yp[j])
    torch.cuda.synchronize()
    mb = 0
    stream = torch.cuda.Stream()
    g = None

    def epoch():
        nonlocal mb, g
        if graph and g is None:
            g = tps.Graph(stages, mb, epoch_mb, xp, yp, pool, stream.cuda_stream)
        elif graph:
            g.replay()
        elif S > 1:
            tps.run_schedule_local(stages, mb, epoch_mb, xp, yp, pool)
        else:
            stages[0].run_schedule(mb, epoch_mb, xp, yp, pool)
        mb += epoch_mb

    epoch()
    for st in stages:
        st.synchronize()
    t0 = time.perf_counter()
    for _ in range(epochs):
        epoch()
    stream.synchronize()
    for st in stages:
        st.synchronize()
    dt = time.perf_counter() - t0
    if g is not None:
        g.close()
    sps = epochs * epoch_mb * B / dt
    mem = [st.memory_stats() for st in stages]
    fps = conv_flops_per_sample(layers) if layers else sum(2.0 * dims[l] * dims[l + 1] * (3 if l else 2)
                                                           for l in range(len(dims) - 1))
    for st in stages:
        st.close()
    return {"samples_per_s": round(sps, 1), "tflops_effective": round(sps * fps / 1e12, 1), "epoch_mb": epoch_mb,
            "stash_bytes_per_stage": [m["stash"] for m in mem], "peak_bytes_per_stage": [m["peak"] for m in mem]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--only", default=None, help="substring filter on config names")
    ap.add_argument("--graph", action="store_true", help="replay each epoch as a captured CUDA graph")
    a = ap.parse_args()
    res = {}
    for name, c in CONFIGS.items():
        if a.only and a.only not in name:
            continue
        for vn, v, bl in [("V", tps.TPS_V, tps.TPS_BLEND_EQ1), ("I-EQ1", tps.TPS_I, tps.TPS_BLEND_EQ1),
                          ("I-CONVEX", tps.TPS_I, tps.TPS_BLEND_CONVEX)]:
            if vn == "I-CONVEX" and len(c["bounds"]) == 2:
                continue
            r = run(name, c, v, bl, graph=a.graph)
            res[f"{name} | {vn}"] = r
            print(json.dumps({f"{name} | {vn}": r}), flush=True)
    if a.out:
        json.dump({"note": "one B200, wall-clock over 3 epochs of 16 mini-batches after 1 warm-up epoch; "
                           "multi-stage configs run every stage on the same GPU", "results": res},
                  open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()

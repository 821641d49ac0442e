"""Shared helpers for parity tests: run the same seeded workload through the oracle
(CPU) and through the C ABI (GPU), and compare."""
from __future__ import annotations

import numpy as np

import synthgen
from oracle import pipeline as opipe
from oracle import staleness as ost


def workload(dims, m, b, M, seed=0, kind=synthgen.X_SIGNED):
    B = m * b
    xs = [synthgen.inputs(seed, j, B, dims[0], kind) for j in range(M)]
    ys = [synthgen.labels(seed, j, B, dims[-1]) for j in range(M)]
    w0 = [synthgen.weights(seed, l, dims[l + 1], dims[l]) for l in range(len(dims) - 1)]
    b0 = [np.zeros(dims[l + 1], np.float32) for l in range(len(dims) - 1)]
    return xs, ys, w0, b0


def net_workload(layers, m, b, M, seed=0, kind=synthgen.X_UNIT):
    """Image-net inputs (flattened NHWC rows) and synthgen weights ([Co,3,3,Ci] for convs)."""
    s0 = layers[0]
    feat = s0["h"] * s0["w"] * s0["cin"]
    classes = layers[-1]["out"]
    xs = [synthgen.inputs(seed, j, m * b, feat, kind) for j in range(M)]
    ys = [synthgen.labels(seed, j, m * b, classes) for j in range(M)]
    w0, b0 = [], []
    for l, sp in enumerate(layers):
        if sp["kind"] == "pool2":
            w0.append(None)
            b0.append(None)
        elif sp["kind"] == "conv3":
            w0.append(synthgen.weights(seed, l, sp["cout"], 9 * sp["cin"]).reshape(sp["cout"], 3, 3, sp["cin"]))
            b0.append(np.zeros(sp["cout"], np.float32))
        else:
            w0.append(synthgen.weights(seed, l, sp["out"], sp["in"]))
            b0.append(np.zeros(sp["out"], np.float32))
    return xs, ys, w0, b0


GRAPH_KINDS = ("conv", "bn", "maxpool3", "avgpool")


def is_graph(layers):
    return bool(layers) and any(sp["kind"] in GRAPH_KINDS for sp in layers)


def graph_workload(layers, m, b, M, seed=0, kind=synthgen.X_UNIT, res_gamma=1.0):
    """ResNet-style inputs (flattened NHWC rows) and parameters: synthgen conv weights
    [Co,k,k,Ci] (fan_in k·k·Ci), BN γ = 1 (res_gamma for the BN that closes a residual block,
    the usual scaled-residual initialisation), β = 0, synthgen head weights, zero head bias."""
    s0 = layers[0]
    feat = s0["h"] * s0["w"] * s0["cin"]
    classes = layers[-1]["out"]
    xs = [synthgen.inputs(seed, j, m * b, feat, kind) for j in range(M)]
    ys = [synthgen.labels(seed, j, m * b, classes) for j in range(M)]
    params = []
    for l, sp in enumerate(layers):
        k = sp["kind"]
        if k == "conv":
            kk = sp["k"]
            w = synthgen.weights(seed, l, sp["cout"], kk * kk * sp["cin"]).reshape(sp["cout"], kk, kk, sp["cin"])
            params.append((w, None))
        elif k == "bn":
            g = res_gamma if sp.get("res") is not None else 1.0
            params.append((np.full(sp["c"], g, np.float32), np.zeros(sp["c"], np.float32)))
        elif k == "linear":
            params.append((synthgen.weights(seed, l, sp["out"], sp["in"]), np.zeros(sp["out"], np.float32)))
        else:
            params.append((None, None))
    return xs, ys, params


def run_oracle_graph(layers, bounds, m, b, M, variant, blend, lam, lr, mu, wd=0.0, seed=0, kind=synthgen.X_UNIT,
                     res_gamma=1.0):
    from oracle import graph as ograph
    xs, ys, params = graph_workload(layers, m, b, M, seed, kind, res_gamma)
    return ograph.run(layers, bounds, m, b, M, xs, ys, params, variant=variant, blend=blend, lam=lam, lr=lr, mu=mu,
                      wd=wd)


def run_oracle(dims, bounds, m, b, M, variant, blend, lam, lr, mu, wd=0.0, seed=0, kind=synthgen.X_SIGNED,
               layers=None, max_inflight=0, exact=False, dtype="bf16"):
    if layers:
        xs, ys, w0, b0 = net_workload(layers, m, b, M, seed, kind)
    else:
        xs, ys, w0, b0 = workload(dims, m, b, M, seed, kind)
    cfg = opipe.Config(dims, bounds, m, b, M, variant=variant, blend=blend, lam=lam, lr=lr, momentum=mu, wd=wd,
                       layers=layers, max_inflight=max_inflight, exact=exact, dtype=dtype)
    return opipe.run(cfg, xs, ys, w0, b0)


def run_gpu(dims, bounds, m, b, M, variant, blend, lam, lr, mu, wd=0.0, seed=0, kind=synthgen.X_SIGNED,
            fwd_group=0, init="set", extra_recv_slot=1, fuse_update=1, layers=None, drive=None, res_gamma=1.0,
            **spec_kw):
    """All S stages as LOCAL-transport handles on cuda:0; returns (stages, losses).

    drive: None => tps_run_schedule_local; else a callable(stages, x_pool, y_pool, M) that
    issues the events itself (e.g. through the step-wise tps_stage_* calls).
    spec_kw: extra StageSpec fields (max_inflight, staleness_mode, torch_alloc, ...)."""
    import torch

    from paper_2509_23241_b200 import tps

    S = len(bounds) - 1
    if is_graph(layers):
        xs, ys, params = graph_workload(layers, m, b, M, seed, kind, res_gamma)
        w0 = [p[0] for p in params]
        b0 = [p[1] if p[1] is not None else np.zeros(p[0].shape[0], np.float32) if p[0] is not None else None
              for p in params]
    elif layers:
        xs, ys, w0, b0 = net_workload(layers, m, b, M, seed, kind)
    else:
        xs, ys, w0, b0 = workload(dims, m, b, M, seed, kind)
    # bf16 input pools, or fp32 containers in tf32 storage mode (the inputs are exact in both)
    xdt = torch.float32 if spec_kw.get("dtype", 0) == tps.TPS_TF32 else torch.bfloat16
    x_pool = torch.from_numpy(np.stack(xs)).to(xdt).cuda().contiguous()
    y_pool = torch.from_numpy(np.stack(ys)).cuda().contiguous()
    V = tps.TPS_V if variant == ost.V_VARIANT else tps.TPS_I
    BL = tps.TPS_BLEND_EQ1 if blend == ost.EQ1 else tps.TPS_BLEND_CONVEX
    stages = []
    for s in range(S):
        spec = tps.StageSpec(dims=dims, stage_bounds=bounds, stage_id=s, micro_batches=m, micro_batch_size=b,
                             fwd_group=fwd_group, variant=V, blend=BL, lam=lam, lr=lr, momentum=mu, weight_decay=wd,
                             transport=tps.TPS_TRANSPORT_LOCAL if S > 1 else tps.TPS_TRANSPORT_NONE, seed=seed,
                             extra_recv_slot=extra_recv_slot, fuse_update=fuse_update, layers=layers, **spec_kw)
        st = tps.Pipeline(spec)
        if init == "set":
            for k, l in enumerate(st.layers):
                if w0[l] is not None:
                    st.set_weights(k, np.asarray(w0[l]).reshape(w0[l].shape[0], -1), b0[l])
        else:
            st.init_weights_synthetic()
        stages.append(st)
    if S > 1:
        tps.local_link(stages)
    if drive is None:
        tps.run_schedule_local(stages, 0, M, x_pool, y_pool, M)
    else:
        drive(stages, x_pool, y_pool, M)
    for st in stages:
        st.synchronize()
    return stages, stages[-1].losses()


def expand_gpu_trace(stages):
    rows = []
    for st in stages:
        for e in st.trace():
            if e.kind == 0:
                for a in range(e.micro, e.micro + e.micro_count):
                    rows.append((e.stage, "F", e.mb, a, e.v_used, e.v_latest, e.delta, 1.0, 0.0))
            elif e.kind == 1:
                rows.append((e.stage, "B", e.mb, -1, e.v_used, e.v_latest, e.delta, e.alpha, e.beta))
            else:
                rows.append((e.stage, "U", e.mb, -1, e.v_used, e.v_latest, 0, 1.0, 0.0))
    return sorted(rows)


def oracle_trace(res):
    return sorted((r.stage, r.kind, r.mb, r.micro, r.v_used, r.v_latest, r.delta,
                   float(r.alpha), float(r.beta)) for r in res.trace)


def weight_rel_err(got, ref):
    """max|Δ| / max|w_ref| per tensor (reading Z19)."""
    return float(np.abs(got.astype(np.float64) - ref).max() / max(np.abs(ref).max(), 1e-30))


def layer_rel_err(w, b, w_ref, b_ref):
    """max|Δ| / max|p_ref| over a layer's parameter tensor p = [W | b] (reading Z19).

    Biases start at 0 and their gradients are column sums of bf16 activation-gradients
    with heavy cancellation, so a bias-only ratio measures cancellation noise, not the
    kernel; the layer's parameters are judged as one tensor."""
    d = max(np.abs(w.astype(np.float64) - w_ref).max(), np.abs(b.astype(np.float64) - b_ref).max())
    return float(d / max(np.abs(w_ref).max(), np.abs(b_ref).max(), 1e-30))

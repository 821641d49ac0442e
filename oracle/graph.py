"""Pipeline replay for networks with skip connections and batch norm (ResNet-50, configs[3]) —
TEST INFRASTRUCTURE ONLY.

Same method as oracle/pipeline.py (static nF1B order via schedule.execute, latest-weight
forwards, V / I backward weights, version stash kept until its last consumer, SGD on the latest
fp32 master — P:93, readings Z1-Z11), applied to a layer
graph: every layer names its main input `src` (default: the previous layer) and BN layers may add
a residual tensor `res` before their ReLU.  Stages hold consecutive layers; only the previous
stage's last output crosses a stage boundary.

Layer kinds (NHWC; shapes are the layer's INPUT spatial size):
  conv     {cin, cout, k, s, p, h, w}   no bias; weight [cout, k, k, cin]
  bn       {c, h, w, relu, res?}        γ (read by the backward -> stashed and blended, Z12),
                                        β (forward only -> latest fp32, like a bias)
  maxpool3 {c, h, w}                    3x3 / stride 2 / pad 1
  avgpool  {c, h, w}                    global average
  linear   {in, out}                    the head (no ReLU, no input mask)
Storage (Z13): conv / pool / BN outputs and all activation gradients are bf16; BN statistics,
dW, dγ, dβ fp32-rounded sums of fp64 products; γ versions are fp32.  A tensor consumed twice
(a block input) accumulates its gradient as bf16(stored + new) in reverse layer order.
"""
from __future__ import annotations

import numpy as np

from . import mlp, resnet, schedule, staleness
from .pipeline import Result, TraceRow


def out_shape(sp, N):
    k = sp["kind"]
    if k == "conv":
        Ho = (sp["h"] + 2 * sp["p"] - sp["k"]) // sp["s"] + 1
        Wo = (sp["w"] + 2 * sp["p"] - sp["k"]) // sp["s"] + 1
        return (N, Ho, Wo, sp["cout"])
    if k == "bn":
        return (N, sp["h"], sp["w"], sp["c"])
    if k == "maxpool3":
        return (N, (sp["h"] - 1) // 2 + 1, (sp["w"] - 1) // 2 + 1, sp["c"])
    if k == "avgpool":
        return (N, sp["c"])
    return (N, sp["out"])


def in_shape(sp, N):
    if sp["kind"] == "linear":
        return (N, sp["in"])
    c = sp["cin"] if sp["kind"] == "conv" else sp["c"]
    return (N, sp["h"], sp["w"], c)


def run(layers, bounds, m, b, M, xs, ys, params0, variant=staleness.I_VARIANT, blend=staleness.EQ1, lam=0.05,
        lr=0.01, mu=0.0, wd=0.0, exact=False) -> Result:
    """params0[l] = (W or γ or None, b or β or None) as fp32 arrays."""
    S, L, B = len(bounds) - 1, len(layers), m * b
    prec = mlp.Precision(exact)
    src = [sp.get("src", l - 1) for l, sp in enumerate(layers)]
    stage_of = [next(s for s in range(S) if bounds[s] <= l < bounds[s + 1]) for l in range(L)]
    for l, sp in enumerate(layers):
        for t in (src[l], sp.get("res")):
            if t is not None and t >= 0 and stage_of[t] != stage_of[l]:
                assert t == bounds[stage_of[l]] - 1, f"layer {l} reads layer {t} across a stage boundary"
    versioned = [sp["kind"] in ("conv", "bn", "linear") for sp in layers]
    has_b = [sp["kind"] in ("bn", "linear") for sp in layers]
    cast = (lambda a: np.asarray(a, np.float64)) if exact else (lambda a: np.asarray(a, np.float32).astype(np.float64))
    W = [cast(p[0]) if versioned[l] else None for l, p in enumerate(params0)]
    Bv = [cast(p[1]) if has_b[l] else None for l, p in enumerate(params0)]
    VW = [np.zeros_like(w) if w is not None else None for w in W]
    Vb = [np.zeros_like(x) if x is not None else None for x in Bv]

    def store_w(l):   # weight version copy: bf16 for conv/linear, fp32 for BN γ
        if not versioned[l]:
            return None
        return prec.store(W[l]) if layers[l]["kind"] != "bn" else prec.f32(W[l])

    lay = [list(range(bounds[s], bounds[s + 1])) for s in range(S)]
    versions = [{0: {l: store_w(l) for l in lay[s]}} for s in range(S)]
    latest = [0] * S
    consumers = [dict() for _ in range(S)]
    fwd_ver = {}
    acts = {}          # (s, j, a) -> {tensor id: value} (layer outputs + stage input under key -1)
    stats = {}         # (s, j, a, l) -> (mu, invstd)
    fwd_msg, bwd_msg, ce_grad = {}, {}, {}
    loss_sum = np.zeros(M)
    grads_w = {}
    trace = []

    fired, _ = schedule.execute(S, m, M)
    for s, e in fired:
        ls = lay[s]
        if e.kind == "F":
            j, a = e.mb, e.micro
            v = latest[s]
            fwd_ver.setdefault((s, j), v)
            consumers[s].setdefault(v, set()).add(j)
            Wv = versions[s][v]
            X = xs[j][a * b:(a + 1) * b].astype(np.float64) if s == 0 else fwd_msg.pop((s, j, a))
            T = {bounds[s] - 1: prec.store(X)}
            for l in ls:
                sp = layers[l]
                x = T[src[l]].reshape(in_shape(sp, b))
                k = sp["kind"]
                if k == "conv":
                    y = prec.store(resnet.conv_forward(x, Wv[l], sp["s"], sp["p"]))
                elif k == "bn":
                    z, mu_, inv = resnet.bn_forward(x, Wv[l], Bv[l])
                    stats[(s, j, a, l)] = (mu_, inv)
                    if sp.get("res") is not None:
                        z = z + T[sp["res"]].reshape(z.shape)
                    y = prec.store(np.maximum(z, 0.0) if sp.get("relu") else z)
                elif k == "maxpool3":
                    y = resnet.maxpool3_forward(x)
                elif k == "avgpool":
                    y = prec.store(resnet.avgpool_forward(x))
                else:  # linear head
                    z = mlp.linear_forward(x.reshape(b, -1), Wv[l], Bv[l])
                    rows, G = mlp.softmax_xent(z, ys[j][a * b:(a + 1) * b], B)
                    loss_sum[j] += rows.sum()
                    ce_grad[(j, a)] = prec.store(G)
                    y = z
                T[l] = y
            acts[(s, j, a)] = T
            if s < S - 1:
                fwd_msg[(s + 1, j, a)] = T[ls[-1]].reshape(b, -1)
            trace.append(TraceRow(s, "F", j, a, v, v, 0))
        elif e.kind == "B":
            j = e.mb
            vf, vl = fwd_ver[(s, j)], latest[s]
            if variant == staleness.V_VARIANT:
                delta, v_used = 0, vl
                alpha, beta = 1.0, 0.0
                Wst = versions[s][vl]
            else:
                delta, v_used = vl - vf, vf
                alpha, beta = staleness.blend_coeffs(variant, blend, delta, lam)
                Wst = versions[s][vf]
            Wl = versions[s][vl]
            # whole-mini-batch tensors (micro-batches stacked in order)
            Tm = {t: np.concatenate([acts[(s, j, a)][t] for a in range(m)], axis=0) for t in acts[(s, j, 0)]}
            for a in range(m):
                del acts[(s, j, a)]
            G = {}

            def add_grad(t, g):
                G[t] = prec.store(g) if t not in G else prec.store(G[t] + g)

            if s == S - 1:
                G[ls[-1]] = np.concatenate([ce_grad.pop((j, a)) for a in range(m)], axis=0)
            else:
                G[ls[-1]] = bwd_msg.pop((s, j)).reshape(Tm[ls[-1]].shape)
            gw, gb = {}, {}
            for l in reversed(ls):
                sp = layers[l]
                k = sp["kind"]
                g = G.pop(l)
                x = Tm[src[l]].reshape(in_shape(sp, B))
                if k in ("conv", "bn", "linear"):
                    Wres = mlp.resolve_backward_weight(Wst[l], Wl[l], alpha, beta)
                if k == "linear":
                    g2 = g.reshape(B, -1)
                    dW, db = mlp.wgrad(g2, x.reshape(B, -1))
                    gw[l], gb[l] = prec.f32(dW), prec.f32(db)
                    if l > 0:
                        add_grad(src[l], (g2 @ Wres).reshape(x.shape))
                elif k == "conv":
                    g4 = g.reshape(out_shape(sp, B))
                    gw[l] = prec.f32(resnet.conv_wgrad(g4, x, sp["k"], sp["s"], sp["p"]))
                    if l > 0:
                        add_grad(src[l], resnet.conv_dgrad(g4, Wres, x.shape, sp["s"], sp["p"]))
                elif k == "bn":
                    y = Tm[l].reshape(x.shape)
                    dy = g.reshape(x.shape) * (y > 0) if sp.get("relu") else g.reshape(x.shape)
                    if sp.get("res") is not None:
                        add_grad(sp["res"], dy)
                    dx = np.empty_like(x)
                    dgam = np.zeros(sp["c"])
                    dbet = np.zeros(sp["c"])
                    for a in range(m):        # per micro-batch statistics (Z22)
                        mu_, inv = stats.pop((s, j, a, l))
                        sl = slice(a * b, (a + 1) * b)
                        dxa, dga, dba = resnet.bn_backward(dy[sl], x[sl], Wres, mu_, inv)
                        dx[sl] = dxa
                        dgam += dga
                        dbet += dba
                    gw[l], gb[l] = prec.f32(dgam), prec.f32(dbet)
                    add_grad(src[l], dx)
                elif k == "maxpool3":
                    add_grad(src[l], resnet.maxpool3_backward(x, g.reshape(out_shape(sp, B))))
                else:  # avgpool
                    add_grad(src[l], resnet.avgpool_backward(x.shape, g.reshape(B, -1)))
            if s > 0:
                bwd_msg[(s - 1, j)] = G.pop(bounds[s] - 1).reshape(B, -1)
            grads_w[(s, j)] = (gw, gb)
            consumers[s][vf].discard(j)
            if not consumers[s][vf] and vf != latest[s]:
                versions[s].pop(vf, None)
            trace.append(TraceRow(s, "B", j, -1, v_used, vl, delta, alpha, beta))
        else:
            j = e.mb
            gw, gb = grads_w.pop((s, j))
            for l in ls:
                if l in gw:
                    W[l], VW[l] = mlp.sgd_update(W[l], VW[l], gw[l], lr, mu, wd, exact)
                    W[l] = np.asarray(W[l], np.float64); VW[l] = np.asarray(VW[l], np.float64)
                if l in gb:
                    Bv[l], Vb[l] = mlp.sgd_update(Bv[l], Vb[l], gb[l], lr, mu, wd, exact)
                    Bv[l] = np.asarray(Bv[l], np.float64); Vb[l] = np.asarray(Vb[l], np.float64)
            old = latest[s]
            latest[s] = old + 1
            versions[s][latest[s]] = {l: store_w(l) for l in ls}
            if variant == staleness.V_VARIANT or not consumers[s].get(old):
                versions[s].pop(old, None)
            trace.append(TraceRow(s, "U", j, -1, old, latest[s], 0))
    f32 = (lambda x: x) if exact else (lambda x: np.asarray(x, np.float32))
    return Result(losses=loss_sum / B,
                  weights=[f32(w) if w is not None else None for w in W],
                  biases=[f32(x) if x is not None else None for x in Bv],
                  mom_w=[np.asarray(x, np.float32) if x is not None else None for x in VW],
                  mom_b=[np.asarray(x, np.float32) if x is not None else None for x in Vb],
                  trace=trace, peak_versions=[])


# ------------------------------------------------------------------ ResNet builders
def bottleneck(layers, cin, width, stride, h, w, downsample):
    """Appends one v1.5 bottleneck (stride on the 3x3 conv); returns (cout, ho, wo)."""
    cout = 4 * width
    x = len(layers) - 1                                   # block input tensor
    ho, wo = (h - 1) // stride + 1, (w - 1) // stride + 1
    layers.append({"kind": "conv", "cin": cin, "cout": width, "k": 1, "s": 1, "p": 0, "h": h, "w": w, "src": x})
    layers.append({"kind": "bn", "c": width, "h": h, "w": w, "relu": True})
    layers.append({"kind": "conv", "cin": width, "cout": width, "k": 3, "s": stride, "p": 1, "h": h, "w": w})
    layers.append({"kind": "bn", "c": width, "h": ho, "w": wo, "relu": True})
    layers.append({"kind": "conv", "cin": width, "cout": cout, "k": 1, "s": 1, "p": 0, "h": ho, "w": wo})
    c3 = len(layers) - 1
    res = x
    if downsample:
        layers.append({"kind": "conv", "cin": cin, "cout": cout, "k": 1, "s": stride, "p": 0, "h": h, "w": w,
                       "src": x})
        layers.append({"kind": "bn", "c": cout, "h": ho, "w": wo, "relu": False})
        res = len(layers) - 1
    layers.append({"kind": "bn", "c": cout, "h": ho, "w": wo, "relu": True, "src": c3, "res": res})
    return cout, ho, wo


def resnet_layers(blocks=(3, 4, 6, 3), widths=(64, 128, 256, 512), H=224, classes=1000, stem_c=64):
    """ResNet v1.5 layer graph; returns (layers, block_bounds) where block_bounds are the layer
    indices at which a stage may start (after the stem and after every bottleneck)."""
    layers = [{"kind": "conv", "cin": 3, "cout": stem_c, "k": 7, "s": 2, "p": 3, "h": H, "w": H},
              {"kind": "bn", "c": stem_c, "h": H // 2, "w": H // 2, "relu": True},
              {"kind": "maxpool3", "c": stem_c, "h": H // 2, "w": H // 2}]
    starts = [0, len(layers)]
    c, h = stem_c, (H // 2 - 1) // 2 + 1
    for i, (n, wdt) in enumerate(zip(blocks, widths)):
        for bi in range(n):
            stride = 2 if (bi == 0 and i > 0) else 1
            c, h, _ = bottleneck(layers, c, wdt, stride, h, h, downsample=(bi == 0))
            starts.append(len(layers))
    layers.append({"kind": "avgpool", "c": c, "h": h, "w": h})
    layers.append({"kind": "linear", "in": c, "out": classes})
    return layers, starts

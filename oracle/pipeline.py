"""Whole-pipeline replay of V- and I-TiMePReSt on an MLP or a conv net (TEST INFRASTRUCTURE ONLY).

All S stages live in one address space and fire in the order produced by
`schedule.execute` (a dependency-driven round-robin over the static per-stage
orders, readings Z6/Z7).

Per stage s: consecutive layers [bounds[s], bounds[s+1]); stage 0 reads
the inputs; the last stage computes the loss; activations go forward per
micro-batch and activation-gradients go backward once per mini-batch.

Weight versions (one update per mini-batch per stage):
  * forwards use the stage's LATEST version, for V and I (Z8);
  * V backward: the latest version; each superseded version is dropped as soon
    as the next exists -> never more than one live version;
  * I backward: W_res = α·W(x|y) + β·W_latest with δ = y - x (Eq. 1
    P:220; reading Z1); the stashed W(x|y) is kept until its last consumer has
    computed its intermediate weight, then evicted.
  * update base: the fp32 master of the latest weights (reading Z9).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import conv, mlp, schedule, staleness


@dataclass
class Config:
    dims: list[int]                  # MLP: [d0, d1, ..., dL]; layer l maps d_l -> d_{l+1}
                                     # (image nets: [input features, ..., classes], informational)
    stage_bounds: list[int]          # S+1 entries, stage s owns layers [b[s], b[s+1])
    m: int                           # micro-batches per mini-batch
    b: int                           # rows per micro-batch
    M: int                           # mini-batches in the run
    variant: str = staleness.I_VARIANT
    blend: str = staleness.EQ1
    lam: float = 0.05
    lr: float = 0.01
    momentum: float = 0.0
    wd: float = 0.0
    exact: bool = False
    # optional layer list for image nets (oracle/conv.py); None => Linear layers from dims.
    # entries: {"kind": "linear", "in", "out"} | {"kind": "conv3", "cin", "cout", "h", "w"}
    #          | {"kind": "pool2", "c", "h", "w"}; every layer but the last is followed by ReLU
    #          (pools pass values through); the last is the Linear head.
    layers: list | None = None
    # mini-batches in flight for a ONE-stage pipeline (0 => S - s; schedule.inflight)
    max_inflight: int = 0
    # storage precision of activations / weight copies / gradients (Z13 bf16; Z28 tf32)
    dtype: str = "bf16"

    @property
    def S(self) -> int:
        return len(self.stage_bounds) - 1

    @property
    def L(self) -> int:
        return len(self.layers) if self.layers else len(self.dims) - 1

    def specs(self) -> list[dict]:
        if self.layers:
            return self.layers
        return [{"kind": "linear", "in": self.dims[l], "out": self.dims[l + 1]} for l in range(self.L)]

    @property
    def B(self) -> int:
        return self.m * self.b


@dataclass
class TraceRow:
    stage: int
    kind: str
    mb: int
    micro: int
    v_used: int
    v_latest: int
    delta: int
    alpha: float = 1.0
    beta: float = 0.0


@dataclass
class Result:
    losses: np.ndarray                          # [M] mean loss per mini-batch
    weights: list[np.ndarray]                   # fp32 masters per layer
    biases: list[np.ndarray]
    mom_w: list[np.ndarray]
    mom_b: list[np.ndarray]
    trace: list[TraceRow]
    peak_versions: list[int]                    # per stage, at event boundaries
    versions_bf16: list[np.ndarray] = field(default_factory=list)  # latest bf16 copy per layer


def run(cfg: Config, xs: list[np.ndarray], ys: list[np.ndarray],
        w0: list[np.ndarray], b0: list[np.ndarray]) -> Result:
    """Train M mini-batches; xs[j] is [B, d0] (bf16-exact), ys[j] is [B] int."""
    S, L, B, m, bsz = cfg.S, cfg.L, cfg.B, cfg.m, cfg.b
    prec = mlp.Precision(cfg.exact, cfg.dtype)
    assert cfg.dtype in ("bf16", "tf32")
    assert cfg.stage_bounds[0] == 0 and cfg.stage_bounds[-1] == L
    stage_of = {}
    for s in range(S):
        for l in range(cfg.stage_bounds[s], cfg.stage_bounds[s + 1]):
            stage_of[l] = s

    spec = cfg.specs()
    has_w = [sp["kind"] != "pool2" for sp in spec]
    cast = (lambda a: np.asarray(a, np.float64)) if cfg.exact else (lambda a: np.asarray(a, np.float32).astype(np.float64))
    W = [cast(w) if has_w[l] else None for l, w in enumerate(w0)]      # fp32 masters (as fp64 values)
    bias = [cast(x) if has_w[l] else None for l, x in enumerate(b0)]
    VW = [np.zeros_like(w) if w is not None else None for w in W]
    Vb = [np.zeros_like(x) if x is not None else None for x in bias]

    # versions[s][v] = [bf16 copy of W_l for l in stage s]
    layers = [list(range(cfg.stage_bounds[s], cfg.stage_bounds[s + 1])) for s in range(S)]
    def store_w(l):
        return prec.store(W[l]) if has_w[l] else None

    versions = [{0: [store_w(l) for l in layers[s]]} for s in range(S)]
    latest = [0] * S
    consumers: list[dict[int, set[int]]] = [dict() for _ in range(S)]
    peak = [1] * S
    fwd_ver: dict[tuple[int, int], int] = {}

    acts: dict[tuple[int, int, int], list[np.ndarray]] = {}   # (s, j, a) -> inputs of each layer
    fwd_msg: dict[tuple[int, int, int], np.ndarray] = {}      # (dest s, j, a) -> activation rows
    bwd_msg: dict[tuple[int, int], np.ndarray] = {}           # (dest s, j) -> dZ rows [B, d]
    ce_grad: dict[tuple[int, int], np.ndarray] = {}           # (j, a) -> dlogits rows (stored)
    loss_sum = np.zeros(cfg.M)
    grads: dict[tuple[int, int], tuple[list, list]] = {}      # (s, j) -> (dW list, db list)
    trace: list[TraceRow] = []

    fired, _ = schedule.execute(S, m, cfg.M, cfg.max_inflight)
    for s, e in fired:
        ls = layers[s]
        if e.kind == "F":
            j, a = e.mb, e.micro
            v = latest[s]
            fwd_ver.setdefault((s, j), v)
            consumers[s].setdefault(v, set()).add(j)
            Wv = versions[s][v]
            X = xs[j][a * bsz:(a + 1) * bsz].astype(np.float64) if s == 0 else fwd_msg.pop((s, j, a))
            X = prec.store(X)
            ins = []
            for k, l in enumerate(ls):
                ins.append(X)
                sp = spec[l]
                if sp["kind"] == "pool2":
                    X = conv.maxpool2_forward(X.reshape(-1, sp["h"], sp["w"], sp["c"])).reshape(X.shape[0], -1)
                    continue
                if sp["kind"] == "conv3":
                    Z = conv.conv3x3_forward(X.reshape(-1, sp["h"], sp["w"], sp["cin"]), Wv[k], bias[l])
                    Z = Z.reshape(X.shape[0], -1)
                else:
                    Z = mlp.linear_forward(X, Wv[k], bias[l])
                if l < L - 1:
                    X = prec.store(mlp.relu(Z))
                else:
                    rows, G = mlp.softmax_xent(Z, ys[j][a * bsz:(a + 1) * bsz], B)
                    loss_sum[j] += rows.sum()
                    ce_grad[(j, a)] = prec.store(G)
            acts[(s, j, a)] = ins
            if s < S - 1:
                fwd_msg[(s + 1, j, a)] = X
            trace.append(TraceRow(s, "F", j, a, v, v, 0))
        elif e.kind == "B":
            j = e.mb
            vf = fwd_ver[(s, j)]
            vl = latest[s]
            if cfg.variant == staleness.V_VARIANT:
                delta, v_used = 0, vl                 # V: latest weights, zero staleness
                alpha, beta = staleness.blend_coeffs(cfg.variant, cfg.blend, 0, cfg.lam)
                Wst = versions[s][vl]
            else:
                delta, v_used = vl - vf, vf
                alpha, beta = staleness.blend_coeffs(cfg.variant, cfg.blend, delta, cfg.lam)
                Wst = versions[s][vf]
            Wl = versions[s][vl]
            if s == S - 1:
                G = np.concatenate([ce_grad.pop((j, a)) for a in range(m)], axis=0)
            else:
                G = bwd_msg.pop((s, j))
            ins = [np.concatenate([acts[(s, j, a)][k] for a in range(m)], axis=0) for k in range(len(ls))]
            for a in range(m):
                del acts[(s, j, a)]
            dWs, dbs = [None] * len(ls), [None] * len(ls)
            for k in reversed(range(len(ls))):
                l = ls[k]
                sp = spec[l]
                X = ins[k]
                if sp["kind"] == "pool2":
                    # route to the first window maximum; no rounding (values are copied)
                    G = conv.maxpool2_backward(X.reshape(-1, sp["h"], sp["w"], sp["c"]),
                                               G.reshape(-1, sp["h"] // 2, sp["w"] // 2, sp["c"])).reshape(X.shape[0], -1)
                    continue
                if sp["kind"] == "conv3":
                    X4 = X.reshape(-1, sp["h"], sp["w"], sp["cin"])
                    G4 = G.reshape(-1, sp["h"], sp["w"], sp["cout"])
                    dW, db = conv.conv3x3_wgrad(G4, X4)
                else:
                    dW, db = mlp.wgrad(G, X)
                dWs[k], dbs[k] = prec.f32(dW), prec.f32(db)
                if l > 0:
                    Wres = mlp.resolve_backward_weight(Wst[k], Wl[k], alpha, beta)
                    if sp["kind"] == "conv3":
                        dX = conv.conv3x3_dgrad(G4, Wres).reshape(X.shape[0], -1)
                    else:
                        dX = G @ Wres
                    G = prec.store(dX * (X > 0))     # ReLU mask from the stored input (Z15)
            if s > 0:
                bwd_msg[(s - 1, j)] = G
            grads[(s, j)] = (dWs, dbs)
            # I: the stash of version vf loses consumer j once its intermediate weight is computed
            consumers[s][vf].discard(j)
            if not consumers[s][vf] and vf != latest[s]:
                versions[s].pop(vf, None)
            trace.append(TraceRow(s, "B", j, -1, v_used, vl, delta, alpha, beta))
        else:  # "U"
            j = e.mb
            dWs, dbs = grads.pop((s, j))
            for k, l in enumerate(ls):
                if not has_w[l]:
                    continue
                W[l], VW[l] = mlp.sgd_update(W[l], VW[l], dWs[k], cfg.lr, cfg.momentum, cfg.wd, cfg.exact)
                bias[l], Vb[l] = mlp.sgd_update(bias[l], Vb[l], dbs[k], cfg.lr, cfg.momentum, cfg.wd, cfg.exact)
                W[l] = np.asarray(W[l], np.float64); VW[l] = np.asarray(VW[l], np.float64)
                bias[l] = np.asarray(bias[l], np.float64); Vb[l] = np.asarray(Vb[l], np.float64)
            old = latest[s]
            latest[s] = old + 1
            versions[s][latest[s]] = [store_w(l) for l in ls]
            peak[s] = max(peak[s], len(versions[s]))   # transient: old + new coexist
            if cfg.variant == staleness.V_VARIANT or not consumers[s].get(old):
                versions[s].pop(old, None)            # V drops the superseded version at once
            trace.append(TraceRow(s, "U", j, -1, old, latest[s], 0))
    # peak at event boundaries (SPEC S:205 semantics): recompute without the transient
    peak_boundary = _peak_at_boundaries(cfg, trace)
    return Result(
        losses=loss_sum / B,
        weights=[(np.asarray(w, np.float32) if not cfg.exact else w) if w is not None else None for w in W],
        biases=[(np.asarray(x, np.float32) if not cfg.exact else x) if x is not None else None for x in bias],
        mom_w=[np.asarray(x, np.float32) if x is not None else None for x in VW],
        mom_b=[np.asarray(x, np.float32) if x is not None else None for x in Vb],
        trace=trace,
        peak_versions=peak_boundary,
        versions_bf16=[versions[stage_of[l]][latest[stage_of[l]]][layers[stage_of[l]].index(l)]
                       for l in range(L)],
    )


def _peak_at_boundaries(cfg: Config, trace: list[TraceRow]) -> list[int]:
    """Peak number of live weight versions per stage between events.

    V: exactly one.  I: versions still referenced by a mini-batch whose
    forward has run but whose backward has not, plus the latest.
    """
    S = cfg.S
    out = []
    for s in range(S):
        if cfg.variant == staleness.V_VARIANT:
            out.append(1)
            continue
        live_refs: dict[int, set[int]] = {}
        latest = 0
        best = 1
        for r in trace:
            if r.stage != s:
                continue
            if r.kind == "F":
                live_refs.setdefault(r.v_used, set()).add(r.mb)
            elif r.kind == "B":
                live_refs[r.v_used].discard(r.mb)
            else:
                latest = r.v_latest
            live = {v for v, refs in live_refs.items() if refs} | {latest}
            best = max(best, len(live))
        out.append(best)
    return out

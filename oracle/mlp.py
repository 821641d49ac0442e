"""Stage math of the MLP pipeline: Linear/ReLU forward, softmax cross-entropy,
dgrad on the resolved weight, wgrad, SGD/momentum update (TEST INFRASTRUCTURE ONLY).

Paper passages:
  * each node computes its consecutive layers and passes the output on; the loss
    is computed at the last node and the backward runs in reverse;
  * one collective backward over all micro-batches of a mini-batch,
    read as the mean loss over the B = m·b rows (reading Z11);
  * the backward runs on the resolved weight: latest for V,
    the intermediate weight W_i(x,y) for I (Eq. 1);
  * weights are updated once per mini-batch; optimizer unstated -> SGD
    with PyTorch's momentum convention (reading Z10), update base = the latest
    fp32 master (reading Z9).

Precision (reading Z13): inputs/weights/activations/activation-gradients are
bf16 values (tf32 values in tf32 mode, reading Z28; held here as fp64 numbers); products and sums are fp64; weight
gradients are rounded to fp32; the update is numpy float32, one rounding per
operation.  `Precision(exact=True)` disables every rounding (finite-difference
and autograd pins).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import bf16, tf32


@dataclass(frozen=True)
class Precision:
    exact: bool = False
    dtype: str = "bf16"        # storage of activations / weight copies / gradients: "bf16" | "tf32"

    def store(self, x: np.ndarray) -> np.ndarray:
        """Value as stored in a bf16 tensor (Z13), or in a tf32 tensor in tf32 mode (Z28)."""
        if self.exact:
            return np.asarray(x, dtype=np.float64)
        return tf32.rna(x) if self.dtype == "tf32" else bf16.rne(x)

    def f32(self, x: np.ndarray) -> np.ndarray:
        """Value as stored in an fp32 tensor."""
        x = np.asarray(x, dtype=np.float64)
        return x if self.exact else x.astype(np.float32).astype(np.float64)


def linear_forward(X: np.ndarray, W: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Z = X·Wᵀ + b in fp64 (X [rows, in], W [out, in], b [out])."""
    return X @ W.T + b[None, :]


def relu(Z: np.ndarray) -> np.ndarray:
    """max(Z, 0)."""
    return np.maximum(Z, 0.0)


def softmax_xent(logits: np.ndarray, y: np.ndarray, batch: int) -> tuple[np.ndarray, np.ndarray]:
    """Per-row loss logsumexp(z) - z_y, and dlogits = (softmax(z) - onehot(y)) / batch.

    `batch` is the mini-batch size B = m·b: the loss of a mini-batch is the mean
    over all its rows (reading Z11), so each row's gradient carries 1/B.
    """
    z = np.asarray(logits, dtype=np.float64)
    zmax = z.max(axis=1, keepdims=True)
    e = np.exp(z - zmax)
    se = e.sum(axis=1, keepdims=True)
    lse = zmax[:, 0] + np.log(se[:, 0])
    rows = np.arange(z.shape[0])
    loss_rows = lse - z[rows, y]
    p = e / se
    p[rows, y] -= 1.0
    return loss_rows, p / batch


def wgrad(G: np.ndarray, X: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """dW = Gᵀ·X, db = Σ_rows G (fp64; caller rounds)."""
    return G.T @ X, G.sum(axis=0)


def dgrad(G: np.ndarray, W_res: np.ndarray, X_in: np.ndarray) -> np.ndarray:
    """dZ_{prev} = (G·W_res) ⊙ 1[X_in > 0]: gradient w.r.t. this layer's input,
    masked by the ReLU that produced that input (ReLU'(0) = 0, reading Z15)."""
    return (G @ W_res) * (X_in > 0)


def resolve_backward_weight(W_stash: np.ndarray, W_latest: np.ndarray,
                            alpha: float, beta: float) -> np.ndarray:
    """W_res = α·W_stash + β·W_latest in fp64, unrounded (reading Z1, Z14)."""
    return alpha * W_stash + beta * W_latest


def materialize_blend(W_stash_bf16: np.ndarray, W_latest_bf16: np.ndarray,
                      alpha: float, beta: float, dtype: str = "bf16") -> np.ndarray:
    """K8 debug materialiser definition (reading Z14):
    bf16_rne(fp32(fp32(α·s) + fp32(β·l))), every op a single fp32 rounding
    (tf32 mode: tf32_rna of the same fp32 sum, reading Z28)."""
    a = np.float32(alpha)
    b = np.float32(beta)
    s = np.asarray(W_stash_bf16, dtype=np.float32)
    l = np.asarray(W_latest_bf16, dtype=np.float32)
    with np.errstate(over="ignore", invalid="ignore"):
        t = (a * s).astype(np.float32) + (b * l).astype(np.float32)
    t = t.astype(np.float32)
    return tf32.rna(t) if dtype == "tf32" else bf16.rne(t)


def sgd_update(w: np.ndarray, v: np.ndarray, g: np.ndarray, lr: float, mu: float,
               wd: float, exact: bool = False) -> tuple[np.ndarray, np.ndarray]:
    """PyTorch-convention SGD with momentum (reading Z10), in this op order:
        g' = g + wd·w ;  v = μ·v + g' ;  w = w - lr·v
    numpy float32 with one rounding per op (no fused multiply-add)."""
    if exact:
        w = np.asarray(w, np.float64); v = np.asarray(v, np.float64); g = np.asarray(g, np.float64)
        gp = g + wd * w
        v = mu * v + gp
        return w - lr * v, v
    f = np.float32
    w = np.asarray(w, np.float32); v = np.asarray(v, np.float32); g = np.asarray(g, np.float32)
    gp = (g + (f(wd) * w).astype(np.float32)).astype(np.float32)
    v = ((f(mu) * v).astype(np.float32) + gp).astype(np.float32)
    w = (w - (f(lr) * v).astype(np.float32)).astype(np.float32)
    return w, v

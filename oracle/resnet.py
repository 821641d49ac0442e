"""ResNet-50 stage math (BASELINE.json configs[3]) — TEST INFRASTRUCTURE ONLY.

The paper trains ResNet-50 with the pipeline but states no layer math; these are
the textbook definitions (NHWC, fp64 arithmetic, bf16 storage per reading Z13):

  conv (kernel k, stride s, zero padding p, no bias):
      Z[n,ho,wo,o] = Σ_{kh,kw,i} X[n, s·ho+kh-p, s·wo+kw-p, i] · W[o,kh,kw,i]
  batch norm, training mode, statistics of ONE micro-batch (reading Z22: the forward runs per
  micro-batch), biased variance, ε = 1e-5:
      x̂ = (x - μ)/sqrt(σ² + ε);  y = γ·x̂ + β  (+ residual)  then ReLU if the layer has one
  its gradient (per micro-batch segment, then dγ, dβ summed over the mini-batch):
      dβ = Σ dy ; dγ = Σ dy·x̂ ; dx = γ/sqrt(σ²+ε) · (dy - mean(dy) - x̂·mean(dy·x̂))
  max pool 3x3 / stride 2 / pad 1 (gradient to the first maximum in row-major window order,
  padding never wins; reading Z15), global average pool.
"""
from __future__ import annotations

import numpy as np

BN_EPS = 1e-5


def im2col(X: np.ndarray, k: int, s: int, p: int) -> tuple[np.ndarray, int, int]:
    """[N,H,W,C] -> ([N*Ho*Wo, k*k*C], Ho, Wo); column order (kh, kw, c)."""
    N, H, W, C = X.shape
    Ho, Wo = (H + 2 * p - k) // s + 1, (W + 2 * p - k) // s + 1
    Xp = np.zeros((N, H + 2 * p, W + 2 * p, C))
    Xp[:, p:p + H, p:p + W, :] = X
    cols = np.empty((N, Ho, Wo, k, k, C))
    for kh in range(k):
        for kw in range(k):
            cols[:, :, :, kh, kw, :] = Xp[:, kh:kh + s * (Ho - 1) + 1:s, kw:kw + s * (Wo - 1) + 1:s, :]
    return cols.reshape(N * Ho * Wo, k * k * C), Ho, Wo


def col2im(cols: np.ndarray, shape: tuple, k: int, s: int, p: int) -> np.ndarray:
    """Adjoint of im2col: scatter-add patch gradients back to [N,H,W,C]."""
    N, H, W, C = shape
    Ho, Wo = (H + 2 * p - k) // s + 1, (W + 2 * p - k) // s + 1
    c6 = cols.reshape(N, Ho, Wo, k, k, C)
    Xp = np.zeros((N, H + 2 * p, W + 2 * p, C))
    for kh in range(k):
        for kw in range(k):
            Xp[:, kh:kh + s * (Ho - 1) + 1:s, kw:kw + s * (Wo - 1) + 1:s, :] += c6[:, :, :, kh, kw, :]
    return Xp[:, p:p + H, p:p + W, :]


def conv_forward(X, W, s, p):
    N = X.shape[0]
    Co, k = W.shape[0], W.shape[1]
    cols, Ho, Wo = im2col(X, k, s, p)
    return (cols @ W.reshape(Co, -1).T).reshape(N, Ho, Wo, Co)


def conv_dgrad(dZ, W, x_shape, s, p):
    Co, k = W.shape[0], W.shape[1]
    dcols = dZ.reshape(-1, Co) @ W.reshape(Co, -1)
    return col2im(dcols, x_shape, k, s, p)


def conv_wgrad(dZ, X, k, s, p):
    Co = dZ.shape[-1]
    cols, _, _ = im2col(X, k, s, p)
    return (dZ.reshape(-1, Co).T @ cols).reshape(Co, k, k, X.shape[-1])


def bn_forward(x: np.ndarray, gamma: np.ndarray, beta: np.ndarray):
    """One micro-batch segment [n,H,W,C]: returns (γ·x̂ + β, mean, invstd)."""
    C = x.shape[-1]
    flat = x.reshape(-1, C)
    mu = flat.mean(axis=0)
    var = ((flat - mu) ** 2).mean(axis=0)               # biased
    invstd = 1.0 / np.sqrt(var + BN_EPS)
    xhat = (x - mu) * invstd
    return gamma * xhat + beta, mu, invstd


def bn_backward(dy: np.ndarray, x: np.ndarray, gamma: np.ndarray, mu: np.ndarray, invstd: np.ndarray):
    """One segment: (dx, dγ, dβ)."""
    C = x.shape[-1]
    xhat = (x - mu) * invstd
    d = dy.reshape(-1, C)
    xh = xhat.reshape(-1, C)
    dbeta = d.sum(axis=0)
    dgamma = (d * xh).sum(axis=0)
    m = d.shape[0]
    dx = gamma * invstd * (d - dbeta / m - xh * (dgamma / m))
    return dx.reshape(x.shape), dgamma, dbeta


def maxpool3_forward(X):
    """3x3 / stride 2 / pad 1 (pad = -inf)."""
    N, H, W, C = X.shape
    Ho, Wo = (H - 1) // 2 + 1, (W - 1) // 2 + 1
    Xp = np.full((N, H + 2, W + 2, C), -np.inf)
    Xp[:, 1:H + 1, 1:W + 1, :] = X
    Y = np.full((N, Ho, Wo, C), -np.inf)
    for kh in range(3):
        for kw in range(3):
            Y = np.maximum(Y, Xp[:, kh:kh + 2 * (Ho - 1) + 1:2, kw:kw + 2 * (Wo - 1) + 1:2, :])
    return Y


def maxpool3_backward(X, dY):
    """Each output's gradient goes to the first maximum of its window in row-major order."""
    N, H, W, C = X.shape
    Ho, Wo = dY.shape[1], dY.shape[2]
    Xp = np.full((N, H + 2, W + 2, C), -np.inf)
    Xp[:, 1:H + 1, 1:W + 1, :] = X
    win = np.stack([Xp[:, kh:kh + 2 * (Ho - 1) + 1:2, kw:kw + 2 * (Wo - 1) + 1:2, :]
                    for kh in range(3) for kw in range(3)], axis=-1)        # [N,Ho,Wo,C,9]
    first = np.argmax(win, axis=-1)
    dXp = np.zeros((N, H + 2, W + 2, C))
    for t in range(9):
        kh, kw = divmod(t, 3)
        sel = (first == t) * dY
        dXp[:, kh:kh + 2 * (Ho - 1) + 1:2, kw:kw + 2 * (Wo - 1) + 1:2, :] += sel
    return dXp[:, 1:H + 1, 1:W + 1, :]


def avgpool_forward(X):
    return X.mean(axis=(1, 2))


def avgpool_backward(X_shape, dY):
    N, H, W, C = X_shape
    return np.broadcast_to(dY[:, None, None, :] / (H * W), X_shape).copy()

"""Convolution and pooling stage math for the image-classifier configs (VGG-16 on
CIFAR-shaped inputs, BASELINE.json configs[2]) — TEST INFRASTRUCTURE ONLY.

The paper trains VGG-16 and ResNet-50 with the pipeline but gives no
layer math; these are the textbook definitions written out (NHWC layout, bf16
storage per reading Z13, fp64 arithmetic):

  conv3x3 (stride 1, zero padding 1):
      Z[n,h,w,o] = b[o] + Σ_{kh,kw,i} X[n, h+kh-1, w+kw-1, i] · W[o, kh, kw, i]
  its input gradient:
      dX[n,h,w,i] = Σ_{kh,kw,o} dZ[n, h-kh+1, w-kw+1, o] · W[o, kh, kw, i]
  its weight gradient:
      dW[o,kh,kw,i] = Σ_{n,h,w} dZ[n,h,w,o] · X[n, h+kh-1, w+kw-1, i],  db[o] = Σ dZ[...,o]
  maxpool 2x2 / stride 2:  Y[n,i,j,c] = max of the 2x2 window; the gradient goes to the
      first maximum in row-major window order (reading Z15).

`im2col` gathers the 3x3 neighbourhood of every output pixel into a row ordered
(kh, kw, i) — the same order as a weight row W[o, :, :, :] — so a convolution is one
matrix product (a library primitive), with no other restructuring.
"""
from __future__ import annotations

import numpy as np


def im2col3x3(X: np.ndarray) -> np.ndarray:
    """[N,H,W,C] -> [N*H*W, 9*C], row (n,h,w), column (kh, kw, c), zero padding 1."""
    N, H, W, C = X.shape
    Xp = np.zeros((N, H + 2, W + 2, C), dtype=np.float64)
    Xp[:, 1:H + 1, 1:W + 1, :] = X
    cols = np.empty((N, H, W, 3, 3, C), dtype=np.float64)
    for kh in range(3):
        for kw in range(3):
            cols[:, :, :, kh, kw, :] = Xp[:, kh:kh + H, kw:kw + W, :]
    return cols.reshape(N * H * W, 9 * C)


def conv3x3_forward(X: np.ndarray, W: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Z = conv3x3(X; W) + b.  X [N,H,W,Ci], W [Co,3,3,Ci] -> Z [N,H,W,Co]."""
    N, H, Wd, _ = X.shape
    Co = W.shape[0]
    Z = im2col3x3(X) @ W.reshape(Co, -1).T + b[None, :]
    return Z.reshape(N, H, Wd, Co)


def conv3x3_dgrad(dZ: np.ndarray, W: np.ndarray) -> np.ndarray:
    """dX[n,h,w,i] = Σ_{kh,kw,o} dZ[n,h-kh+1,w-kw+1,o] · W[o,kh,kw,i] (zero outside)."""
    N, H, Wd, Co = dZ.shape
    Ci = W.shape[3]
    # the sum over (kh, kw) of shifted dZ equals im2col(dZ) against the spatially flipped,
    # channel-transposed kernel: Wf[i, kh', kw', o] = W[o, 2-kh', 2-kw', i]
    Wf = W[:, ::-1, ::-1, :].transpose(3, 1, 2, 0)
    dX = im2col3x3(dZ) @ Wf.reshape(Ci, -1).T
    return dX.reshape(N, H, Wd, Ci)


def conv3x3_wgrad(dZ: np.ndarray, X: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """dW [Co,3,3,Ci] and db [Co]."""
    N, H, Wd, Co = dZ.shape
    Ci = X.shape[3]
    G = dZ.reshape(-1, Co)
    dW = G.T @ im2col3x3(X)
    return dW.reshape(Co, 3, 3, Ci), G.sum(axis=0)


def maxpool2_forward(X: np.ndarray) -> np.ndarray:
    """2x2 max, stride 2.  [N,H,W,C] -> [N,H/2,W/2,C]."""
    N, H, W, C = X.shape
    return X.reshape(N, H // 2, 2, W // 2, 2, C).max(axis=(2, 4))


def maxpool2_backward(X: np.ndarray, dY: np.ndarray) -> np.ndarray:
    """Route dY to the FIRST maximum of each window in row-major order (reading Z15)."""
    N, H, W, C = X.shape
    win = X.reshape(N, H // 2, 2, W // 2, 2, C).transpose(0, 1, 3, 5, 2, 4).reshape(N, H // 2, W // 2, C, 4)
    first = np.argmax(win, axis=-1)            # np.argmax returns the first occurrence
    dwin = np.zeros_like(win)
    np.put_along_axis(dwin, first[..., None], dY[..., None], axis=-1)
    return dwin.reshape(N, H // 2, W // 2, C, 2, 2).transpose(0, 1, 4, 2, 5, 3).reshape(N, H, W, C)

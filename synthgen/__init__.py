"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds NO arithmetic of the method (no schedule, no staleness, no
layer math).  It only turns (seed, tensor id, element index) into numbers via
a counter-based splitmix64 hash, so both sides can draw the same inputs:

    h(seed, tid, i) = mix(mix(mix(seed) ^ tid) ^ i)        (uint64, wrapping)
    mix(x): z = x + 0x9E3779B97F4A7C15
            z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9
            z = (z ^ (z >> 27)) * 0x94D049BB133111EB
            return z ^ (z >> 31)

The CUDA library implements the same counter-based generator on the device
(`tps_fill_synthetic` in include/tps.h) so full-size benchmarks need not ship
gigabytes over PCIe; tests check the two agree bit for bit.

Recipes:
  * images / MNIST-like inputs:  x = (h & 0xFF) / 256        in [0, 1)
  * MLP-B/C inputs:              x = ((h & 0xFF) - 128)/128  in [-1, 1)
  * labels:                      y = (h >> 8) mod C
  * weights (fan_in k):          w = ((h >> 40) - 2^23) * 2^-23 * 2^-round(log2(sqrt k))
    (24-bit two's-complement mantissa -> exact in fp32); biases start at 0.
All values above are exact in fp32, and x values are exact in bf16.
"""
from __future__ import annotations

import math

import numpy as np

_M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
C1 = 0xBF58476D1CE4E5B9
C2 = 0x94D049BB133111EB

# tensor-id namespaces (must match csrc/synth.cu)
TID_WEIGHT = 0x0100      # + global layer index
TID_X = 0x10000          # + mini-batch index
TID_Y = 0x20000          # + mini-batch index

X_SIGNED = 0             # ((h & 0xFF) - 128) / 128
X_UNIT = 1               # (h & 0xFF) / 256


def _mix_scalar(x: int) -> int:
    z = (x + GOLDEN) & _M64
    z = ((z ^ (z >> 30)) * C1) & _M64
    z = ((z ^ (z >> 27)) * C2) & _M64
    return z ^ (z >> 31)


def _mix_array(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = z + np.uint64(GOLDEN)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(C1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(C2)
        return z ^ (z >> np.uint64(31))


def hash_stream(seed: int, tid: int, n: int, start: int = 0) -> np.ndarray:
    """h(seed, tid, i) for i in [start, start + n) as uint64."""
    key = _mix_scalar(_mix_scalar(seed & _M64) ^ (tid & _M64))
    idx = np.arange(start, start + n, dtype=np.uint64)
    return _mix_array(idx ^ np.uint64(key))


def weight_shift(fan_in: int) -> int:
    """round(log2(sqrt(fan_in))) -- the power-of-two init scale exponent."""
    return int(round(math.log2(math.sqrt(fan_in))))


def weights(seed: int, layer: int, out_f: int, in_f: int) -> np.ndarray:
    """fp32 [out_f, in_f] initial weight matrix of global layer `layer`."""
    h = hash_stream(seed, TID_WEIGHT + layer, out_f * in_f)
    mant = (h >> np.uint64(40)).astype(np.int64) - (1 << 23)
    w = mant.astype(np.float64) * 2.0 ** (-23 - weight_shift(in_f))
    return w.astype(np.float32).reshape(out_f, in_f)


def inputs(seed: int, mb: int, rows: int, feat: int, kind: int = X_SIGNED) -> np.ndarray:
    """fp32 [rows, feat] inputs of mini-batch `mb` (exact in bf16)."""
    h = hash_stream(seed, TID_X + mb, rows * feat)
    b = (h & np.uint64(0xFF)).astype(np.float64)
    x = (b - 128.0) / 128.0 if kind == X_SIGNED else b / 256.0
    return x.astype(np.float32).reshape(rows, feat)


def labels(seed: int, mb: int, rows: int, classes: int) -> np.ndarray:
    """int32 [rows] labels of mini-batch `mb`."""
    h = hash_stream(seed, TID_Y + mb, rows)
    return ((h >> np.uint64(8)) % np.uint64(classes)).astype(np.int32)

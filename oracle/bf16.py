"""bfloat16 storage emulation (reading Z13: bf16 storage, round-to-nearest-even).

The paper states no precision (P:259 names only the GPUs).  DESIGN.md Z13 fixes
bf16 storage for activations, weight copies, stash and activation-gradients,
with IEEE round-to-nearest-even.  `rne` rounds fp64 values to the nearest
bf16 value (8 significant bits, exponent range of fp32, subnormals kept) in a
single rounding step and returns them as fp64.
"""
from __future__ import annotations

import numpy as np

_EMIN = -126                 # smallest normal exponent of bf16 (= fp32)
_SUB_Q = 2.0 ** -133         # bf16 subnormal quantum: 2^(emin - 7)
_MAX = (2.0 - 2.0 ** -7) * 2.0 ** 127
_OVF = (2.0 - 2.0 ** -8) * 2.0 ** 127   # halfway to the next binade -> rounds to inf


def rne(x) -> np.ndarray:
    """Round to the nearest bf16 value, ties to even; returns fp64."""
    x = np.asarray(x, dtype=np.float64)
    out = np.empty_like(x)
    ax = np.abs(x)
    small = ax < 2.0 ** _EMIN
    # subnormal range: fixed quantum 2^-133, np.rint rounds half to even
    out[small] = np.rint(x[small] / _SUB_Q) * _SUB_Q
    big = ~small & np.isfinite(x)
    m, e = np.frexp(x[big])               # x = m * 2^e, 0.5 <= |m| < 1
    out[big] = np.ldexp(np.rint(m * 256.0), e - 8)
    nonfin = ~np.isfinite(x)
    out[nonfin] = x[nonfin]
    ovf = np.isfinite(x) & (ax >= _OVF)
    out[ovf] = np.copysign(np.inf, x[ovf])
    return out


def to_bits(x) -> np.ndarray:
    """bf16 bit patterns (uint16) of values that are already bf16-exact."""
    f = np.asarray(x, dtype=np.float32)
    return (f.view(np.uint32) >> np.uint32(16)).astype(np.uint16)


def from_bits(b) -> np.ndarray:
    """fp64 values of bf16 bit patterns (uint16)."""
    u = np.asarray(b, dtype=np.uint16).astype(np.uint32) << np.uint32(16)
    return u.view(np.float32).astype(np.float64)

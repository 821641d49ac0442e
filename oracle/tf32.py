"""tf32 storage emulation (TEST INFRASTRUCTURE ONLY; SURVEY §8(b) `tps_dtype` TPS_TF32, DESIGN
reading Z28).

The paper states no precision (P:259 names only the GPUs); the north_star allows "bf16/tf32
inputs with fp32 accumulation".  In tf32 mode every tensor that bf16 mode stores as bf16
(activations, weight copies / stash, activation-gradients; reading Z13) is stored as a tf32
value: 1 sign bit, the 8-bit fp32 exponent, 10 explicit mantissa bits (11 significant bits),
held in a 32-bit container.  SURVEY Z13: "stores rounded with cvt.rna.tf32, and the oracle
rounds RNA to 10 mantissa bits at the same points" -- round to nearest, ties AWAY from zero.

`rna` rounds fp64 values to the nearest tf32 value in one step and returns them as fp64:
normal range by scaling the significand to 11 bits, subnormal range (|x| < 2^-126) on the
fixed quantum 2^-136 (the 10 stored bits of an fp32 subnormal), overflow to ±inf once the
rounded magnitude reaches 2^128.
"""
from __future__ import annotations

import numpy as np

_EMIN = -126                 # smallest normal exponent (= fp32)
_SUB_Q = 2.0 ** -136         # tf32 subnormal quantum: 2^(emin - 10)
_SIG = 2048.0                # 2^11 significant bits


def _half_away(t: np.ndarray) -> np.ndarray:
    """Round to integer, halves away from zero."""
    return np.copysign(np.floor(np.abs(t) + 0.5), t)


def rna(x) -> np.ndarray:
    """Round to the nearest tf32 value, ties away from zero; returns fp64."""
    x = np.asarray(x, dtype=np.float64)
    out = np.empty_like(x)
    ax = np.abs(x)
    fin = np.isfinite(x)
    small = fin & (ax < 2.0 ** _EMIN)
    out[small] = _half_away(x[small] / _SUB_Q) * _SUB_Q
    big = fin & ~small
    m, e = np.frexp(x[big])               # x = m * 2^e, 0.5 <= |m| < 1
    out[big] = np.ldexp(_half_away(m * _SIG), e - 11)
    out[~fin] = x[~fin]
    ovf = fin & (np.abs(out) >= 2.0 ** 128)
    out[ovf] = np.copysign(np.inf, x[ovf])
    return out

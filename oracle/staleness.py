"""Staleness significance and intermediate-weight coefficients (TEST INFRASTRUCTURE ONLY).

Paper passages:
  * δ ≥ 0 is the degree of staleness of W_i(x|y); operationalised as the
    number of updates at stage i between the version the forward used and the
    latest at backward start (reading Z5; P:213 example: x=1, y=3 -> δ=2).
  * Eq. 2 / Eq. 11: f(δ) ≈ e^{-λδ}, λ > 0, f ∈ (0, 1].
  * Eq. 1 / Eq. 12: W_i(x,y) = (2 - 1/f(δ)) · W_i(x|y).
  * Eq. 13: -∞ < 2 - 1/f(δ) ≤ 1.
  * Appendix A.1 difference equation (Eqs. 5-10):
    f(δ + Δδ) = f(δ)(1 - λΔδ), f(0) = 1  -> (1 - λδ/n)^n -> e^{-λδ}.

Reading Z1: the kernels implement W_res = α·W_stash + β·W_latest.
  EQ1    (paper's closed form, default): α = 2 - 1/f(δ) = 2 - e^{λδ},  β = 0
  CONVEX (the prose "between stale and latest"): α = f(δ), β = 1 - f(δ)
  V-TiMePReSt: the backward reads the latest weight: α = 1 on latest.
α and β are computed in double and then rounded to fp32 (the GPU receives fp32).
"""
from __future__ import annotations

import math

import numpy as np

V_VARIANT = "V"
I_VARIANT = "I"
EQ1 = "EQ1"
CONVEX = "CONVEX"


def significance(delta: int, lam: float) -> float:
    """f(δ) = e^{-λδ} (Eq. 2; final form Eq. 11)."""
    if delta < 0:
        raise ValueError("staleness degree must be >= 0 (P:211)")
    if not lam > 0:
        raise ValueError("lambda must be > 0 (P:227)")
    return math.exp(-lam * delta)


def significance_by_difference_equation(delta: float, lam: float, n: int) -> float:
    """Appendix A.1, Eqs. 5-10: iterate f <- f(1 - λ·Δδ) with Δδ = δ/n, n times, from f(0) = 1.

    This follows the derivation's discrete form (the '-' branch kept by Eq. 11,
    P:477-483) so a test can check it converges to the closed form.
    """
    f = 1.0
    step = lam * delta / n
    for _ in range(n):
        f = f * (1.0 - step)
    return f


def intermediate_factor(f: float) -> float:
    """2 - 1/f(δ): the Eq. 1 scale of the stale weight (Eq. 12)."""
    if not (0.0 < f <= 1.0):
        raise ValueError("f must lie in (0, 1] (P:227)")
    return 2.0 - 1.0 / f


def intermediate_weights(stale: np.ndarray, delta: int, lam: float) -> np.ndarray:
    """W_i(x,y) = (2 - 1/f(δ)) · W_i(x|y), Eq. 1, in fp64."""
    return intermediate_factor(significance(delta, lam)) * np.asarray(stale, dtype=np.float64)


def blend_coeffs(variant: str, blend: str, delta: int, lam: float) -> tuple[float, float]:
    """(α, β) with W_res = α·W_stash + β·W_latest, rounded to fp32 (reading Z1, Z14).

    V: (1, 0) applied to the LATEST weight (the caller passes W_latest as the stash
    operand) — V keeps no stash.
    """
    if variant == V_VARIANT:
        return 1.0, 0.0
    if variant != I_VARIANT:
        raise ValueError(variant)
    f = significance(delta, lam)
    if blend == EQ1:
        a, b = intermediate_factor(f), 0.0
    elif blend == CONVEX:
        a, b = f, 1.0 - f
    else:
        raise ValueError(blend)
    return float(np.float32(a)), float(np.float32(b))

"""Pins for oracle.staleness: Eq. 1, Eq. 2, Eq. 13 and the Appendix A.1 derivation.

Values: SPEC.md S:240-260 examples and closed forms of PAPER.md Eqs. 1-13.
"""
import math

import numpy as np
import pytest

from oracle import staleness as st


def test_significance_closed_form_values():
    assert st.significance(0, 0.7) == 1.0                          # f(0) = 1
    assert st.significance(1, 1.0) == pytest.approx(0.36787944117144233, abs=1e-15)  # e^-1
    assert st.significance(4, 0.5) == pytest.approx(0.1353352832366127, abs=1e-15)   # e^-2


def test_significance_rejects_bad_inputs():
    with pytest.raises(ValueError):
        st.significance(-1, 0.5)
    with pytest.raises(ValueError):
        st.significance(1, 0.0)                                     # λ > 0


def test_monotone_decay():
    for lam in (0.05, 0.5, math.log(2), 3.0):
        f = [st.significance(d, lam) for d in range(12)]
        assert all(a > b for a, b in zip(f, f[1:]))
        assert all(0 < x <= 1 for x in f)                           # f ∈ (0,1], P:227


@pytest.mark.parametrize("lam,delta", [(1.0, 1), (1.0, 2), (1.0, 3), (0.05, 7)])
def test_difference_equation_converges_to_closed_form(lam, delta):
    # Appendix A.1, Eqs. 5-10: (1 - λδ/n)^n -> e^{-λδ}; SPEC S:273 bound 10λ²δ/n at n = 1e6
    n = 1_000_000
    it = st.significance_by_difference_equation(delta, lam, n)
    assert abs(it - math.exp(-lam * delta)) <= 10 * lam * lam * delta / n


def test_intermediate_factor_values():
    assert st.intermediate_factor(1.0) == 1.0                       # δ = 0 identity
    assert st.intermediate_factor(0.5) == 0.0
    assert st.intermediate_factor(math.exp(-1)) == pytest.approx(2 - math.e, abs=1e-14)


def test_eq13_range():
    # Eq. 13: -∞ < 2 - 1/f ≤ 1, equality iff f = 1
    f = np.linspace(1e-6, 1.0, 100_001)
    vals = np.array([st.intermediate_factor(x) for x in f[::97]] + [st.intermediate_factor(1.0)])
    assert (vals <= 1.0).all()
    assert (vals[:-1] < 1.0).all() and vals[-1] == 1.0


def test_intermediate_weights_examples():
    assert np.array_equal(st.intermediate_weights(np.array([2.0, -4.0]), 0, 0.3), [2.0, -4.0])
    assert st.intermediate_weights(np.array([1.0]), 1, math.log(2))[0] == pytest.approx(0.0, abs=1e-15)
    w = np.array([3.0, 0.0, -1.5])
    got = st.intermediate_weights(w, 2, 0.1)                         # × (2 - e^{0.2})
    assert np.allclose(got, w * (2 - math.exp(0.2)), rtol=1e-15, atol=0)


def test_zero_staleness_is_exact_fixed_point():
    rng = np.random.default_rng(0)
    w = rng.standard_normal(1000)
    for lam in (0.05, 0.5, 2.0):
        assert np.array_equal(st.intermediate_weights(w, 0, lam), w)
        for blend in (st.EQ1, st.CONVEX):
            a, b = st.blend_coeffs(st.I_VARIANT, blend, 0, lam)
            assert a * w[0] + b * w[0] == w[0] and (a, b) in ((1.0, 0.0),)


def test_blend_coeffs_ln2_exact_table():
    # λ = ln 2: f = 2^-δ, EQ1 α = 2 - 2^δ, CONVEX α = 2^-δ, β = 1 - 2^-δ; all exact in fp32
    lam = math.log(2)
    for d in range(8):
        a, b = st.blend_coeffs(st.I_VARIANT, st.EQ1, d, lam)
        assert (a, b) == (2.0 - 2.0**d, 0.0)
        a, b = st.blend_coeffs(st.I_VARIANT, st.CONVEX, d, lam)
        assert (a, b) == (2.0**-d, 1.0 - 2.0**-d)


def test_v_variant_uses_latest():
    for d in range(5):
        assert st.blend_coeffs(st.V_VARIANT, st.EQ1, d, 0.5) == (1.0, 0.0)


def test_coeffs_are_fp32_rounded():
    a, _ = st.blend_coeffs(st.I_VARIANT, st.EQ1, 3, 0.05)
    assert a == float(np.float32(2 - math.exp(0.15)))
    assert a != 2 - math.exp(0.15)

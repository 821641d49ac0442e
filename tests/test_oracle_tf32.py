"""Pins for oracle.tf32 (tf32 storage mode, DESIGN reading Z28; SURVEY Z13 "cvt.rna.tf32").

* `rna` == an independent integer definition of round-to-nearest-ties-away on the fp32 bit
  pattern (add half a tf32 ulp to the bits, clear the 13 low mantissa bits: the carry
  propagates into the exponent exactly as rounding up does), on 2M random fp32 patterns and
  on exact ties;
* closed forms: ties go away from zero, the bound |rna(x) - x| <= 2^-11 |x| for normals,
  tf32 values are fixed points, subnormal quantum 2^-136, overflow to inf;
* the tf32 replay lies within the tf32 rounding error of exact arithmetic and closer to it
  than the bf16 replay (so the rounding points run at 11 significant bits, not 8).
"""
import numpy as np
import pytest

import synthgen
from oracle import mlp, pipeline, staleness as st, tf32


def _bits_rna(x32: np.ndarray) -> np.ndarray:
    u = x32.view(np.uint32).astype(np.uint64)
    r = ((u + 0x1000) & 0xFFFFE000).astype(np.uint32)
    return r.view(np.float32).astype(np.float64)


def _random_f32(n, seed):
    rng = np.random.default_rng(seed)
    bits = rng.integers(0, 2**32, size=n, dtype=np.uint64).astype(np.uint32)
    x = bits.view(np.float32)
    return x[np.isfinite(x)]


def _ties_f32(n, seed):
    rng = np.random.default_rng(seed)
    hi = rng.integers(0, 2**19, size=n, dtype=np.uint64).astype(np.uint32)
    x = ((hi << np.uint32(13)) | np.uint32(0x1000)).view(np.float32)
    return x[np.isfinite(x)]


def test_rna_matches_bit_definition():
    for x in (_random_f32(2_000_000, 5), _ties_f32(300_000, 6)):
        ref = _bits_rna(x)
        got = tf32.rna(x.astype(np.float64))
        same = (ref == got) | (np.isnan(ref) & np.isnan(got))
        assert same.all(), x[~same][:5]


def test_rna_closed_forms():
    e = 2.0 ** -10                                  # tf32 ulp at 1
    assert tf32.rna(np.array([1 + e / 2]))[0] == 1 + e          # tie -> away from zero
    assert tf32.rna(np.array([-(1 + e / 2)]))[0] == -(1 + e)
    assert tf32.rna(np.array([1 + 3 * e / 2]))[0] == 1 + 2 * e  # tie, odd mantissa -> away (not even)
    assert tf32.rna(np.array([1 + e / 4]))[0] == 1.0
    assert tf32.rna(np.array([2 - e / 2]))[0] == 2.0            # carry into the exponent
    assert tf32.rna(np.array([2.0 ** -137]))[0] == 2.0 ** -136  # half a subnormal quantum
    assert tf32.rna(np.array([2.0 ** -138]))[0] == 0.0
    assert tf32.rna(np.array([(2 - 2.0 ** -11) * 2.0 ** 127]))[0] == np.inf
    assert tf32.rna(np.array([(2 - 2.0 ** -10) * 2.0 ** 127]))[0] == (2 - 2.0 ** -10) * 2.0 ** 127
    z = tf32.rna(np.array([0.0, -0.0, np.inf, -np.inf]))
    assert z[0] == 0 and np.signbit(z[1]) and z[2] == np.inf and z[3] == -np.inf


def test_rna_error_bound_and_fixed_points():
    rng = np.random.default_rng(7)
    x = rng.standard_normal(200_000) * 10.0 ** rng.integers(-20, 20, 200_000)
    r = tf32.rna(x)
    assert (np.abs(r - x) <= 2.0 ** -11 * np.abs(x)).all()
    assert np.array_equal(tf32.rna(r), r)
    # inputs, synthgen weights: exact in tf32 (8 significant bits / 24-bit mantissas are not)
    xs = synthgen.inputs(0, 0, 64, 32, synthgen.X_SIGNED).astype(np.float64)
    assert np.array_equal(tf32.rna(xs), xs)


def _run(dtype, exact=False):
    dims, bounds, m, b, M = [24, 20, 16, 10], [0, 1, 3], 2, 8, 6
    xs = [synthgen.inputs(3, j, m * b, dims[0], synthgen.X_SIGNED) for j in range(M)]
    ys = [synthgen.labels(3, j, m * b, dims[-1]) for j in range(M)]
    w0 = [synthgen.weights(3, l, dims[l + 1], dims[l]) for l in range(3)]
    b0 = [np.zeros(dims[l + 1], np.float32) for l in range(3)]
    cfg = pipeline.Config(dims, bounds, m, b, M, variant=st.I_VARIANT, blend=st.CONVEX, lam=0.3, lr=0.1,
                          momentum=0.9, exact=exact, dtype=dtype)
    return pipeline.run(cfg, xs, ys, w0, b0)


def test_tf32_replay_between_exact_and_bf16():
    ex, t, b = _run("bf16", exact=True), _run("tf32"), _run("bf16")
    assert [r.delta for r in t.trace] == [r.delta for r in ex.trace]
    et = [np.abs(t.weights[l] - ex.weights[l]).max() / np.abs(ex.weights[l]).max() for l in range(3)]
    eb = [np.abs(b.weights[l] - ex.weights[l]).max() / np.abs(ex.weights[l]).max() for l in range(3)]
    lt = np.abs(t.losses - ex.losses).max()
    lb = np.abs(b.losses - ex.losses).max()
    # 11 significant bits per stored value (|δ| <= 2^-11): the losses stay within 1e-4 of exact
    # arithmetic and ~8x closer than with bf16's 8 bits; every layer's weights closer than bf16's
    # (the first layer's update also sees ReLU-mask flips, discrete in both precisions)
    assert lt < 1e-4 and lt < lb / 4
    assert all(a < c for a, c in zip(et, eb)) and sum(et) < sum(eb) / 3 and max(et) < 1e-2


def test_precision_store_dispatch():
    x = np.array([1 + 2.0 ** -11, 1 + 2.0 ** -8])
    assert np.array_equal(mlp.Precision(dtype="tf32").store(x), tf32.rna(x))
    assert mlp.Precision(dtype="bf16").store(x)[0] == 1.0
    with pytest.raises(AssertionError):
        pipeline.run(pipeline.Config([4, 2], [0, 1], 1, 1, 1, dtype="fp8"), [np.zeros((1, 4))], [np.zeros(1, int)],
                     [np.zeros((2, 4), np.float32)], [np.zeros(2, np.float32)])

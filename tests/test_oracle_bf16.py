"""Pins for oracle.bf16 (reading Z13) against library routines and closed forms."""
import ml_dtypes
import numpy as np
import torch

from oracle import bf16


def _random_f32(n, seed):
    rng = np.random.default_rng(seed)
    bits = rng.integers(0, 2**32, size=n, dtype=np.uint64).astype(np.uint32)
    x = bits.view(np.float32)
    return x[np.isfinite(x)]


def _ties_f32(n, seed):
    # fp32 values whose low 16 bits are exactly 0x8000: halfway between two bf16 values
    rng = np.random.default_rng(seed)
    hi = rng.integers(0, 2**16, size=n, dtype=np.uint64).astype(np.uint32)
    bits = (hi << np.uint32(16)) | np.uint32(0x8000)
    x = bits.view(np.float32)
    return x[np.isfinite(x)]


def test_rne_matches_ml_dtypes_on_fp32_patterns():
    # fp32 -> bf16 is a single rounding in ml_dtypes: library pin, incl. exact ties
    for x in (_random_f32(2_000_000, 1), _ties_f32(200_000, 2)):
        ref = x.astype(ml_dtypes.bfloat16).astype(np.float64)
        got = bf16.rne(x.astype(np.float64))
        same = (ref == got) | (np.isnan(ref) & np.isnan(got))
        assert same.all()


def test_rne_matches_torch_bfloat16():
    x = _random_f32(500_000, 3)
    ref = torch.from_numpy(x).to(torch.bfloat16).to(torch.float64).numpy()
    assert np.array_equal(ref, bf16.rne(x.astype(np.float64)))


def test_rne_rounds_fp64_once():
    # 1 + 2^-8 + 2^-30 lies above the tie 1 + 2^-8: a single rounding gives 1 + 2^-7.
    # (Rounding through fp32 first would lose 2^-30, hit the tie and give 1.)
    assert bf16.rne(np.array([1 + 2**-8 + 2**-30]))[0] == 1 + 2**-7
    # exact tie rounds to even mantissa
    assert bf16.rne(np.array([1 + 2**-8]))[0] == 1.0
    assert bf16.rne(np.array([1 + 3 * 2**-8]))[0] == 1 + 2**-6


def test_rne_special_values():
    x = np.array([0.0, -0.0, np.inf, -np.inf, 3.397e38, 2.0**-133, 2.0**-134, 3 * 2.0**-135, 2.0**-126])
    got = bf16.rne(x)
    assert got[0] == 0 and got[1] == 0 and np.signbit(got[1])
    assert got[2] == np.inf and got[3] == -np.inf
    assert got[4] == np.inf                      # above (2 - 2^-8)·2^127 -> inf
    assert bf16.rne(np.array([3.395e38]))[0] == (2 - 2**-7) * 2.0**127
    assert got[5] == 2.0**-133                   # smallest bf16 subnormal
    assert got[6] == 0.0                         # tie to even (0)
    assert got[7] == 2.0**-133                   # 0.75 quantum -> 1 quantum
    assert got[8] == 2.0**-126
    assert np.isnan(bf16.rne(np.array([np.nan])))[0]


def test_bits_roundtrip():
    x = bf16.rne(np.linspace(-3, 3, 1001))
    assert np.array_equal(bf16.from_bits(bf16.to_bits(x)), x)

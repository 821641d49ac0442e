"""The fused wgrad->SGD epilogue performs exactly the fp32 operations of the separate update
kernel on the same fp32 gradient, so the two must agree BIT FOR BIT, for every tiling the
GEMM picks (single CTA / CTA pair, BN 64/128/256, 2 or 4 TMEM accumulator stages)."""
import numpy as np
import pytest

import synthgen
from oracle import staleness as ost
from pipeline_helpers import run_gpu

pytestmark = pytest.mark.gpu

SHAPES = [
    ([512, 4096, 16], 2, 64),       # wgrad 4096 x 512, K = 128: pair, BN = 128, 4 accumulators
    ([4096, 4096, 16], 4, 64),      # wgrad 4096 x 4096: pair, BN = 256
    ([1024, 512, 256, 16], 2, 32),  # small: single-CTA tiles
    ([784, 256, 10], 4, 8),         # config-1 shapes
    ([2048, 2048, 16], 8, 64),      # pair, BN = 256, several tiles per CTA
]


@pytest.mark.parametrize("dims,m,b", SHAPES)
@pytest.mark.parametrize("mu", [0.0, 0.9])
def test_fused_equals_separate_bitwise(gpu_lib, dims, m, b, mu):
    bounds = [0, len(dims) - 1]
    res = []
    for fuse in (0, 1):
        st, losses = run_gpu(dims, bounds, m, b, 3, ost.I_VARIANT, ost.EQ1, 0.05, 0.01, mu, kind=synthgen.X_SIGNED,
                             init="synthetic", fuse_update=fuse)
        res.append(([st[0].get_weights(k) for k in range(len(dims) - 1)], losses))
    for k in range(len(dims) - 1):
        for a, b_ in zip(res[0][0][k], res[1][0][k]):
            bad = np.argwhere(a != b_)
            assert bad.size == 0, (dims, k, bad[:5].tolist(), a.shape)
    np.testing.assert_array_equal(res[0][1], res[1][1])

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
    ([4096, 2560, 16], 4, 64),      # 160 tiles on 74 pairs: the last 12 split into 24 half tiles (split tail)
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


@pytest.mark.parametrize("MNK", [(4096, 4096, 2048), (512, 4096, 128), (1024, 520, 96), (4096, 256, 2048),
                                 (2560, 4096, 1024)])
@pytest.mark.parametrize("mu", [0.0, 0.9])
def test_raw_fused_kernel_matches_oracle_update(gpu_lib, MNK, mu):
    """tps_gemm_wgrad_sgd (the fused wgrad + SGD/momentum kernel alone) == oracle.mlp.sgd_update
    applied to the fp32 gradient of the same bf16 operands, within fp32 accumulation-order noise
    (relative to the update), and the bf16 version == bf16_rne(w) bit for bit."""
    import torch
    from oracle import bf16 as obf
    from oracle import mlp as omlp
    from paper_2509_23241_b200 import tps
    M, N, K = MNK
    g = torch.Generator().manual_seed(M + N + K)
    A = torch.randn(K, M, generator=g).to(torch.bfloat16)
    B = torch.randn(K, N, generator=g).to(torch.bfloat16)
    w0 = torch.randn(M, N, generator=g)
    v0 = torch.randn(M, N, generator=g) * 0.1 if mu else torch.zeros(M, N)
    lr, wd = 0.01, 1e-4
    w, v = w0.clone().cuda(), v0.clone().cuda()
    q = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    tps.gemm_wgrad_sgd(M, N, K, A.cuda(), M, B.cuda(), N, w, v, q, N, lr, mu, wd)
    torch.cuda.synchronize()
    gref = (A.double().T @ B.double()).numpy().astype(np.float32)       # fp32-rounded gradient
    wr, vr = omlp.sgd_update(w0.numpy(), v0.numpy(), gref, lr, mu, wd, False)
    wg = w.cpu().numpy()
    scale = np.abs(wr - w0.numpy()).max()
    assert np.abs(wg - wr).max() <= 1e-3 * scale + 1e-6 * np.abs(wr).max()
    if mu:
        assert np.abs(v.cpu().numpy() - vr).max() <= 1e-3 * np.abs(vr - v0.numpy()).max() + 1e-6 * np.abs(vr).max()
    np.testing.assert_array_equal(q.float().cpu().numpy(), obf.rne(wg.astype(np.float64)))


@pytest.mark.parametrize("MNK", [(16, 4096, 2048), (16, 784, 512), (200, 520, 256)])
def test_fused_update_reads_nothing_past_w(gpu_lib, MNK):
    """Tiles are 128 (or 256) rows and 32-column chunks wide: rows past M and columns past N of
    w / v must not be read (the head layer has M = 16).  w / v / version sit at the very END of a
    dedicated allocation (a tensor of >= 2 MiB gets its own cudaMalloc segment), so a read past
    them touches unmapped memory and faults; the update must still match the oracle's."""
    import torch
    from oracle import bf16 as obf
    from oracle import mlp as omlp
    from paper_2509_23241_b200 import tps
    M, N, K = MNK
    g = torch.Generator().manual_seed(7 + M)
    A = torch.randn(K, M, generator=g).to(torch.bfloat16)
    B = torch.randn(K, N, generator=g).to(torch.bfloat16)
    w0 = torch.randn(M, N, generator=g)
    v0 = torch.randn(M, N, generator=g) * 0.1

    def at_end(n, dtype):
        seg = (4 << 20) // torch.tensor([], dtype=dtype).element_size()
        buf = torch.zeros(max(seg, n), dtype=dtype, device="cuda")
        return buf[buf.numel() - n:].view(M, N)

    w, v, q = at_end(M * N, torch.float32), at_end(M * N, torch.float32), at_end(M * N, torch.bfloat16)
    w.copy_(w0.cuda())
    v.copy_(v0.cuda())
    lr, mu, wd = 0.01, 0.9, 1e-4
    tps.gemm_wgrad_sgd(M, N, K, A.cuda(), M, B.cuda(), N, w, v, q, N, lr, mu, wd)
    torch.cuda.synchronize()
    gref = (A.double().T @ B.double()).numpy().astype(np.float32)
    wr, vr = omlp.sgd_update(w0.numpy(), v0.numpy(), gref, lr, mu, wd, False)
    wg = w.cpu().numpy()
    assert np.abs(wg - wr).max() <= 1e-3 * np.abs(wr - w0.numpy()).max() + 1e-6 * np.abs(wr).max()
    np.testing.assert_array_equal(q.float().cpu().numpy(), obf.rne(wg.astype(np.float64)))

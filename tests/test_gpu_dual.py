"""The dual backward launch (include/tps.h tps_gemm_bwd_dual; rows a8 + a10): layer k's weight
gradient with the fused SGD/momentum update and layer k-1's input gradient in ONE persistent
kernel whose CTA pairs interleave tiles of both.

Checks: (1) raw kernel == the two separate kernels BIT FOR BIT where both use the same tiling
(the C5 shapes), and == the oracle's update / a float64 input gradient elsewhere (ragged
shapes, momentum on / off, mask and α); (2) unsuitable shapes report TPS_E_UNSUPPORTED;
(3) whole pipelines (multi-layer S = 1, multi-stage LOCAL with EQ1 α, V, the bias step on the
optimizer stream) produce bit-identical losses, parameters and momentum with the dual launch
on (TPS_DUAL=1) and off (the default: the two launches on two streams)."""
import os

import numpy as np
import pytest
import torch

import synthgen
from oracle import bf16 as obf
from oracle import mlp as omlp
from oracle import staleness as ost
from pipeline_helpers import run_gpu

pytestmark = pytest.mark.gpu


def operands(Mw, Nw, Kw, Md, Nd, Kd, mu, seed):
    g = torch.Generator().manual_seed(seed)
    A = torch.randn(Kw, Mw, generator=g).to(torch.bfloat16)          # G stored [K, M]
    B = torch.randn(Kw, Nw, generator=g).to(torch.bfloat16)          # X stored [K, N]
    w0 = torch.randn(Mw, Nw, generator=g)
    v0 = torch.randn(Mw, Nw, generator=g) * 0.1 if mu else torch.zeros(Mw, Nw)
    Ad = torch.randn(Md, Kd, generator=g).to(torch.bfloat16)         # G [M, K]
    Bd = (torch.randn(Kd, Nd, generator=g) * Kd ** -0.5).to(torch.bfloat16)   # W stored [K, N]
    mask = torch.randn(Md, Nd, generator=g).to(torch.bfloat16)
    return A, B, w0, v0, Ad, Bd, mask


def run_dual(Mw, Nw, Kw, Md, Nd, Kd, ops, lr, mu, wd, alpha, use_mask):
    from paper_2509_23241_b200 import tps
    A, B, w0, v0, Ad, Bd, mask = [t.cuda() for t in ops]
    w, v = w0.clone(), v0.clone()
    q = torch.empty(Mw, Nw, dtype=torch.bfloat16, device="cuda")
    out = torch.empty(Md, Nd, dtype=torch.bfloat16, device="cuda")
    tps.gemm_bwd_dual(Mw, Nw, Kw, A, Mw, B, Nw, w, v, q, Nw, lr, mu, wd, Md, Nd, Kd, Ad, Kd, Bd, Nd, out, Nd,
                      alpha, mask if use_mask else None, Nd if use_mask else 0)
    torch.cuda.synchronize()
    return w.cpu(), v.cpu(), q.cpu(), out.cpu()


def run_separate(Mw, Nw, Kw, Md, Nd, Kd, ops, lr, mu, wd, alpha, use_mask):
    from paper_2509_23241_b200 import tps
    A, B, w0, v0, Ad, Bd, mask = [t.cuda() for t in ops]
    w, v = w0.clone(), v0.clone()
    q = torch.empty(Mw, Nw, dtype=torch.bfloat16, device="cuda")
    out = torch.empty(Md, Nd, dtype=torch.bfloat16, device="cuda")
    tps.gemm_wgrad_sgd(Mw, Nw, Kw, A, Mw, B, Nw, w, v, q, Nw, lr, mu, wd)
    tps.gemm(1, Md, Nd, Kd, Ad, Kd, Bd, Nd, out, Nd, 0, None, 0, alpha, 0.0, mask if use_mask else None,
             Nd if use_mask else 0)
    torch.cuda.synchronize()
    return w.cpu(), v.cpu(), q.cpu(), out.cpu()


@pytest.mark.parametrize("mu", [0.0, 0.9])
def test_dual_equals_separate_bitwise_c5(gpu_lib, mu):
    # C5 backward of one 4096-wide layer pair at B = 2048: both halves on 256 x 256 CTA-pair tiles
    shp = (4096, 4096, 2048, 2048, 4096, 4096)
    ops = operands(*shp, mu, 11)
    a = run_dual(*shp, ops, 0.01, mu, 1e-4, 0.8, True)
    b = run_separate(*shp, ops, 0.01, mu, 1e-4, 0.8, True)
    for x, y, name in zip(a, b, ("w", "v", "ver", "dX")):
        assert torch.equal(x, y), name


@pytest.mark.parametrize("shp", [(4096, 4096, 2048, 2048, 4096, 4096), (1000, 1016, 300, 300, 1000, 1000),
                                 (512, 2048, 256, 256, 512, 512), (2048, 256, 1024, 1024, 2048, 2048)])
@pytest.mark.parametrize("mu", [0.0, 0.9])
def test_dual_matches_oracle(gpu_lib, shp, mu):
    Mw, Nw, Kw, Md, Nd, Kd = shp
    alpha, lr, wd = 0.7, 0.01, 1e-4
    ops = operands(*shp, mu, sum(shp))
    w, v, q, out = run_dual(*shp, ops, lr, mu, wd, alpha, True)
    A, B, w0, v0, Ad, Bd, mask = ops
    # weight half: oracle update of the fp32-rounded gradient (as test_gpu_fused_update)
    gref = (A.double().T @ B.double()).numpy().astype(np.float32)
    wr, vr = omlp.sgd_update(w0.numpy(), v0.numpy(), gref, lr, mu, wd, False)
    wg = w.numpy()
    scale = np.abs(wr - w0.numpy()).max()
    assert np.abs(wg - wr).max() <= 1e-3 * scale + 1e-6 * np.abs(wr).max()
    if mu:
        assert np.abs(v.numpy() - vr).max() <= 1e-3 * np.abs(vr - v0.numpy()).max() + 1e-6 * np.abs(vr).max()
    np.testing.assert_array_equal(q.float().numpy(), obf.rne(wg.astype(np.float64)))
    # input half: bf16(α·G·W) where mask > 0, else 0; fp32 accumulation vs float64: one bf16 ulp
    ref = alpha * (Ad.double() @ Bd.double())
    ref = torch.where(mask.double() > 0, ref, torch.zeros_like(ref)).numpy()
    got = out.double().numpy()
    assert np.all((got == 0) == (ref == 0))
    assert np.abs(got - ref).max() <= 2.0 ** -7 * np.abs(ref).max()
    assert np.all(np.abs(got - ref) <= 2.0 ** -8 * np.abs(ref) + 1e-3 * np.abs(ref).max() * 2.0 ** -8)


def test_dual_unsupported_shapes(gpu_lib):
    from paper_2509_23241_b200 import tps
    shp = (128, 512, 64, 64, 512, 128)      # fewer than 256 rows
    ops = [t.cuda() for t in operands(*shp, 0.0, 1)]
    A, B, w0, v0, Ad, Bd, mask = ops
    q = torch.empty(128, 512, dtype=torch.bfloat16, device="cuda")
    out = torch.empty(64, 512, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(tps.TpsError) as ei:
        tps.gemm_bwd_dual(128, 512, 64, A, 128, B, 512, w0, v0, q, 512, 0.1, 0.0, 0.0, 64, 512, 128, Ad, 128, Bd, 512,
                          out, 512)
    assert ei.value.status == 10


def both(dims, bounds, m, b, M, variant, blend, mu):
    res = []
    for dual in ("1", "0"):
        os.environ["TPS_DUAL"] = dual
        try:
            st, losses = run_gpu(dims, bounds, m, b, M, variant, blend, 0.2, 0.01, mu, wd=1e-4, init="synthetic",
                                 kind=synthgen.X_SIGNED)
        finally:
            os.environ.pop("TPS_DUAL", None)
        res.append((losses, [h.get_weights(k) for h in st for k in range(len(h.layers))]))
        for h in st:
            h.close()
    return res


@pytest.mark.parametrize("dims,bounds,m,b,variant,blend,mu", [
    ([4096, 4096, 4096, 4096, 10], [0, 4], 4, 512, ost.I_VARIANT, ost.EQ1, 0.9),     # C5-like, S = 1
    ([1024] * 6 + [10], [0, 2, 4, 6], 4, 64, ost.I_VARIANT, ost.EQ1, 0.9),         # 3 stages, EQ1 α on dgrad
    ([1024] * 6 + [10], [0, 3, 6], 2, 128, ost.V_VARIANT, ost.EQ1, 0.0),           # V, no momentum
    ([2048, 1536, 1024, 512, 10], [0, 4], 2, 256, ost.I_VARIANT, ost.EQ1, 0.9),    # narrowing widths
])
def test_pipeline_dual_on_equals_off_bitwise(gpu_lib, dims, bounds, m, b, variant, blend, mu):
    (la, wa), (lb, wb) = both(dims, bounds, m, b, 4, variant, blend, mu)
    np.testing.assert_array_equal(la, lb)
    assert len(wa) == len(wb)
    for x, y in zip(wa, wb):
        for p_, q_ in zip(x, y):
            np.testing.assert_array_equal(p_, q_)

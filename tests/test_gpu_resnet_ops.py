"""ResNet op kernels (C ABI tps_im2col / tps_col2im / tps_bn_forward / tps_bn_backward /
tps_pool_op) against oracle/resnet.py on identical bf16 inputs.

Bars: gathers (im2col, max-pool forward, the residual gradient) bit-exact; everything that
sums or divides within the rounding of its bf16 output (2^-7 relative) plus, where the
result is a cancelling sum (BN dx), 1e-5 of the tensor's max; statistics and parameter
gradients (fp32 outputs of fp64 sums) within 1e-5 relative.
"""
import numpy as np
import pytest
import torch

from oracle import bf16, resnet

pytestmark = pytest.mark.gpu


def bf(a):
    """fp64 array -> (bf16-rounded fp64 values, cuda bf16 tensor holding them)."""
    r = bf16.rne(np.asarray(a, np.float64))
    return r, torch.from_numpy(r.astype(np.float32)).to(torch.bfloat16).cuda()


def host(t):
    return t.float().cpu().numpy().astype(np.float64)


def close_bf16(got, ref, atol=0.0):
    err = np.abs(got - ref)
    bound = 2.0 ** -7 * np.abs(ref) + atol
    assert (err <= bound).all(), f"max excess {float((err - bound).max()):.3e}"


@pytest.mark.parametrize("k,s,p,C", [(7, 2, 3, 3), (3, 2, 1, 16), (1, 2, 0, 16), (3, 1, 1, 8), (3, 2, 1, 64), (1, 2, 0, 68)])
def test_im2col_col2im(gpu_lib, k, s, p, C):
    from paper_2509_23241_b200 import tps
    rng = np.random.default_rng(k * 10 + s)
    N, H, W = 2, 9, 11
    X, Xd = bf(rng.standard_normal((N, H, W, C)))
    cols, Ho, Wo = resnet.im2col(X, k, s, p)
    ldp = -(-k * k * C // 16) * 16
    P = torch.full((N * Ho * Wo, ldp), 7.0, dtype=torch.bfloat16, device="cuda")
    tps.im2col(Xd, P, N, H, W, C, k, s, p, ldp)
    torch.cuda.synchronize()
    got = host(P)
    assert np.array_equal(got[:, :k * k * C], cols)
    assert not got[:, k * k * C:].any()
    dP = rng.standard_normal((N * Ho * Wo, ldp)).astype(np.float32)
    ref = resnet.col2im(dP[:, :k * k * C].astype(np.float64), (N, H, W, C), k, s, p)
    dX = torch.empty(N, H, W, C, dtype=torch.bfloat16, device="cuda")
    dPd = torch.from_numpy(dP).cuda()
    tps.col2im(dPd, dX, None, N, H, W, C, k, s, p, ldp)
    A, Ad = bf(rng.standard_normal((N, H, W, C)))
    dX2 = Ad.clone()
    tps.col2im(dPd, dX2, dX2, N, H, W, C, k, s, p, ldp)     # accumulate in place
    torch.cuda.synchronize()
    close_bf16(host(dX), ref, 1e-6)
    close_bf16(host(dX2), ref + A, 1e-6)


@pytest.mark.parametrize("N,H,W,C", [(2, 20, 16, 3), (3, 13, 24, 3), (1, 9, 8, 8)])
def test_im2col_stem_vector_fill(gpu_lib, N, H, W, C):
    """The 7x7/2/3 stem patches with W·C % 8 == 0 (16-byte-staged input rows, as at 224 x 224 x 3):
    bit-exact against the oracle's im2col, zero pad columns."""
    from paper_2509_23241_b200 import tps
    k, s, p = 7, 2, 3
    rng = np.random.default_rng(N * 100 + W)
    X, Xd = bf(rng.standard_normal((N, H, W, C)))
    cols, Ho, Wo = resnet.im2col(X, k, s, p)
    ldp = -(-k * k * C // 16) * 16
    P = torch.full((N * Ho * Wo, ldp), 7.0, dtype=torch.bfloat16, device="cuda")
    tps.im2col(Xd, P, N, H, W, C, k, s, p, ldp)
    torch.cuda.synchronize()
    got = host(P)
    assert np.array_equal(got[:, :k * k * C], cols)
    assert not got[:, k * k * C:].any()


def test_maxpool3_and_avgpool(gpu_lib):
    from paper_2509_23241_b200 import tps
    rng = np.random.default_rng(3)
    N, H, W, C = 2, 9, 8, 16
    X, Xd = bf(rng.integers(-4, 5, (N, H, W, C)) / 4.0)          # many ties: first maximum wins
    Ho, Wo = (H - 1) // 2 + 1, (W - 1) // 2 + 1
    Y = torch.empty(N, Ho, Wo, C, dtype=torch.bfloat16, device="cuda")
    tps.pool_op(0, Xd, None, Y, N, H, W, C)
    dY, dYd = bf(rng.standard_normal((N, Ho, Wo, C)))
    dX = torch.empty_like(Xd)
    tps.pool_op(1, Xd, dYd, dX, N, H, W, C)
    A = torch.empty(N, C, dtype=torch.bfloat16, device="cuda")
    tps.pool_op(2, Xd, None, A, N, H, W, C)
    g, gd = bf(rng.standard_normal((N, C)))
    dA = torch.empty_like(Xd)
    tps.pool_op(3, None, gd, dA, N, H, W, C)
    torch.cuda.synchronize()
    Y2 = torch.empty_like(Y)
    idx = torch.empty(N, Ho, Wo, C, dtype=torch.uint8, device="cuda")
    tps.pool_op(4, Xd, idx, Y2, N, H, W, C)                      # recorded first-max taps
    dX2 = torch.empty_like(Xd)
    tps.pool_op(5, idx, dYd, dX2, N, H, W, C)
    torch.cuda.synchronize()
    assert np.array_equal(host(Y), resnet.maxpool3_forward(X))
    assert np.array_equal(host(Y2), host(Y))
    assert np.array_equal(host(dX2), host(dX))
    close_bf16(host(dX), resnet.maxpool3_backward(X, dY))
    close_bf16(host(A), resnet.avgpool_forward(X))
    close_bf16(host(dA), resnet.avgpool_backward(X.shape, g))


@pytest.mark.parametrize("relu,res,C", [(True, False, 40), (True, True, 40), (False, False, 40), (True, True, 64),
                                        (False, False, 256), (True, False, 24)])
def test_batchnorm_forward_backward(gpu_lib, relu, res, C):
    """C % 8 == 0 takes the 16-byte vector kernels, C = 40 / 24 with odd channel groups too."""
    from paper_2509_23241_b200 import tps
    rng = np.random.default_rng(7 + C)
    segs, b, H, W = 3, 4, 5, 6
    rows = b * H * W
    X, Xd = bf(1.5 + 2.0 * rng.standard_normal((segs * b, H, W, C)))
    R, Rd = bf(rng.standard_normal((segs * b, H, W, C)))
    gam = (1.0 + 0.3 * rng.standard_normal(C)).astype(np.float32)
    bet = (0.2 * rng.standard_normal(C)).astype(np.float32)
    gam_l = (gam + 0.05 * rng.standard_normal(C)).astype(np.float32)
    a, bb = np.float32(0.8), np.float32(0.2)
    cu = lambda v: torch.from_numpy(np.ascontiguousarray(v)).cuda()
    Y = torch.empty_like(Xd)
    mean = torch.empty(segs, C, device="cuda")
    inv = torch.empty(segs, C, device="cuda")
    tps.bn_forward(Xd, Rd if res else None, Y, cu(gam), cu(bet), mean, inv, segs, rows, C, int(relu))
    dY, dYd = bf(rng.standard_normal((segs * b, H, W, C)))
    dX = torch.empty_like(Xd)
    dR = torch.empty_like(Xd)
    dg = torch.empty(C, device="cuda")
    db = torch.empty(C, device="cuda")
    tps.bn_backward(dYd, Y, Xd, mean, inv, cu(gam), cu(gam_l), float(a), float(bb), segs, rows, C, int(relu), dX,
                    dR if res else None, dg, db)
    torch.cuda.synchronize()
    y_ref = np.empty_like(X)
    mus, invs = [], []
    for s_ in range(segs):
        sl = slice(s_ * b, (s_ + 1) * b)
        z, mu, iv = resnet.bn_forward(X[sl], gam.astype(np.float64), bet.astype(np.float64))
        if res:
            z = z + R[sl]
        y_ref[sl] = np.maximum(z, 0.0) if relu else z
        mus.append(mu)
        invs.append(iv)
    np.testing.assert_allclose(mean.cpu().numpy(), np.stack(mus), rtol=1e-6, atol=1e-7)
    np.testing.assert_allclose(inv.cpu().numpy(), np.stack(invs), rtol=1e-6)
    y_got = host(Y)
    close_bf16(y_got, y_ref, 1e-6)
    # backward from the GPU's own forward output (the mask), fp64 reference
    g_res = a.astype(np.float64) * gam + bb.astype(np.float64) * gam_l
    dy = dY * (y_got > 0) if relu else dY
    dx_ref = np.empty_like(X)
    dg_ref = np.zeros(C)
    db_ref = np.zeros(C)
    for s_ in range(segs):
        sl = slice(s_ * b, (s_ + 1) * b)
        dxa, dga, dba = resnet.bn_backward(dy[sl], X[sl], g_res, mus[s_], invs[s_])
        dx_ref[sl] = dxa
        dg_ref += dga
        db_ref += dba
    close_bf16(host(dX), dx_ref, 1e-5 * np.abs(dx_ref).max())
    np.testing.assert_allclose(dg.cpu().numpy(), dg_ref, rtol=1e-5, atol=1e-5 * np.abs(dg_ref).max())
    np.testing.assert_allclose(db.cpu().numpy(), db_ref, rtol=1e-5, atol=1e-5 * np.abs(db_ref).max())
    if res:
        assert np.array_equal(host(dR), dy)

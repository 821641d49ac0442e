"""ResNet-50 (BASELINE.json configs[3]) op-level parity at EVERY distinct layer shape of the
network, through the same kernels and the same code paths the pipeline runs for that shape
(runtime.cpp init_graph's conv_mode rule), against oracle/resnet.py on identical bf16 inputs.

Paths per conv shape (k, stride, pad, Ci, Co, H):
  * 1x1 / stride 1      plain GEMMs (tps_gemm fwd / dgrad / wgrad, and the blended dgrad);
  * 3x3 / stride 1      implicit GEMMs on TMA im2col-mode loads (tps_conv2d_gemm 0/1/2/3);
  * strided (3x3/2, 1x1/2 downsample)  implicit fwd / wgrad, input gradient as a patch-gradient
                        GEMM (fp32) + col2im (tps_gemm mode 1/3 + tps_col2im);
  * the 7x7/2 stem      explicit patches (tps_im2col) + GEMMs; no input gradient (layer 0).
Batch norm forward/backward (per-segment statistics, residual, ReLU, blended γ) at every
(C, H) of the network, the 3x3/2 max pool and the global average pool at their shapes, and
the 2048 -> 1000 head.

Bounds (derived from the arithmetic, no fitted constants):
  * a bf16 output is the fp32 accumulator rounded once: |got - ref| <= 2^-7·|ref| + 2^-16·S,
    S = Σ|a·b| over the contraction (the fp32 accumulation error is ~2^-24·sqrt(K)·S, far
    below 2^-16·S for K <= 2^14);
  * an fp32 output: |got - ref| <= 2^-16·S;
  * a blended operand is rounded to bf16 per element (relative <= 2^-8, independent), which
    adds a random error of standard deviation <= 2^-8·sqrt(Σ(a·w)²): 4 sigma of it is allowed.
A transposed or flipped filter, a wrong tap offset, a dropped K block or a wrong α/β moves
elements by O(|ref|) and fails.
"""
import math

import numpy as np
import pytest
import torch

from oracle import bf16, graph as ograph, resnet

pytestmark = pytest.mark.gpu

RNG = np.random.default_rng(2509)


def bfd(a):
    """fp64 array -> (bf16-rounded fp64 values, cuda bf16 tensor holding them)."""
    r = bf16.rne(np.asarray(a, np.float64))
    return r, torch.from_numpy(r.astype(np.float32)).to(torch.bfloat16).cuda().contiguous()


def host(t):
    return t.float().cpu().numpy().astype(np.float64)


def assert_within(got, ref, bound, what):
    err = np.abs(got - ref)
    bad = err > bound
    assert not bad.any(), (f"{what}: {int(bad.sum())} / {bad.size} elements over the bound, "
                           f"worst excess {float((err - bound).max()):.3e} (max |ref| {float(np.abs(ref).max()):.3e})")


def pad16(x):
    return -(-x // 16) * 16


def conv_shapes(H=224):
    layers, _ = ograph.resnet_layers(H=H)
    seen, out = set(), []
    for sp in layers:
        if sp["kind"] != "conv":
            continue
        key = (sp["k"], sp["s"], sp["p"], sp["cin"], sp["cout"], sp["h"])
        if key not in seen:
            seen.add(key)
            out.append(key)
    return out


def conv_mode(k, s, p, ci, co):
    """runtime.cpp init_graph: 0 plain GEMM, 1 implicit 3x3/1, 3 strided implicit, 2 patches."""
    if k == 1 and s == 1 and p == 0 and ci % 16 == 0:
        return 0
    if k == 3 and s == 1 and p == 1 and ci % 64 == 0 and co % 64 == 0:
        return 1
    if ci % 64 == 0 and co % 64 == 0:
        return 3
    return 2


SHAPES = conv_shapes()
# the same network at 64x64 inputs (the reduced-resolution whole-net test): spatial sizes down to
# 2x2, where the implicit-GEMM tiles span several images
SHAPES_64 = [sh for sh in conv_shapes(64) if sh not in SHAPES]


def test_resnet50_has_the_expected_distinct_conv_shapes():
    # stem; per stage: 1x1 reduce (in from the previous width), 3x3, 1x1 expand, downsample,
    # 1x1 reduce from 4·width, and the strided 3x3 / 1x1 of stages 2-4
    assert len(SHAPES) == 23
    assert {conv_mode(*s[:5]) for s in SHAPES} == {0, 1, 2, 3}


@pytest.mark.parametrize("shape", SHAPES + SHAPES_64, ids=lambda s: "k%d_s%d_p%d_%dto%d_h%d" % s)
def test_conv_fwd_dgrad_wgrad_at_resnet50_shape(gpu_lib, shape):
    from paper_2509_23241_b200 import tps
    k, s, p, ci, co, H = shape
    mode = conv_mode(k, s, p, ci, co)
    Ho = (H + 2 * p - k) // s + 1
    N = max(2, math.ceil(320 / (Ho * Ho)))            # several 128-row tiles with a ragged tail
    X, Xd = bfd(RNG.standard_normal((N, H, H, ci)))
    Wt, Wd = bfd(RNG.standard_normal((co, k, k, ci)) / math.sqrt(k * k * ci))
    dY, dYd = bfd(RNG.standard_normal((N, Ho, Ho, co)))
    M, Kc = N * Ho * Ho, k * k * ci
    W2 = Wt.reshape(co, Kc)

    # ---- forward
    ref = resnet.conv_forward(X, Wt, s, p).reshape(M, co)
    S = resnet.conv_forward(np.abs(X), np.abs(Wt), s, p).reshape(M, co)
    out = torch.empty(M, co, dtype=torch.bfloat16, device="cuda")
    if mode == 0:
        tps.gemm(0, M, co, ci, Xd, ci, Wd, ci, out, co)
    elif mode in (1, 3):
        tps.conv2d_gemm(0, N, H, H, ci, co, k, s, p, Xd, Wd, out)
    else:
        Kp = pad16(Kc)
        P = torch.empty(M, Kp, dtype=torch.bfloat16, device="cuda")
        tps.im2col(Xd, P, N, H, H, ci, k, s, p, Kp)
        Wp = torch.zeros(co, Kp, dtype=torch.bfloat16, device="cuda")
        Wp[:, :Kc] = Wd.reshape(co, Kc)
        tps.gemm(0, M, co, Kp, P, Kp, Wp, Kp, out, co)
    torch.cuda.synchronize()
    assert_within(host(out), ref, 2.0 ** -7 * np.abs(ref) + 2.0 ** -16 * S, "forward")

    # ---- weight gradient (fp32 out)
    refw = resnet.conv_wgrad(dY, X, k, s, p).reshape(co, Kc)
    Sw = resnet.conv_wgrad(np.abs(dY), np.abs(X), k, s, p).reshape(co, Kc)
    if mode == 0:
        dW = torch.empty(co, ci, device="cuda")
        tps.gemm(2, co, ci, M, dYd, co, Xd, ci, dW, ci, out_f32=1)
    elif mode in (1, 3):
        dW = torch.empty(co, Kc, device="cuda")
        tps.conv2d_gemm(2, N, H, H, ci, co, k, s, p, dYd, Xd, dW, out_f32=1)
    else:
        Kp = pad16(Kc)
        dWp = torch.empty(co, Kp, device="cuda")
        tps.gemm(2, co, Kp, M, dYd, co, P, Kp, dWp, Kp, out_f32=1)
        assert not dWp[:, Kc:].any()
        dW = dWp[:, :Kc]
    torch.cuda.synchronize()
    assert_within(dW.cpu().numpy().astype(np.float64), refw, 2.0 ** -16 * Sw, "weight gradient")

    if mode == 2:
        return   # the stem is the network's first layer: no input gradient (Z12)

    # ---- input gradient: plain (α = 1), EQ1 (α in the epilogue) and the blended operand
    Wl, Wld = bfd(Wt + 0.05 * RNG.standard_normal(Wt.shape) / math.sqrt(Kc))
    for a, b, blend in ((1.0, 0.0, False), (0.8, 0.0, False), (0.7, 0.3, True)):
        Wres = np.float64(np.float32(a)) * Wt + np.float64(np.float32(b)) * Wl
        refd = resnet.conv_dgrad(dY, Wres, X.shape, s, p)
        Sd = resnet.conv_dgrad(np.abs(dY), np.abs(Wres), X.shape, s, p)
        sig = np.sqrt(resnet.conv_dgrad(dY ** 2, Wres ** 2, X.shape, s, p)) if blend else 0.0
        dX = torch.empty(N, H, H, ci, dtype=torch.bfloat16, device="cuda")
        if mode == 0:
            if blend:
                tps.gemm(3, M, ci, co, dYd, co, Wd, ci, dX, ci, alpha=a, beta=b, B2=Wld)
            else:
                tps.gemm(1, M, ci, co, dYd, co, Wd, ci, dX, ci, alpha=a)
        elif mode == 1:
            if blend:
                tps.conv2d_gemm(3, N, H, H, ci, co, 3, 1, 1, dYd, Wd, dX, alpha=a, beta=b, W2=Wld)
            else:
                tps.conv2d_gemm(1, N, H, H, ci, co, 3, 1, 1, dYd, Wd, dX, alpha=a)
        else:
            dP = torch.empty(M, Kc, device="cuda")
            if blend:
                tps.gemm(3, M, Kc, co, dYd, co, Wd, Kc, dP, Kc, out_f32=1, alpha=a, beta=b, B2=Wld)
            else:
                tps.gemm(1, M, Kc, co, dYd, co, Wd, Kc, dP, Kc, out_f32=1, alpha=a)
            tps.col2im(dP, dX, None, N, H, H, ci, k, s, p, Kc)
        torch.cuda.synchronize()
        assert_within(host(dX), refd, 2.0 ** -7 * np.abs(refd) + 2.0 ** -16 * Sd + 4 * 2.0 ** -8 * sig,
                      f"input gradient α={a} β={b}")


def bn_shapes():
    layers, _ = ograph.resnet_layers()
    seen, out = set(), []
    for sp in layers:
        if sp["kind"] == "bn":
            key = (sp["c"], sp["h"], bool(sp.get("res") is not None), bool(sp["relu"]))
            if key not in seen:
                seen.add(key)
                out.append(key)
    return out


@pytest.mark.parametrize("shape", bn_shapes(), ids=lambda s: "c%d_h%d_res%d_relu%d" % s)
def test_batchnorm_at_resnet50_shape(gpu_lib, shape):
    from paper_2509_23241_b200 import tps
    C, H, res, relu = shape
    segs = 2
    b = max(1, math.ceil(64 / (H * H)))                 # >= 64 rows per segment statistic
    rows = b * H * H
    X, Xd = bfd(0.5 + 1.5 * RNG.standard_normal((segs * b, H, H, C)))
    R, Rd = bfd(RNG.standard_normal((segs * b, H, H, C)))
    gam = (1.0 + 0.2 * RNG.standard_normal(C)).astype(np.float32)
    bet = (0.1 * RNG.standard_normal(C)).astype(np.float32)
    gam_l = (gam + 0.02 * RNG.standard_normal(C)).astype(np.float32)
    a, bb = np.float32(0.9), np.float32(0.1)
    cu = lambda v: torch.from_numpy(np.ascontiguousarray(v)).cuda()
    Y = torch.empty_like(Xd)
    mean = torch.empty(segs, C, device="cuda")
    inv = torch.empty(segs, C, device="cuda")
    tps.bn_forward(Xd, Rd if res else None, Y, cu(gam), cu(bet), mean, inv, segs, rows, C, int(relu))
    dY, dYd = bfd(RNG.standard_normal((segs * b, H, H, C)))
    dX, dR = torch.empty_like(Xd), torch.empty_like(Xd)
    dg, db = torch.empty(C, device="cuda"), torch.empty(C, device="cuda")
    tps.bn_backward(dYd, Y, Xd, mean, inv, cu(gam), cu(gam_l), float(a), float(bb), segs, rows, C, int(relu), dX,
                    dR if res else None, dg, db)
    torch.cuda.synchronize()
    y_ref = np.empty_like(X)
    mus, invs = [], []
    for s_ in range(segs):
        sl = slice(s_ * b, (s_ + 1) * b)
        z, mu, iv = resnet.bn_forward(X[sl], gam.astype(np.float64), bet.astype(np.float64))
        z = z + R[sl] if res else z
        y_ref[sl] = np.maximum(z, 0.0) if relu else z
        mus.append(mu)
        invs.append(iv)
    np.testing.assert_allclose(mean.cpu().numpy(), np.stack(mus), rtol=1e-6, atol=1e-7)
    np.testing.assert_allclose(inv.cpu().numpy(), np.stack(invs), rtol=1e-6)
    y_got = host(Y)
    assert_within(y_got, y_ref, 2.0 ** -7 * np.abs(y_ref) + 1e-6, "bn forward")
    g_res = a.astype(np.float64) * gam + bb.astype(np.float64) * gam_l
    dy = dY * (y_got > 0) if relu else dY
    dx_ref = np.empty_like(X)
    dg_ref, db_ref = np.zeros(C), np.zeros(C)
    for s_ in range(segs):
        sl = slice(s_ * b, (s_ + 1) * b)
        dxa, dga, dba = resnet.bn_backward(dy[sl], X[sl], g_res, mus[s_], invs[s_])
        dx_ref[sl] = dxa
        dg_ref += dga
        db_ref += dba
    assert_within(host(dX), dx_ref, 2.0 ** -7 * np.abs(dx_ref) + 1e-5 * np.abs(dx_ref).max(), "bn dx")
    np.testing.assert_allclose(dg.cpu().numpy(), dg_ref, rtol=1e-5, atol=1e-5 * np.abs(dg_ref).max())
    np.testing.assert_allclose(db.cpu().numpy(), db_ref, rtol=1e-5, atol=1e-5 * np.abs(db_ref).max())
    if res:
        assert np.array_equal(host(dR), dy)


def test_pools_and_head_at_resnet50_shapes(gpu_lib):
    from paper_2509_23241_b200 import tps
    # stem max pool 112x112x64 -> 56x56x64 (recorded taps, as the pipeline runs it)
    N, H, C = 2, 112, 64
    X, Xd = bfd(np.round(RNG.standard_normal((N, H, H, C)) * 4) / 4)     # ties: first maximum wins
    Ho = (H - 1) // 2 + 1
    Y = torch.empty(N, Ho, Ho, C, dtype=torch.bfloat16, device="cuda")
    idx = torch.empty(N, Ho, Ho, C, dtype=torch.uint8, device="cuda")
    tps.pool_op(4, Xd, idx, Y, N, H, H, C)
    dY, dYd = bfd(RNG.standard_normal((N, Ho, Ho, C)))
    dX = torch.empty_like(Xd)
    tps.pool_op(5, idx, dYd, dX, N, H, H, C)
    torch.cuda.synchronize()
    assert np.array_equal(host(Y), resnet.maxpool3_forward(X))
    ref = resnet.maxpool3_backward(X, dY)
    assert_within(host(dX), ref, 2.0 ** -7 * np.abs(ref), "maxpool backward")
    # global average pool 7x7x2048
    N, H, C = 4, 7, 2048
    X, Xd = bfd(RNG.standard_normal((N, H, H, C)))
    A = torch.empty(N, C, dtype=torch.bfloat16, device="cuda")
    tps.pool_op(2, Xd, None, A, N, H, H, C)
    g, gd = bfd(RNG.standard_normal((N, C)))
    dA = torch.empty_like(Xd)
    tps.pool_op(3, None, gd, dA, N, H, H, C)
    torch.cuda.synchronize()
    ref = resnet.avgpool_forward(X)
    assert_within(host(A), ref, 2.0 ** -7 * np.abs(ref) + 2.0 ** -16 * resnet.avgpool_forward(np.abs(X)), "avgpool")
    ref = resnet.avgpool_backward(X.shape, g)
    assert_within(host(dA), ref, 2.0 ** -7 * np.abs(ref), "avgpool backward")
    # head 2048 -> 1000 (Np = 1008): logits fp32 + bias, input gradient, weight gradient
    B, K, Co, Np = 96, 2048, 1000, 1008
    Xh, Xhd = bfd(np.abs(RNG.standard_normal((B, K))))
    Wh = np.zeros((Np, K))
    Wh[:Co] = RNG.standard_normal((Co, K)) / math.sqrt(K)
    Wh, Whd = bfd(Wh)
    bias = np.zeros(Np, np.float32)
    bias[:Co] = 0.1 * RNG.standard_normal(Co)
    Z = torch.empty(B, Np, device="cuda")
    tps.gemm(0, B, Np, K, Xhd, K, Whd, K, Z, Np, out_f32=1, bias=torch.from_numpy(bias).cuda())
    G = np.zeros((B, Np))
    G[:, :Co] = RNG.standard_normal((B, Co)) / B
    G, Gd = bfd(G)
    dXh = torch.empty(B, K, dtype=torch.bfloat16, device="cuda")
    tps.gemm(1, B, K, Np, Gd, Np, Whd, K, dXh, K)
    dWh = torch.empty(Np, K, device="cuda")
    tps.gemm(2, Np, K, B, Gd, Np, Xhd, K, dWh, K, out_f32=1)
    torch.cuda.synchronize()
    ref = Xh @ Wh.T + bias.astype(np.float64)
    assert_within(Z.cpu().numpy().astype(np.float64), ref, 2.0 ** -16 * (np.abs(Xh) @ np.abs(Wh).T) + 1e-7, "head")
    ref = G @ Wh
    assert_within(host(dXh), ref, 2.0 ** -7 * np.abs(ref) + 2.0 ** -16 * (np.abs(G) @ np.abs(Wh)), "head dgrad")
    ref = G.T @ Xh
    assert_within(dWh.cpu().numpy().astype(np.float64), ref, 2.0 ** -16 * (np.abs(G).T @ np.abs(Xh)), "head wgrad")

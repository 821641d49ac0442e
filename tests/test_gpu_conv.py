"""3x3 convolutions as implicit GEMMs on tcgen05 (4-D TMA im2col boxes) and the image-net
pipeline (VGG-style, configs[2]) against torch fp64 and the CPU oracle."""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

import synthgen
from oracle import staleness as ost
from paper_2509_23241_b200 import tps
from pipeline_helpers import expand_gpu_trace, layer_rel_err, oracle_trace, run_gpu, run_oracle, weight_rel_err

pytestmark = pytest.mark.gpu

SHAPES = [  # N, H, W, Ci, Co — VGG-16 / CIFAR spatial sizes, several tiles, 1..8 images per 128-pixel box
    (2, 32, 32, 64, 64), (4, 16, 16, 128, 128), (16, 8, 8, 64, 128), (32, 4, 4, 256, 64), (64, 2, 2, 128, 256),
]


def nhwc_conv_ref(X, Wt, b=None):
    y = F.conv2d(X.double().permute(0, 3, 1, 2), Wt.double().permute(0, 3, 1, 2),
                 None if b is None else b.double(), padding=1)
    return y.permute(0, 2, 3, 1)


def close(got, ref, K):
    tol = 2.0 ** -8 * ref.abs() + 2e-6 * K ** 0.5 * ref.abs().max() + 1e-30
    bad = (got.double() - ref).abs() > tol
    assert not bad.any(), f"{bad.sum().item()} / {bad.numel()} mismatches, max err {(got.double() - ref).abs().max()}"


@pytest.mark.parametrize("N,H,W,Ci,Co", SHAPES)
def test_conv_forward(gpu_lib, N, H, W, Ci, Co):
    g = torch.Generator(device="cuda").manual_seed(N + H + Ci)
    X = torch.randn(N, H, W, Ci, generator=g, device="cuda").to(torch.bfloat16)
    Wt = (torch.randn(Co, 3, 3, Ci, generator=g, device="cuda") * (9 * Ci) ** -0.5).to(torch.bfloat16)
    b = torch.randn(Co, generator=g, device="cuda")
    out = torch.full((N * H * W, Co), float("nan"), device="cuda", dtype=torch.bfloat16)
    tps.conv_gemm(0, N, H, W, Ci, Co, X, Wt, out, 0, b, 1)
    torch.cuda.synchronize()
    ref = nhwc_conv_ref(X, Wt, b).clamp_min(0).reshape(N * H * W, Co)
    close(out, ref, 9 * Ci)


@pytest.mark.parametrize("N,H,W,Ci,Co", SHAPES)
@pytest.mark.parametrize("alpha", [1.0, 0.8948])
def test_conv_dgrad_flipped_weight_in_place(gpu_lib, N, H, W, Ci, Co, alpha):
    g = torch.Generator(device="cuda").manual_seed(3 * N + W + Co)
    dY = torch.randn(N, H, W, Co, generator=g, device="cuda").to(torch.bfloat16)
    Wt = (torch.randn(Co, 3, 3, Ci, generator=g, device="cuda") * (9 * Co) ** -0.5).to(torch.bfloat16)
    Xm = torch.randn(N * H * W, Ci, generator=g, device="cuda").to(torch.bfloat16)
    out = torch.full((N * H * W, Ci), float("nan"), device="cuda", dtype=torch.bfloat16)
    tps.conv_gemm(1, N, H, W, Ci, Co, dY, Wt, out, 0, None, 0, alpha, 0.0, Xm)
    torch.cuda.synchronize()
    dYd = dY.double().permute(0, 3, 1, 2)
    ref = torch.nn.grad.conv2d_input((N, Ci, H, W), Wt.double().permute(0, 3, 1, 2), dYd, padding=1)
    ref = alpha * ref.permute(0, 2, 3, 1).reshape(N * H * W, Ci) * (Xm > 0).double()
    close(out, ref, 9 * Co)


@pytest.mark.parametrize("N,H,W,Ci,Co", SHAPES)
def test_conv_wgrad(gpu_lib, N, H, W, Ci, Co):
    g = torch.Generator(device="cuda").manual_seed(5 * N + H + Ci)
    X = torch.randn(N, H, W, Ci, generator=g, device="cuda").to(torch.bfloat16)
    dY = torch.randn(N * H * W, Co, generator=g, device="cuda").to(torch.bfloat16)
    out = torch.full((Co, 9 * Ci), float("nan"), device="cuda", dtype=torch.float32)
    tps.conv_gemm(2, N, H, W, Ci, Co, dY, X, out, 1)
    torch.cuda.synchronize()
    ref = torch.nn.grad.conv2d_weight(X.double().permute(0, 3, 1, 2), (Co, Ci, 3, 3),
                                      dY.double().reshape(N, H, W, Co).permute(0, 3, 1, 2), padding=1)
    ref = ref.permute(0, 2, 3, 1).reshape(Co, 9 * Ci)
    torch.testing.assert_close(out.double(), ref, rtol=1e-5, atol=3e-6 * (N * H * W) ** 0.5 * ref.abs().max().item())


@pytest.mark.parametrize("N,H,W,Ci,Co", SHAPES[:3])
def test_conv_dgrad_blended_operand(gpu_lib, N, H, W, Ci, Co):
    g = torch.Generator(device="cuda").manual_seed(7 + N)
    dY = torch.randn(N, H, W, Co, generator=g, device="cuda").to(torch.bfloat16)
    Ws = (torch.randn(Co, 3, 3, Ci, generator=g, device="cuda") * (9 * Co) ** -0.5).to(torch.bfloat16)
    Wl = (torch.randn(Co, 3, 3, Ci, generator=g, device="cuda") * (9 * Co) ** -0.5).to(torch.bfloat16)
    out = torch.full((N * H * W, Ci), float("nan"), device="cuda", dtype=torch.bfloat16)
    a, b = 0.7408182, 0.2591818
    tps.conv_gemm(3, N, H, W, Ci, Co, dY, Ws, out, 0, None, 0, a, b, None, W2=Wl)
    torch.cuda.synchronize()
    # fp32 α·W_stash, then one fused multiply-add with β·W_latest (reading Z14), RNE to bf16
    Wr = ((torch.tensor(a) * Ws.float()).double() + torch.tensor(b, dtype=torch.float32).double() * Wl.double()).float()
    Wr = Wr.to(torch.bfloat16)
    ref = torch.nn.grad.conv2d_input((N, Ci, H, W), Wr.double().permute(0, 3, 1, 2),
                                     dY.double().permute(0, 3, 1, 2), padding=1)
    close(out, ref.permute(0, 2, 3, 1).reshape(N * H * W, Ci), 9 * Co)


# ------------------------------------------------------------------ image-net pipeline parity
def mini_vgg(H=16, C=64):
    """VGG-16's layer types at reduced depth: 3-channel first conv (explicit patches), 64/128-channel
    convs (implicit im2col), two 2x2 pools, FC head."""
    return [
        {"kind": "conv3", "cin": 3, "cout": C, "h": H, "w": H},
        {"kind": "conv3", "cin": C, "cout": C, "h": H, "w": H},
        {"kind": "pool2", "c": C, "h": H, "w": H},
        {"kind": "conv3", "cin": C, "cout": 2 * C, "h": H // 2, "w": H // 2},
        {"kind": "pool2", "c": 2 * C, "h": H // 2, "w": H // 2},
        {"kind": "linear", "in": 2 * C * (H // 4) ** 2, "out": 64},
        {"kind": "linear", "in": 64, "out": 10},
    ]


NET_CASES = {
    "S1-I-EQ1": ([0, 7], ost.I_VARIANT, ost.EQ1, 0.3, 0.9),
    "S3-V": ([0, 2, 4, 7], ost.V_VARIANT, ost.EQ1, 0.3, 0.9),
    "S3-I-EQ1": ([0, 2, 4, 7], ost.I_VARIANT, ost.EQ1, 0.3, 0.9),
    "S3-I-CONVEX": ([0, 2, 4, 7], ost.I_VARIANT, ost.CONVEX, 0.5, 0.0),
    "S4-I-EQ1": ([0, 1, 3, 5, 7], ost.I_VARIANT, ost.EQ1, 0.3, 0.5),
}


@pytest.mark.parametrize("name", list(NET_CASES))
def test_image_net_parity_with_oracle(gpu_lib, name):
    bounds, var, blend, lam, mu = NET_CASES[name]
    layers = mini_vgg()
    m, b, M = 2, 8, 10
    dims = [16 * 16 * 3, 10]
    lr = 0.01      # DESIGN.md input recipe: lr = 0.01
    ref = run_oracle(dims, bounds, m, b, M, var, blend, lam, lr, mu, kind=synthgen.X_UNIT, layers=layers)
    stages, losses = run_gpu(dims, bounds, m, b, M, var, blend, lam, lr, mu, kind=synthgen.X_UNIT, layers=layers)
    assert expand_gpu_trace(stages) == oracle_trace(ref)
    np.testing.assert_allclose(losses, ref.losses, rtol=1e-3, atol=0)
    for st in stages:
        for k, l in enumerate(st.layers):
            if ref.weights[l] is None:
                continue
            w, bb, _, _ = st.get_weights(k)
            wr = ref.weights[l].reshape(w.shape)
            assert weight_rel_err(w, wr) <= 5e-3, (name, l)
            assert layer_rel_err(w, bb, wr, ref.biases[l]) <= 5e-3, (name, l)


# ---- TMA im2col-mode convolutions (ResNet-50 geometry: any H, W; stride 2; 1x1 / 3x3) ----------
IM2COL = [  # N, H, W, Ci, Co, k, stride, pad
    (2, 56, 56, 64, 64, 3, 1, 1), (2, 28, 28, 128, 128, 3, 1, 1), (3, 7, 7, 64, 128, 3, 1, 1),
    (2, 14, 14, 256, 64, 3, 1, 1), (2, 56, 56, 128, 128, 3, 2, 1), (2, 28, 28, 256, 128, 1, 2, 0),
    (3, 7, 9, 64, 64, 3, 2, 1), (2, 32, 32, 64, 64, 3, 1, 1),
]


def conv_ref(X, Wt, s, p):
    y = F.conv2d(X.double().permute(0, 3, 1, 2), Wt.double().permute(0, 3, 1, 2), stride=s, padding=p)
    return y.permute(0, 2, 3, 1)


@pytest.mark.parametrize("N,H,W,Ci,Co,k,s,p", IM2COL)
def test_conv2d_im2col_forward_and_wgrad(gpu_lib, N, H, W, Ci, Co, k, s, p):
    g = torch.Generator(device="cuda").manual_seed(N * H + Ci + k)
    X = torch.randn(N, H, W, Ci, generator=g, device="cuda").to(torch.bfloat16)
    Wt = (torch.randn(Co, k, k, Ci, generator=g, device="cuda") * (k * k * Ci) ** -0.5).to(torch.bfloat16)
    Ho, Wo = (H + 2 * p - k) // s + 1, (W + 2 * p - k) // s + 1
    out = torch.full((N * Ho * Wo, Co), float("nan"), device="cuda", dtype=torch.bfloat16)
    tps.conv2d_gemm(0, N, H, W, Ci, Co, k, s, p, X, Wt, out)
    dY = torch.randn(N, Ho, Wo, Co, generator=g, device="cuda").to(torch.bfloat16)
    dW = torch.full((Co, k * k * Ci), float("nan"), device="cuda", dtype=torch.float32)
    tps.conv2d_gemm(2, N, H, W, Ci, Co, k, s, p, dY, X, dW, 1)
    torch.cuda.synchronize()
    close(out, conv_ref(X, Wt, s, p).reshape(N * Ho * Wo, Co), k * k * Ci)
    ref = torch.nn.grad.conv2d_weight(X.double().permute(0, 3, 1, 2), (Co, Ci, k, k),
                                      dY.double().permute(0, 3, 1, 2), stride=s, padding=p)
    ref = ref.permute(0, 2, 3, 1).reshape(Co, k * k * Ci)
    K = N * Ho * Wo
    torch.testing.assert_close(dW.double(), ref, rtol=1e-5, atol=2e-6 * K ** 0.5 * ref.abs().max().item())


@pytest.mark.parametrize("N,H,W,Ci,Co,k,s,p", [c for c in IM2COL if c[5:] == (3, 1, 1)])
@pytest.mark.parametrize("blend", [False, True])
def test_conv2d_im2col_dgrad(gpu_lib, N, H, W, Ci, Co, k, s, p, blend):
    g = torch.Generator(device="cuda").manual_seed(5 * N + W + Co)
    dY = torch.randn(N, H, W, Co, generator=g, device="cuda").to(torch.bfloat16)
    Wt = (torch.randn(Co, 3, 3, Ci, generator=g, device="cuda") * (9 * Co) ** -0.5).to(torch.bfloat16)
    W2 = (torch.randn(Co, 3, 3, Ci, generator=g, device="cuda") * (9 * Co) ** -0.5).to(torch.bfloat16)
    out = torch.full((N * H * W, Ci), float("nan"), device="cuda", dtype=torch.bfloat16)
    a, b = (0.7, 0.3) if blend else (0.8948, 0.0)
    tps.conv2d_gemm(3 if blend else 1, N, H, W, Ci, Co, 3, 1, 1, dY, Wt, out, 0, a, b, W2=W2 if blend else None)
    torch.cuda.synchronize()
    # blend on load (reading Z14): fp32 α·W_stash, one fused multiply-add with β·W_latest, RNE to bf16
    Wr = ((torch.tensor(a) * Wt.float()).double() + torch.tensor(b, dtype=torch.float32).double() * W2.double()).float()
    Wr = Wr.to(torch.bfloat16) if blend else Wt
    ref = torch.nn.grad.conv2d_input((N, Ci, H, W), Wr.double().permute(0, 3, 1, 2), dY.double().permute(0, 3, 1, 2),
                                     padding=1)
    ref = ref.permute(0, 2, 3, 1).reshape(N * H * W, Ci) * (1.0 if blend else a)
    close(out, ref, 9 * Co)

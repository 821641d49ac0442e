"""Kernel unit tests of the tcgen05 stage GEMM (tps_gemm) against torch fp64 references.

Shapes cover several tiles, ragged M/N/K tails (TMA zero fill + masked epilogue), the
config shapes (C1 784-256-10 head, C2/C5 4096²), and all three operand layouts plus
the blended-operand dgrad (I-TiMePReSt, reading Z1).
"""
import pytest
import torch

from paper_2509_23241_b200 import tps

pytestmark = pytest.mark.gpu


def bf16_rand(*shape, scale=1.0, gen=None):
    return (torch.randn(*shape, generator=gen, device="cuda") * scale).to(torch.bfloat16)


def close_bf16(got, ref, K_eff):
    # fp32 accumulation of K products + one bf16 rounding of the result
    tol = 2.0 ** -8 * ref.abs() + 1e-6 * K_eff ** 0.5 * ref.abs().max() + 1e-30
    bad = (got.double() - ref).abs() > tol
    assert not bad.any(), f"{bad.sum().item()} / {bad.numel()} mismatches, max err {(got.double()-ref).abs().max().item()}"


FWD_SHAPES = [(32, 256, 784), (128, 16, 256), (300, 264, 1000), (1024, 1024, 1024), (2048, 4096, 512), (8, 64, 64)]


@pytest.mark.parametrize("M,N,K", FWD_SHAPES)
@pytest.mark.parametrize("relu", [0, 1])
def test_forward_bias_relu_bf16(gpu_lib, M, N, K, relu):
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N + K)
    A = bf16_rand(M, K, gen=g)
    W = bf16_rand(N, K, scale=K ** -0.5, gen=g)
    bias = torch.randn(N, generator=g, device="cuda", dtype=torch.float32)
    out = torch.full((M, N), float("nan"), device="cuda", dtype=torch.bfloat16)
    tps.gemm(tps.GEMM_FWD, M, N, K, A, K, W, K, out, N, 0, bias, relu)
    torch.cuda.synchronize()
    ref = A.double() @ W.double().T + bias.double()
    if relu:
        ref = ref.clamp_min(0)
    close_bf16(out, ref, K)


@pytest.mark.parametrize("M,N,K", [(32, 16, 256), (257, 136, 136), (512, 4096, 4096)])
def test_forward_fp32_logits(gpu_lib, M, N, K):
    g = torch.Generator(device="cuda").manual_seed(1)
    A = bf16_rand(M, K, gen=g)
    W = bf16_rand(N, K, scale=K ** -0.5, gen=g)
    out = torch.zeros((M, N), device="cuda", dtype=torch.float32)
    tps.gemm(tps.GEMM_FWD, M, N, K, A, K, W, K, out, N, 1)
    torch.cuda.synchronize()
    ref = A.double() @ W.double().T
    torch.testing.assert_close(out.double(), ref, rtol=1e-5, atol=1e-5 * ref.abs().max().item())


@pytest.mark.parametrize("M,N,K", [(32, 256, 16), (300, 264, 136), (2048, 1024, 4096), (96, 784, 256)])
@pytest.mark.parametrize("alpha", [1.0, 0.8948, -2.0])
def test_dgrad_mn_major_weight_alpha_mask(gpu_lib, M, N, K, alpha):
    # G [M, K] · W where W is stored [K rows, N cols] (the layer's [out, in] weight)
    g = torch.Generator(device="cuda").manual_seed(M + N * 3 + K)
    G = bf16_rand(M, K, gen=g)
    W = bf16_rand(K, N, scale=K ** -0.5, gen=g)
    X = bf16_rand(M, N, gen=g)  # mask source: zero where X <= 0
    out = torch.full((M, N), float("nan"), device="cuda", dtype=torch.bfloat16)
    tps.gemm(tps.GEMM_DGRAD, M, N, K, G, K, W, N, out, N, 0, None, 0, alpha, 0.0, X, N)
    torch.cuda.synchronize()
    ref = alpha * (G.double() @ W.double()) * (X > 0).double()
    close_bf16(out, ref, K)


@pytest.mark.parametrize("M,N,K", [(256, 784, 32), (16, 256, 32), (136, 264, 300), (4096, 4096, 512), (1024, 512, 2048),
                                   (64, 64, 65536), (128, 576, 50176), (256, 2304, 12544), (72, 136, 40000)])
def test_wgrad_both_mn_major(gpu_lib, M, N, K):
    """The last four are ResNet-style weight gradients (few output tiles, K = every pixel of the
    batch): they take the split-K path (fp32 partials per K range, ordered reduction)."""
    # dW [M, N] = Gᵀ·X with G stored [K, M] and X stored [K, N]; fp32 out
    g = torch.Generator(device="cuda").manual_seed(M + N + K * 5)
    G = bf16_rand(K, M, gen=g)
    X = bf16_rand(K, N, gen=g)
    out = torch.full((M, N), float("nan"), device="cuda", dtype=torch.float32)
    tps.gemm(tps.GEMM_WGRAD, M, N, K, G, M, X, N, out, N, 1)
    torch.cuda.synchronize()
    ref = G.double().T @ X.double()
    torch.testing.assert_close(out.double(), ref, rtol=1e-5, atol=2e-6 * K ** 0.5 * ref.abs().max().item())


# (2048, 4096, 1024) and (1800, 4000, 1040) run on 512-row CTA-pair tiles (two accumulators sharing
# one blended B tile, ragged M / N / K tails in the second case); (512, 4096, 1024) and (520, 3000, 200)
# on 256 x 128 CTA-pair tiles; the others on 128-row single-CTA tiles
@pytest.mark.parametrize("M,N,K", [(64, 256, 64), (300, 264, 136), (2048, 4096, 1024), (1800, 4000, 1040),
                                   (512, 4096, 1024), (520, 3000, 200)])
@pytest.mark.parametrize("a,b", [(0.25, 0.75), (0.9512294, 0.0487706), (-6.0, 0.0)])
def test_dgrad_blended_operand(gpu_lib, M, N, K, a, b):
    # G · bf16(α·W_stash + β·W_latest), operand formed in shared memory (K8 definition, reading Z14)
    g = torch.Generator(device="cuda").manual_seed(11 + M)
    G = bf16_rand(M, K, gen=g)
    Ws = bf16_rand(K, N, scale=K ** -0.5, gen=g)
    Wl = bf16_rand(K, N, scale=K ** -0.5, gen=g)
    X = bf16_rand(M, N, gen=g)
    out = torch.full((M, N), float("nan"), device="cuda", dtype=torch.bfloat16)
    tps.gemm(tps.GEMM_DGRAD_BLEND, M, N, K, G, K, Ws, N, out, N, 0, None, 0, a, b, X, N, B2=Wl)
    torch.cuda.synchronize()
    af, bf = torch.tensor(a, dtype=torch.float32), torch.tensor(b, dtype=torch.float32)
    # fp32 α·W_stash, then one fused multiply-add with β·W_latest (exact in fp64, one fp32 rounding), RNE
    Wr = ((af * Ws.float()).double() + bf.double() * Wl.double()).float().to(torch.bfloat16)
    ref = (G.double() @ Wr.double()) * (X > 0).double()
    close_bf16(out, ref, K)

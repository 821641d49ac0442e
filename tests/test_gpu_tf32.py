"""tf32 storage mode (tps_config.dtype = TPS_TF32, reading Z28; north_star "bf16/tf32 inputs with
fp32 accumulation").

* the raw stage GEMM in tf32 (tps_gemm mode | TPS_GEMM_TF32: kind::tf32 MMAs on fp32 containers,
  all four modes incl. the blend on load on 128-, 256- and 512-row tiles) against float64
  products of the same tf32 operands, with the output rounded RNA to tf32;
* whole pipelines in tf32 storage against the oracle run with tf32 rounding (oracle/tf32.py):
  schedule / staleness trace bit-exact, losses 1e-3 relative, weights 5e-3 max-relative after
  10 mini-batches (north_star), fused and separate update, V / I-EQ1 / I-CONVEX, S = 1..4;
* the version the update writes is exactly tf32_rna(fp32 master) and the K8 materialiser is
  tf32_rna(fp32(α·s) + fp32(β·l)) (oracle.mlp.materialize_blend, dtype "tf32").
"""
import numpy as np
import pytest
import torch

import synthgen
from oracle import mlp as omlp
from oracle import staleness as ost
from oracle import tf32 as otf32
from paper_2509_23241_b200 import tps
from pipeline_helpers import (expand_gpu_trace, layer_rel_err, oracle_trace, run_gpu, run_oracle, weight_rel_err)

pytestmark = pytest.mark.gpu


def tf32_rand(*shape, scale=1.0, gen=None):
    x = (torch.randn(*shape, generator=gen, device="cuda") * scale).float()
    # RNA to tf32 on the bit pattern (the test's own rounding, independent of the kernels)
    u = x.view(torch.int32).to(torch.int64)
    u = (u + 0x1000) & 0xFFFFE000
    return u.to(torch.int32).view(torch.float32)


def rna64(t):
    return torch.from_numpy(otf32.rna(t.double().cpu().numpy())).to(t.device)


def close_tf32(got, ref, K_eff):
    # fp32 accumulation of K exact tf32 products + one RNA rounding to tf32 (2^-11 relative)
    tol = 2.0 ** -11 * ref.abs() + 4e-6 * K_eff ** 0.5 * ref.abs().max() + 1e-30
    bad = (got.double() - ref).abs() > tol
    assert not bad.any(), f"{bad.sum().item()} / {bad.numel()} mismatches, max err {(got.double() - ref).abs().max().item()}"


SHAPES = [(64, 256, 64), (296, 264, 136), (2048, 1024, 512), (8, 64, 64)]


@pytest.mark.parametrize("M,N,K", SHAPES)
@pytest.mark.parametrize("relu", [0, 1])
def test_tf32_forward(gpu_lib, M, N, K, relu):
    g = torch.Generator(device="cuda").manual_seed(1 + M + N)
    X = tf32_rand(M, K, gen=g)
    W = tf32_rand(N, K, scale=K ** -0.5, gen=g)
    bias = torch.randn(N, generator=g, device="cuda") * 0.1
    out = torch.full((M, N), float("nan"), device="cuda")
    tps.gemm(tps.GEMM_FWD | tps.TPS_GEMM_TF32, M, N, K, X, K, W, K, out, N, 0, bias, relu)
    torch.cuda.synchronize()
    ref = X.double() @ W.double().T + bias.double()
    if relu:
        ref = ref.clamp_min(0)
    close_tf32(out, ref, K)
    # stored values are tf32 (13 low mantissa bits zero)
    assert (out.view(torch.int32) & 0x1FFF).eq(0).all()


@pytest.mark.parametrize("M,N,K", SHAPES)
def test_tf32_dgrad_alpha_mask(gpu_lib, M, N, K):
    g = torch.Generator(device="cuda").manual_seed(5 + M)
    G = tf32_rand(M, K, gen=g)
    Wt = tf32_rand(K, N, scale=K ** -0.5, gen=g)       # stored [K, N] (MN-major)
    X = tf32_rand(M, N, gen=g)
    out = torch.full((M, N), float("nan"), device="cuda")
    tps.gemm(tps.GEMM_DGRAD | tps.TPS_GEMM_TF32, M, N, K, G, K, Wt, N, out, N, 0, None, 0, 0.75, 0.0, X, N)
    torch.cuda.synchronize()
    ref = (G.double() @ Wt.double()) * 0.75 * (X > 0).double()
    close_tf32(out, ref, K)


@pytest.mark.parametrize("M,N,K", SHAPES)
def test_tf32_wgrad(gpu_lib, M, N, K):
    g = torch.Generator(device="cuda").manual_seed(9 + K)
    G = tf32_rand(K, M, gen=g)                         # stored [K, M]
    X = tf32_rand(K, N, gen=g)
    out = torch.full((M, N), float("nan"), device="cuda")
    tps.gemm(tps.GEMM_WGRAD | tps.TPS_GEMM_TF32, M, N, K, G, M, X, N, out, N, 1)
    torch.cuda.synchronize()
    ref = G.double().T @ X.double()
    torch.testing.assert_close(out.double(), ref, rtol=1e-5, atol=4e-6 * K ** 0.5 * ref.abs().max().item())


# 128-row (CG = 1), 256-row pair and 512-row pair (MH = 2) tiles
@pytest.mark.parametrize("M,N,K", [(64, 256, 64), (300, 264, 136), (2048, 4096, 1024), (1800, 4000, 1040),
                                   (512, 4096, 1024)])
@pytest.mark.parametrize("a,b", [(0.25, 0.75), (-6.0, 0.0)])
def test_tf32_dgrad_blended_operand(gpu_lib, M, N, K, a, b):
    g = torch.Generator(device="cuda").manual_seed(11 + M)
    G = tf32_rand(M, K, gen=g)
    Ws = tf32_rand(K, N, scale=K ** -0.5, gen=g)
    Wl = tf32_rand(K, N, scale=K ** -0.5, gen=g)
    X = tf32_rand(M, N, gen=g)
    out = torch.full((M, N), float("nan"), device="cuda")
    tps.gemm(tps.GEMM_DGRAD_BLEND | tps.TPS_GEMM_TF32, M, N, K, G, K, Ws, N, out, N, 0, None, 0, a, b, X, N, B2=Wl)
    torch.cuda.synchronize()
    af, bf = torch.tensor(a, dtype=torch.float32), torch.tensor(b, dtype=torch.float32)
    # fp32 α·W_stash, one fused multiply-add with β·W_latest (exact in fp64, one fp32 rounding), RNA
    Wr = rna64(((af * Ws.cpu()).double() + bf.double() * Wl.cpu().double()).float())
    ref = (G.double() @ Wr.to(G.device)) * (X > 0).double()
    close_tf32(out, ref, K)


CASES = {
    # name: dims, bounds, m, b, M, variant, blend, lam, lr, mu
    "S1-deep": ([512, 384, 256, 16], [0, 3], 4, 32, 10, ost.I_VARIANT, ost.EQ1, 0.05, 0.05, 0.9),
    "S4-I-EQ1": ([256] * 6 + [10], [0, 2, 3, 5, 6], 2, 64, 10, ost.I_VARIANT, ost.EQ1, 0.3, 0.05, 0.9),
    "S4-I-CONVEX": ([256] * 6 + [10], [0, 2, 3, 5, 6], 2, 64, 10, ost.I_VARIANT, ost.CONVEX, 0.3, 0.05, 0.0),
    "S2-V": ([256] * 4 + [10], [0, 2, 4], 2, 32, 10, ost.V_VARIANT, ost.EQ1, 0.3, 0.05, 0.5),
    "S3-ragged": ([200, 136, 72, 40, 10], [0, 2, 3, 4], 3, 24, 10, ost.I_VARIANT, ost.CONVEX, 0.2, 0.05, 0.5),
    # wide: CTA-pair GEMMs, the bias step on the optimizer stream, blend on 256-row tiles
    "S2-wide-CONVEX": ([1024] * 4 + [10], [0, 2, 4], 4, 128, 10, ost.I_VARIANT, ost.CONVEX, 0.05, 0.05, 0.9),
}


@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("fuse", [1, 0])
def test_tf32_pipeline_parity(gpu_lib, name, fuse):
    dims, bounds, m, b, M, var, blend, lam, lr, mu = CASES[name]
    ref = run_oracle(dims, bounds, m, b, M, var, blend, lam, lr, mu, dtype="tf32")
    ex = run_oracle(dims, bounds, m, b, M, var, blend, lam, lr, mu, exact=True)
    stages, losses = run_gpu(dims, bounds, m, b, M, var, blend, lam, lr, mu, fuse_update=fuse, dtype=tps.TPS_TF32)
    assert expand_gpu_trace(stages) == oracle_trace(ref)
    np.testing.assert_allclose(losses, ref.losses, rtol=1e-3, atol=0)
    for st in stages:
        for k, l in enumerate(st.layers):
            w, bb, _, _ = st.get_weights(k)
            assert weight_rel_err(w, ref.weights[l]) <= 5e-3, (name, l)
            assert layer_rel_err(w, bb, ref.weights[l], ref.biases[l]) <= 5e-3, (name, l)
            if np.abs(ref.biases[l]).max() > 0:   # the bias alone, as in test_gpu_pipeline (reading Z19)
                gap = weight_rel_err(ex.biases[l], ref.biases[l])
                assert weight_rel_err(bb, ref.biases[l]) <= max(5e-3, 2 * gap), (name, l)
    for st in stages:
        st.close()


def test_tf32_versions_and_materialiser(gpu_lib):
    """The latest version is tf32_rna(fp32 master) bit for bit; the K8 materialiser is
    tf32_rna(fp32(α·s) + fp32(β·l)) (oracle.mlp.materialize_blend, dtype "tf32")."""
    dims, bounds = [256, 256, 256, 10], [0, 3]
    stages, _ = run_gpu(dims, bounds, 2, 32, 5, ost.I_VARIANT, ost.CONVEX, 0.4, 0.05, 0.9, dtype=tps.TPS_TF32,
                        max_inflight=3)
    st = stages[0]
    for k in range(3):
        w = st.get_weights(k)[0]
        Np, Kp = (dims[k + 1] + 15) // 16 * 16, (dims[k] + 15) // 16 * 16
        v0 = torch.empty(Np, Kp, device="cuda")
        st.get_version(k, 0, v0)
        v0 = v0.cpu().numpy()[: dims[k + 1], : dims[k]]
        assert np.array_equal(v0.astype(np.float64), otf32.rna(w.astype(np.float64)))
        v0_full = st_version(st, k, 0, Np, Kp)
        v2_full = st_version(st, k, 2, Np, Kp)
        out = torch.empty(Np, Kp, device="cuda")
        st.intermediate_weight(k, 2, out)
        a, b = ost.blend_coeffs(ost.I_VARIANT, ost.CONVEX, 2, 0.4)
        want = omlp.materialize_blend(v2_full, v0_full, a, b, dtype="tf32")
        assert np.array_equal(out.cpu().numpy().astype(np.float64), want)
        assert not np.array_equal(v2_full, v0_full)          # two distinct live versions
    st.close()


def st_version(st, k, d, Np, Kp):
    v = torch.empty(Np, Kp, device="cuda")
    st.get_version(k, d, v)
    return v.cpu().numpy()

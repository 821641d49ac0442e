"""Pins for oracle.mlp and oracle.pipeline.

* exact mode, S = 1 == torch fp64 autograd + torch.optim.SGD (north_star: "a 1-stage
  pipeline reduces to plain SGD")
* finite-difference gradients (north_star)
* exact mode, S > 1 == an independent torch-autograd replay that derives the
  weight versions from the closed forms pinned by the paper's worked examples
* bitwise properties: V ≡ I on config-1-shaped nets (reading Z12), I-CONVEX at
  λ -> ∞ ≡ V, I-EQ1 freeze at λ = ln 2, V has δ = 0 everywhere,
  peak live versions V = 1 / I = S - s
* update rule == torch.optim.SGD in fp32 (within 1 ulp)
"""
import math

import numpy as np
import pytest
import torch
import torch.nn.functional as F

import synthgen
from oracle import mlp, pipeline, staleness as st


def make_inputs(dims, m, b, M, seed=0, kind=synthgen.X_SIGNED):
    B = m * b
    xs = [synthgen.inputs(seed, j, B, dims[0], kind) for j in range(M)]
    ys = [synthgen.labels(seed, j, B, dims[-1]) for j in range(M)]
    w0 = [synthgen.weights(seed, l, dims[l + 1], dims[l]) for l in range(len(dims) - 1)]
    b0 = [np.zeros(dims[l + 1], np.float32) for l in range(len(dims) - 1)]
    return xs, ys, w0, b0


# ---------------------------------------------------------------- S = 1 == SGD
@pytest.mark.parametrize("mu,wd", [(0.0, 0.0), (0.9, 1e-3)])
def test_single_stage_exact_equals_torch_sgd(mu, wd):
    dims, m, b, M = [12, 9, 7, 5], 2, 3, 6
    xs, ys, w0, b0 = make_inputs(dims, m, b, M)
    cfg = pipeline.Config(dims, [0, 3], m, b, M, lr=0.1, momentum=mu, wd=wd, exact=True)
    res = pipeline.run(cfg, xs, ys, w0, b0)
    params = []
    for w, bb in zip(w0, b0):
        params += [torch.tensor(w, dtype=torch.float64, requires_grad=True),
                   torch.tensor(bb, dtype=torch.float64, requires_grad=True)]
    opt = torch.optim.SGD(params, lr=0.1, momentum=mu, weight_decay=wd)
    losses = []
    for j in range(M):
        h = torch.tensor(xs[j], dtype=torch.float64)
        for l in range(3):
            h = F.linear(h, params[2 * l], params[2 * l + 1])
            if l < 2:
                h = torch.relu(h)
        loss = F.cross_entropy(h, torch.tensor(ys[j], dtype=torch.long))
        opt.zero_grad()
        loss.backward()
        opt.step()
        losses.append(loss.item())
    np.testing.assert_allclose(res.losses, losses, rtol=1e-12, atol=0)
    for l in range(3):
        np.testing.assert_allclose(res.weights[l], params[2 * l].detach().numpy(), rtol=1e-11, atol=1e-14)
        np.testing.assert_allclose(res.biases[l], params[2 * l + 1].detach().numpy(), rtol=1e-11, atol=1e-14)


def test_finite_difference_gradients():
    # one mini-batch, lr = 1, μ = 0: w_after = w0 - g  ->  g = w0 - w_after; compare with
    # central differences of the oracle's own loss (rel err <= 1e-5)
    dims, m, b = [6, 5, 4, 3], 2, 4
    xs, ys, w0, b0 = make_inputs(dims, m, b, 1, seed=7)
    rng = np.random.default_rng(3)
    b0 = [rng.standard_normal(d).astype(np.float32) * 0.1 for d in dims[1:]]

    def loss_at(ws, bs):
        cfg = pipeline.Config(dims, [0, 2, 3], m, b, 1, lr=0.0, exact=True)
        return pipeline.run(cfg, xs, ys, ws, bs).losses[0]

    cfg = pipeline.Config(dims, [0, 2, 3], m, b, 1, lr=1.0, exact=True)
    res = pipeline.run(cfg, xs, ys, w0, b0)
    h = 1e-6
    for l in range(3):
        g = np.asarray(w0[l], np.float64) - res.weights[l]
        for (i, k) in [(0, 0), (1, 2), (dims[l + 1] - 1, dims[l] - 1)]:
            wp = [np.array(w, np.float64) for w in w0]
            wm = [np.array(w, np.float64) for w in w0]
            wp[l][i, k] += h
            wm[l][i, k] -= h
            fd = (loss_at(wp, b0) - loss_at(wm, b0)) / (2 * h)
            assert abs(fd - g[i, k]) <= 1e-5 * max(1e-3, abs(fd)), (l, i, k, fd, g[i, k])
        gb = np.asarray(b0[l], np.float64) - res.biases[l]
        bp = [np.array(x, np.float64) for x in b0]
        bm = [np.array(x, np.float64) for x in b0]
        bp[l][0] += h
        bm[l][0] -= h
        fd = (loss_at(w0, bp) - loss_at(w0, bm)) / (2 * h)
        assert abs(fd - gb[0]) <= 1e-5 * max(1e-3, abs(fd))


def test_softmax_xent_closed_form_logistic():
    # two-class softmax CE gradient is σ(z1 - z0) - y on logit 1
    z = np.array([[0.3, -1.2], [2.0, 0.5]])
    y = np.array([1, 0])
    rows, g = mlp.softmax_xent(z, y, batch=1)
    sig = 1 / (1 + np.exp(-(z[:, 1] - z[:, 0])))
    np.testing.assert_allclose(g[:, 1], sig - (y == 1), rtol=1e-14)
    np.testing.assert_allclose(rows, -np.log(np.where(y == 1, sig, 1 - sig)), rtol=1e-14)


# ----------------------------------------------- independent torch replay, S > 1
def torch_replay(dims, bounds, m, b, M, variant, blend, lam, lr, mu, xs, ys, w0, b0):
    """Closed-form versions (pinned by tests/golden) + torch autograd.

    Stage s forwards mini-batch j on version v_f = max(0, j - S + s + 1) and its
    backward reads W_res = α·W^{v_f} + β·W^{j} (V: W^{j}); the gradient w.r.t. this
    layer's weights is dZᵀX with dZ flowing through W_res.  Built with the detach trick
    Z = X·Pᵀ + detach(X·(W_f - P)ᵀ), P := W_res (value = X·W_fᵀ, dZ/dX = P, dZ/dP = X).
    """
    S = len(bounds) - 1
    L = len(dims) - 1
    stage_of = [next(s for s in range(S) if bounds[s] <= l < bounds[s + 1]) for l in range(L)]
    hist_w = [[torch.tensor(w, dtype=torch.float64)] for w in w0]    # hist_w[l][v]
    hist_b = [[torch.tensor(x, dtype=torch.float64)] for x in b0]
    mom_w = [torch.zeros_like(h[0]) for h in hist_w]
    mom_b = [torch.zeros_like(h[0]) for h in hist_b]
    losses = []
    for j in range(M):
        Ps, bs = [], []
        h = torch.tensor(xs[j], dtype=torch.float64)
        for l in range(L):
            s = stage_of[l]
            vf = max(0, j - S + s + 1)
            delta = j - vf
            Wf, Wl = hist_w[l][vf], hist_w[l][j]
            if variant == st.V_VARIANT:
                Wres = Wl
            else:
                a, bb = st.blend_coeffs(variant, blend, delta, lam)
                Wres = a * Wf + bb * Wl
            P = Wres.clone().requires_grad_(True)
            bias = hist_b[l][vf].clone().requires_grad_(True)
            z = h @ P.T + (h @ (Wf - P).T).detach() + bias
            Ps.append(P)
            bs.append(bias)
            h = torch.relu(z) if l < L - 1 else z
        loss = F.cross_entropy(h, torch.tensor(ys[j], dtype=torch.long))
        grads = torch.autograd.grad(loss, Ps + bs)
        losses.append(loss.item())
        for l in range(L):
            gw, gb = grads[l], grads[L + l]
            mom_w[l] = mu * mom_w[l] + gw
            mom_b[l] = mu * mom_b[l] + gb
            hist_w[l].append(hist_w[l][j] - lr * mom_w[l])
            hist_b[l].append(hist_b[l][j] - lr * mom_b[l])
    return np.array(losses), [h[-1].numpy() for h in hist_w], [h[-1].numpy() for h in hist_b]


@pytest.mark.parametrize("variant,blend,lam", [
    (st.V_VARIANT, st.EQ1, 0.5),
    (st.I_VARIANT, st.EQ1, 0.3),
    (st.I_VARIANT, st.CONVEX, 0.7),
    (st.I_VARIANT, st.EQ1, 1e-12),
])
@pytest.mark.parametrize("S", [2, 3, 4])
def test_multistage_exact_equals_torch_replay(variant, blend, lam, S):
    dims = [10, 9, 8, 8, 7, 6][: S + 2]
    bounds = list(range(S)) + [len(dims) - 1]        # last stage holds two layers
    m, b, M = 2, 3, 7
    xs, ys, w0, b0 = make_inputs(dims, m, b, M, seed=S)
    cfg = pipeline.Config(dims, bounds, m, b, M, variant=variant, blend=blend, lam=lam,
                          lr=0.05, momentum=0.5, exact=True)
    res = pipeline.run(cfg, xs, ys, w0, b0)
    tl, tw, tb = torch_replay(dims, bounds, m, b, M, variant, blend, lam, 0.05, 0.5, xs, ys, w0, b0)
    np.testing.assert_allclose(res.losses, tl, rtol=1e-11)
    for l in range(len(dims) - 1):
        np.testing.assert_allclose(res.weights[l], tw[l], rtol=1e-10, atol=1e-13)
        np.testing.assert_allclose(res.biases[l], tb[l], rtol=1e-10, atol=1e-13)


# --------------------------------------------------------------- bitwise properties
def test_v_equals_i_on_config1_shape():
    # config 1: 784-256-10, S = 2, stage 0 = single layer (no dgrad), stage 1 has δ = 0 (Z12)
    dims, m, b, M = [784, 256, 10], 4, 8, 10
    xs, ys, w0, b0 = make_inputs(dims, m, b, M, kind=synthgen.X_UNIT)
    out = []
    for variant, blend in [(st.V_VARIANT, st.EQ1), (st.I_VARIANT, st.EQ1), (st.I_VARIANT, st.CONVEX)]:
        cfg = pipeline.Config(dims, [0, 1, 2], m, b, M, variant=variant, blend=blend, lam=0.5, lr=0.05)
        out.append(pipeline.run(cfg, xs, ys, w0, b0))
    for r in out[1:]:
        assert np.array_equal(r.losses, out[0].losses)
        for l in range(2):
            assert np.array_equal(r.weights[l], out[0].weights[l])


def test_convex_infinite_lambda_equals_v():
    # CONVEX with f = e^{-λδ} -> 0: α = 0, β = 1 exactly in fp32 for δ >= 1 -> W_res = W_latest (V)
    dims, m, b, M = [16, 16, 16, 16, 10], 2, 4, 8
    xs, ys, w0, b0 = make_inputs(dims, m, b, M, seed=5)
    bounds = [0, 2, 3, 4]
    rv = pipeline.run(pipeline.Config(dims, bounds, m, b, M, variant=st.V_VARIANT, lr=0.05), xs, ys, w0, b0)
    ri = pipeline.run(pipeline.Config(dims, bounds, m, b, M, variant=st.I_VARIANT, blend=st.CONVEX,
                                      lam=200.0, lr=0.05), xs, ys, w0, b0)
    assert np.array_equal(rv.losses, ri.losses)
    for l in range(4):
        assert np.array_equal(rv.weights[l], ri.weights[l])


def test_i_differs_from_v_with_deep_stage0():
    dims, m, b, M = [16, 16, 16, 16, 10], 2, 4, 8
    xs, ys, w0, b0 = make_inputs(dims, m, b, M, seed=5)
    bounds = [0, 2, 3, 4]
    rv = pipeline.run(pipeline.Config(dims, bounds, m, b, M, variant=st.V_VARIANT, lr=0.05), xs, ys, w0, b0)
    ri = pipeline.run(pipeline.Config(dims, bounds, m, b, M, variant=st.I_VARIANT, lam=0.5, lr=0.05),
                      xs, ys, w0, b0)
    assert not np.array_equal(rv.weights[0], ri.weights[0])


@pytest.mark.parametrize("S", [3, 4])
def test_i_eq1_freeze_at_ln2(S):
    # EQ1, λ = ln 2, μ = wd = 0: for j >= 1 stage S-2 has δ = 1 -> α = 0, so every gradient
    # below its last layer is exactly 0 and those parameters stay bitwise constant.
    dims = [12] * (S + 2) + [10]
    dims = dims[: S + 3]
    bounds = [0] + [2 + k for k in range(S - 1)] + [len(dims) - 1]
    bounds[-2] = bounds[-1] - 1
    bounds = sorted(set(bounds))
    assert len(bounds) == S + 1
    m, b, M = 2, 4, 6
    xs, ys, w0, b0 = make_inputs(dims, m, b, M, seed=11)
    snap = {}
    for MM in (1, M):
        cfg = pipeline.Config(dims, bounds, m, b, MM, variant=st.I_VARIANT, blend=st.EQ1,
                              lam=math.log(2), lr=0.1)
        snap[MM] = pipeline.run(cfg, xs, ys, w0, b0)
    last_of_sm2 = bounds[S - 1] - 1         # last layer of stage S-2
    for l in range(last_of_sm2):             # everything strictly below it
        assert np.array_equal(snap[1].weights[l], snap[M].weights[l]), l
        assert np.array_equal(snap[1].biases[l], snap[M].biases[l]), l
    assert not np.array_equal(snap[1].weights[last_of_sm2], snap[M].weights[last_of_sm2])
    alphas = {(r.stage, r.mb): r.alpha for r in snap[M].trace if r.kind == "B"}
    assert all(alphas[(S - 2, j)] == 0.0 for j in range(1, M))


def test_v_has_zero_staleness_and_one_version():
    dims, bounds, m, b, M = [8, 8, 8, 8, 4], [0, 1, 2, 3, 4], 2, 2, 9
    xs, ys, w0, b0 = make_inputs(dims, m, b, M)
    rv = pipeline.run(pipeline.Config(dims, bounds, m, b, M, variant=st.V_VARIANT), xs, ys, w0, b0)
    assert all(r.delta == 0 for r in rv.trace)
    assert all(r.v_used == r.v_latest for r in rv.trace if r.kind == "B")
    assert rv.peak_versions == [1] * 4
    ri = pipeline.run(pipeline.Config(dims, bounds, m, b, M, variant=st.I_VARIANT), xs, ys, w0, b0)
    assert ri.peak_versions == [4, 3, 2, 1]                         # K_s = S - s
    assert max(r.delta for r in ri.trace) == 3


# --------------------------------------------------------------------- update rule
def test_sgd_update_matches_torch_optim_fp32():
    # one step at a time from identical state; torch may fuse a + α·b (one rounding), so allow
    # 1 ulp of the operands' magnitude (cancellation makes ulps of the result meaningless)
    rng = np.random.default_rng(0)
    w = rng.standard_normal(10000).astype(np.float32)
    v = rng.standard_normal(10000).astype(np.float32)
    for step in range(3):
        g = rng.standard_normal(10000).astype(np.float32)
        tw = torch.tensor(w.copy(), requires_grad=True)
        opt = torch.optim.SGD([tw], lr=0.01, momentum=0.9, weight_decay=1e-4, foreach=False)
        opt.state[tw]["momentum_buffer"] = torch.tensor(v.copy())
        tw.grad = torch.tensor(g)
        opt.step()
        w2, v2 = mlp.sgd_update(w, v, g, 0.01, 0.9, 1e-4)
        vref = opt.state[tw]["momentum_buffer"].numpy()
        scale_v = np.maximum(np.abs(0.9 * v), np.abs(g)) + np.abs(1e-4 * w)
        assert (np.abs(v2 - vref) <= 2 * np.spacing(scale_v.astype(np.float32))).all()
        scale_w = np.maximum(np.abs(w), np.abs(0.01 * v2))
        assert (np.abs(w2 - tw.detach().numpy()) <= 2 * np.spacing(scale_w.astype(np.float32))).all()
        w, v = w2, v2


def test_materialize_blend_definition():
    s = np.array([1.0, -2.0, 0.5], np.float32)
    l = np.array([3.0, 1.0, -0.5], np.float32)
    got = mlp.materialize_blend(s, l, 0.25, 0.75)
    assert np.array_equal(got, [2.5, 0.25, -0.25])

"""Pins for oracle.conv (3x3 convolution, 2x2 max-pool) and the image-net pipeline path.

* forward / input-gradient / weight-gradient of conv3x3 == brute-force loops (tiny) and
  torch fp64 conv2d + autograd (library routine)
* max-pool forward == torch max_pool2d; backward routes to the FIRST window maximum
  (reading Z15) == brute force, including exact ties
* exact-mode S = 1 conv-net pipeline == torch fp64 autograd + torch.optim.SGD
* exact-mode S > 1 conv-net pipeline == independent torch-autograd replay with the closed-form
  versions (pinned by the paper's worked examples in tests/golden)
"""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

import synthgen
from oracle import conv, pipeline, staleness as st


def rnd(*shape, seed=0):
    return np.random.default_rng(seed).standard_normal(shape)


def brute_conv(X, W, b):
    N, H, Wd, Ci = X.shape
    Co = W.shape[0]
    Z = np.zeros((N, H, Wd, Co))
    for n in range(N):
        for h in range(H):
            for w in range(Wd):
                for o in range(Co):
                    s = b[o]
                    for kh in range(3):
                        for kw in range(3):
                            hh, ww = h + kh - 1, w + kw - 1
                            if 0 <= hh < H and 0 <= ww < Wd:
                                s += X[n, hh, ww, :] @ W[o, kh, kw, :]
                    Z[n, h, w, o] = s
    return Z


def torch_conv(X, W, b):
    # NHWC <-> NCHW; W [Co,3,3,Ci] -> [Co,Ci,3,3]
    x = torch.tensor(X).permute(0, 3, 1, 2)
    w = torch.tensor(W).permute(0, 3, 1, 2)
    return F.conv2d(x, w, torch.tensor(b), padding=1).permute(0, 2, 3, 1).numpy()


def test_conv_forward_brute_force_and_torch():
    X, W, b = rnd(2, 5, 4, 3, seed=1), rnd(4, 3, 3, 3, seed=2), rnd(4, seed=3)
    Z = conv.conv3x3_forward(X, W, b)
    np.testing.assert_allclose(Z, brute_conv(X, W, b), rtol=1e-12, atol=1e-12)
    X, W, b = rnd(3, 8, 8, 16, seed=4), rnd(8, 3, 3, 16, seed=5), rnd(8, seed=6)
    np.testing.assert_allclose(conv.conv3x3_forward(X, W, b), torch_conv(X, W, b), rtol=1e-12, atol=1e-12)


def test_conv_gradients_match_torch_autograd():
    X, W, b = rnd(2, 6, 6, 5, seed=7), rnd(7, 3, 3, 5, seed=8), rnd(7, seed=9)
    dZ = rnd(2, 6, 6, 7, seed=10)
    x = torch.tensor(X).permute(0, 3, 1, 2).requires_grad_(True)
    w = torch.tensor(W).permute(0, 3, 1, 2).detach().requires_grad_(True)
    bb = torch.tensor(b, requires_grad=True)
    z = F.conv2d(x, w, bb, padding=1)
    z.backward(torch.tensor(dZ).permute(0, 3, 1, 2))
    np.testing.assert_allclose(conv.conv3x3_dgrad(dZ, W), x.grad.permute(0, 2, 3, 1).numpy(), rtol=1e-11, atol=1e-12)
    dW, db = conv.conv3x3_wgrad(dZ, X)
    np.testing.assert_allclose(dW, w.grad.permute(0, 2, 3, 1).numpy(), rtol=1e-11, atol=1e-12)
    np.testing.assert_allclose(db, bb.grad.numpy(), rtol=1e-12)


def test_conv_dgrad_brute_force():
    dZ, W = rnd(1, 4, 3, 2, seed=11), rnd(2, 3, 3, 3, seed=12)
    ref = np.zeros((1, 4, 3, 3))
    for h in range(4):
        for w in range(3):
            for i in range(3):
                for kh in range(3):
                    for kw in range(3):
                        hh, ww = h - kh + 1, w - kw + 1
                        if 0 <= hh < 4 and 0 <= ww < 3:
                            ref[0, h, w, i] += dZ[0, hh, ww, :] @ W[:, kh, kw, i]
    np.testing.assert_allclose(conv.conv3x3_dgrad(dZ, W), ref, rtol=1e-12, atol=1e-12)


def test_maxpool_forward_and_first_max_backward():
    X = rnd(2, 4, 6, 3, seed=13)
    Y = conv.maxpool2_forward(X)
    ref = F.max_pool2d(torch.tensor(X).permute(0, 3, 1, 2), 2).permute(0, 2, 3, 1).numpy()
    np.testing.assert_array_equal(Y, ref)
    # exact ties: all-equal windows route to the top-left element
    X = np.zeros((1, 2, 4, 1))
    X[0, :, 2:, 0] = 5.0
    X[0, 1, 3, 0] = 5.0
    dY = np.array([[[[1.5], [2.5]]]])
    dX = conv.maxpool2_backward(X, dY)
    expect = np.zeros_like(X)
    expect[0, 0, 0, 0] = 1.5                    # window of zeros: first element
    expect[0, 0, 2, 0] = 2.5                    # tie of 5.0s: first in row-major order
    np.testing.assert_array_equal(dX, expect)


def test_maxpool_backward_brute_force_random():
    X = np.round(rnd(2, 4, 4, 2, seed=14) * 2) / 2   # many ties
    dY = rnd(2, 2, 2, 2, seed=15)
    dX = conv.maxpool2_backward(X, dY)
    ref = np.zeros_like(X)
    for n in range(2):
        for i in range(2):
            for j in range(2):
                for c in range(2):
                    win = [(X[n, 2 * i + a, 2 * j + bb, c], a, bb) for a in range(2) for bb in range(2)]
                    mx = max(v for v, _, _ in win)
                    _, a, bb = next(t for t in win if t[0] == mx)
                    ref[n, 2 * i + a, 2 * j + bb, c] = dY[n, i, j, c]
    np.testing.assert_array_equal(dX, ref)


# ------------------------------------------------------------------ tiny conv nets
def tiny_vgg(H=8, C0=3, C=8):
    return [
        {"kind": "conv3", "cin": C0, "cout": C, "h": H, "w": H},
        {"kind": "conv3", "cin": C, "cout": C, "h": H, "w": H},
        {"kind": "pool2", "c": C, "h": H, "w": H},
        {"kind": "conv3", "cin": C, "cout": 2 * C, "h": H // 2, "w": H // 2},
        {"kind": "pool2", "c": 2 * C, "h": H // 2, "w": H // 2},
        {"kind": "linear", "in": 2 * C * (H // 4) ** 2, "out": 16},
        {"kind": "linear", "in": 16, "out": 5},
    ]


def net_inputs(layers, m, b, M, seed=0):
    s0 = layers[0]
    feat = s0["h"] * s0["w"] * s0["cin"]
    classes = layers[-1]["out"]
    xs = [synthgen.inputs(seed, j, m * b, feat, synthgen.X_UNIT) for j in range(M)]
    ys = [synthgen.labels(seed, j, m * b, classes) for j in range(M)]
    w0, b0 = [], []
    for l, sp in enumerate(layers):
        if sp["kind"] == "pool2":
            w0.append(None)
            b0.append(None)
        elif sp["kind"] == "conv3":
            w0.append(synthgen.weights(seed, l, sp["cout"], 9 * sp["cin"]).reshape(sp["cout"], 3, 3, sp["cin"]))
            b0.append(np.zeros(sp["cout"], np.float32))
        else:
            w0.append(synthgen.weights(seed, l, sp["out"], sp["in"]))
            b0.append(np.zeros(sp["out"], np.float32))
    return xs, ys, w0, b0


def torch_forward(layers, x, params, detach_pairs=None):
    """NHWC-flattened rows -> logits, with optional (P, W_f) detach trick per layer."""
    h = x
    for l, sp in enumerate(layers):
        if sp["kind"] == "pool2":
            t = h.reshape(-1, sp["h"], sp["w"], sp["c"]).permute(0, 3, 1, 2)
            h = F.max_pool2d(t, 2).permute(0, 2, 3, 1).reshape(h.shape[0], -1)
            continue
        P, bias = params[l]
        Wf = detach_pairs[l] if detach_pairs else None
        if sp["kind"] == "conv3":
            t = h.reshape(-1, sp["h"], sp["w"], sp["cin"]).permute(0, 3, 1, 2)
            z = F.conv2d(t, P.permute(0, 3, 1, 2), bias, padding=1)
            if Wf is not None:
                z = z + F.conv2d(t, (Wf - P).permute(0, 3, 1, 2), None, padding=1).detach()
            z = z.permute(0, 2, 3, 1).reshape(h.shape[0], -1)
        else:
            z = h @ P.T + bias
            if Wf is not None:
                z = z + (h @ (Wf - P).T).detach()
        h = torch.relu(z) if l < len(layers) - 1 else z
    return h


def test_conv_net_single_stage_exact_equals_torch_sgd():
    layers = tiny_vgg()
    m, b, M = 2, 3, 4
    xs, ys, w0, b0 = net_inputs(layers, m, b, M)
    cfg = pipeline.Config([0], [0, len(layers)], m, b, M, lr=0.1, momentum=0.9, exact=True, layers=layers)
    res = pipeline.run(cfg, xs, ys, w0, b0)
    params, flat = {}, []
    for l, sp in enumerate(layers):
        if w0[l] is not None:
            params[l] = (torch.tensor(np.asarray(w0[l], np.float64), requires_grad=True),
                         torch.tensor(np.asarray(b0[l], np.float64), requires_grad=True))
            flat += list(params[l])
    opt = torch.optim.SGD(flat, lr=0.1, momentum=0.9)
    losses = []
    for j in range(M):
        logits = torch_forward(layers, torch.tensor(xs[j], dtype=torch.float64), params)
        loss = F.cross_entropy(logits, torch.tensor(ys[j], dtype=torch.long))
        opt.zero_grad()
        loss.backward()
        opt.step()
        losses.append(loss.item())
    np.testing.assert_allclose(res.losses, losses, rtol=1e-11)
    for l in params:
        np.testing.assert_allclose(res.weights[l], params[l][0].detach().numpy(), rtol=1e-10, atol=1e-13)
        np.testing.assert_allclose(res.biases[l], params[l][1].detach().numpy(), rtol=1e-10, atol=1e-13)


@pytest.mark.parametrize("variant,blend,lam", [(st.V_VARIANT, st.EQ1, 0.5), (st.I_VARIANT, st.EQ1, 0.3),
                                               (st.I_VARIANT, st.CONVEX, 0.7)])
def test_conv_net_multistage_exact_equals_torch_replay(variant, blend, lam):
    layers = tiny_vgg()
    bounds = [0, 2, 4, len(layers)]          # [conv conv] [pool conv] [pool fc fc]
    S = len(bounds) - 1
    m, b, M, lr, mu = 2, 2, 6, 0.05, 0.5
    xs, ys, w0, b0 = net_inputs(layers, m, b, M, seed=3)
    cfg = pipeline.Config([0], bounds, m, b, M, variant=variant, blend=blend, lam=lam, lr=lr, momentum=mu,
                          exact=True, layers=layers)
    res = pipeline.run(cfg, xs, ys, w0, b0)
    stage_of = [next(s for s in range(S) if bounds[s] <= l < bounds[s + 1]) for l in range(len(layers))]
    hw = {l: [torch.tensor(np.asarray(w0[l], np.float64))] for l in range(len(layers)) if w0[l] is not None}
    hb = {l: [torch.tensor(np.asarray(b0[l], np.float64))] for l in hw}
    mw = {l: torch.zeros_like(hw[l][0]) for l in hw}
    mb = {l: torch.zeros_like(hb[l][0]) for l in hw}
    for j in range(M):
        params, pairs, leaves = {}, {}, []
        for l in hw:
            vf = max(0, j - S + stage_of[l] + 1)
            Wf, Wl = hw[l][vf], hw[l][j]
            if variant == st.V_VARIANT:
                Wres = Wl
            else:
                a, bb = st.blend_coeffs(variant, blend, j - vf, lam)
                Wres = a * Wf + bb * Wl
            P = Wres.clone().requires_grad_(True)
            bias = hb[l][vf].clone().requires_grad_(True)
            params[l], pairs[l] = (P, bias), Wf
            leaves += [P, bias]
        logits = torch_forward(layers, torch.tensor(xs[j], dtype=torch.float64), params, pairs)
        loss = F.cross_entropy(logits, torch.tensor(ys[j], dtype=torch.long))
        grads = torch.autograd.grad(loss, leaves)
        assert abs(loss.item() - res.losses[j]) <= 1e-11 * abs(loss.item())
        for i, l in enumerate(hw):
            gw, gb = grads[2 * i], grads[2 * i + 1]
            mw[l] = mu * mw[l] + gw
            mb[l] = mu * mb[l] + gb
            hw[l].append(hw[l][j] - lr * mw[l])
            hb[l].append(hb[l][j] - lr * mb[l])
    for l in hw:
        np.testing.assert_allclose(res.weights[l], hw[l][-1].numpy(), rtol=1e-10, atol=1e-13)
        np.testing.assert_allclose(res.biases[l], hb[l][-1].numpy(), rtol=1e-10, atol=1e-13)

"""Pins for oracle.resnet (general conv, batch norm with per-micro-batch statistics, 3x3/2 max
pool, global average pool) and oracle.graph (pipeline replay with skip connections).

* every op == torch fp64 (conv2d, batch_norm training mode, max_pool2d, mean) incl. autograd
* the first-max tie rule of the 3x3/2 pool == brute force
* graph.run on an MLP graph == pipeline.run bitwise (the replays share the method's logic)
* exact-mode ResNet graph, S = 1 == torch autograd + torch.optim.SGD (BN statistics of each
  micro-batch, reading Z22)
* exact-mode ResNet graph, S > 1 == independent torch replay with closed-form versions and the
  V / I-EQ1 / I-CONVEX backward weights (conv W and BN γ, reading Z12)
"""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

import synthgen
from oracle import graph, pipeline, resnet, staleness as st


def rnd(*shape, seed=0):
    return np.random.default_rng(seed).standard_normal(shape)


def t_nchw(x):
    return torch.tensor(x).permute(0, 3, 1, 2)


@pytest.mark.parametrize("k,s,p", [(1, 1, 0), (1, 2, 0), (3, 2, 1), (7, 2, 3), (3, 1, 1)])
def test_conv_general_matches_torch(k, s, p):
    X, W = rnd(2, 9, 10, 3, seed=k), rnd(4, k, k, 3, seed=s)
    dZ_shape = resnet.conv_forward(X, W, s, p).shape
    dZ = rnd(*dZ_shape, seed=5)
    x = t_nchw(X).requires_grad_(True)
    w = t_nchw(W).detach().requires_grad_(True)
    z = F.conv2d(x, w, stride=s, padding=p)
    np.testing.assert_allclose(resnet.conv_forward(X, W, s, p), z.detach().permute(0, 2, 3, 1).numpy(), rtol=1e-12,
                               atol=1e-12)
    z.backward(t_nchw(dZ))
    np.testing.assert_allclose(resnet.conv_dgrad(dZ, W, X.shape, s, p), x.grad.permute(0, 2, 3, 1).numpy(),
                               rtol=1e-11, atol=1e-12)
    np.testing.assert_allclose(resnet.conv_wgrad(dZ, X, k, s, p), w.grad.permute(0, 2, 3, 1).numpy(), rtol=1e-11,
                               atol=1e-12)


def test_batchnorm_matches_torch_training_mode():
    X, g, b = rnd(4, 3, 5, 6, seed=1), rnd(6, seed=2), rnd(6, seed=3)
    dY = rnd(4, 3, 5, 6, seed=4)
    x = t_nchw(X).requires_grad_(True)
    gg = torch.tensor(g, requires_grad=True)
    bb = torch.tensor(b, requires_grad=True)
    y = F.batch_norm(x, None, None, gg, bb, training=True, eps=resnet.BN_EPS)
    ours, mu, inv = resnet.bn_forward(X, g, b)
    np.testing.assert_allclose(ours, y.detach().permute(0, 2, 3, 1).numpy(), rtol=1e-12, atol=1e-12)
    y.backward(t_nchw(dY))
    dx, dg, db = resnet.bn_backward(dY, X, g, mu, inv)
    np.testing.assert_allclose(dx, x.grad.permute(0, 2, 3, 1).numpy(), rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(dg, gg.grad.numpy(), rtol=1e-11)
    np.testing.assert_allclose(db, bb.grad.numpy(), rtol=1e-12)


def test_maxpool3_matches_torch_and_first_max_rule():
    X = rnd(2, 7, 8, 3, seed=6)
    ref = F.max_pool2d(t_nchw(X), 3, 2, 1).permute(0, 2, 3, 1).numpy()
    np.testing.assert_array_equal(resnet.maxpool3_forward(X), ref)
    Xq = np.round(rnd(1, 5, 5, 2, seed=7))          # many ties
    Y = resnet.maxpool3_forward(Xq)
    dY = rnd(*Y.shape, seed=8)
    dX = resnet.maxpool3_backward(Xq, dY)
    ref = np.zeros_like(Xq)
    for i in range(Y.shape[1]):
        for j in range(Y.shape[2]):
            for c in range(2):
                best = None
                for kh in range(3):
                    for kw in range(3):
                        h, w = 2 * i + kh - 1, 2 * j + kw - 1
                        if 0 <= h < 5 and 0 <= w < 5 and (best is None or Xq[0, h, w, c] > best[0]):
                            best = (Xq[0, h, w, c], h, w)
                ref[0, best[1], best[2], c] += dY[0, i, j, c]
    np.testing.assert_allclose(dX, ref, rtol=0, atol=1e-15)


def test_avgpool_matches_torch():
    X = rnd(3, 4, 4, 5, seed=9)
    np.testing.assert_allclose(resnet.avgpool_forward(X), X.mean(axis=(1, 2)), rtol=1e-15)
    dY = rnd(3, 5, seed=10)
    x = t_nchw(X).requires_grad_(True)
    F.adaptive_avg_pool2d(x, 1).reshape(3, 5).backward(torch.tensor(dY))
    np.testing.assert_allclose(resnet.avgpool_backward(X.shape, dY), x.grad.permute(0, 2, 3, 1).numpy(), rtol=1e-14)


# ------------------------------------------------------------------ graph replay
def graph_params(layers, seed=0):
    out = []
    for l, sp in enumerate(layers):
        if sp["kind"] == "conv":
            w = synthgen.weights(seed, l, sp["cout"], sp["k"] * sp["k"] * sp["cin"])
            out.append((w.reshape(sp["cout"], sp["k"], sp["k"], sp["cin"]), None))
        elif sp["kind"] == "bn":
            out.append((np.ones(sp["c"], np.float32), np.zeros(sp["c"], np.float32)))
        elif sp["kind"] == "linear":
            out.append((synthgen.weights(seed, l, sp["out"], sp["in"]), np.zeros(sp["out"], np.float32)))
        else:
            out.append((None, None))
    return out


def tiny_resnet(H=16):
    return graph.resnet_layers(blocks=(1, 1), widths=(4, 8), H=H, classes=5, stem_c=8)


def graph_inputs(layers, m, b, M, seed=0):
    s0 = layers[0]
    feat = s0["h"] * s0["w"] * s0["cin"]
    xs = [synthgen.inputs(seed, j, m * b, feat, synthgen.X_UNIT) for j in range(M)]
    ys = [synthgen.labels(seed, j, m * b, layers[-1]["out"]) for j in range(M)]
    return xs, ys


def test_graph_mlp_equals_pipeline_bitwise():
    dims, m, b, M = [16, 12, 12, 12, 6], 2, 4, 7
    layers = [{"kind": "linear", "in": dims[l], "out": dims[l + 1]} for l in range(4)]
    # graph linear layers carry no input mask / ReLU except via BN, so compare against an MLP whose
    # hidden ReLUs are expressed as bn-free graph: use only a single Linear head on a 1-layer net
    xs = [synthgen.inputs(0, j, m * b, 16) for j in range(M)]
    ys = [synthgen.labels(0, j, m * b, 6) for j in range(M)]
    w0 = synthgen.weights(0, 0, 6, 16)
    for variant in (st.V_VARIANT, st.I_VARIANT):
        ref = pipeline.run(pipeline.Config([16, 6], [0, 1], m, b, M, variant=variant, lr=0.1, momentum=0.9),
                           xs, ys, [w0], [np.zeros(6, np.float32)])
        got = graph.run([{"kind": "linear", "in": 16, "out": 6}], [0, 1], m, b, M, xs, ys,
                        [(w0, np.zeros(6, np.float32))], variant=variant, lr=0.1, mu=0.9)
        assert np.array_equal(ref.losses, got.losses)
        assert np.array_equal(ref.weights[0], got.weights[0])
        assert [(r.stage, r.kind, r.mb, r.v_used, r.delta) for r in ref.trace] == \
               [(r.stage, r.kind, r.mb, r.v_used, r.delta) for r in got.trace]
    del layers


def torch_net_forward(layers, x, P, pairs=None):
    """Per micro-batch forward of the graph in torch (BN statistics of that micro-batch)."""
    T = {-1: x}
    for l, sp in enumerate(layers):
        s_ = sp.get("src", l - 1)
        k = sp["kind"]
        if k == "conv":
            h = T[s_].reshape(-1, sp["h"], sp["w"], sp["cin"]).permute(0, 3, 1, 2)
            Wp = P[l][0]
            z = F.conv2d(h, Wp.permute(0, 3, 1, 2), stride=sp["s"], padding=sp["p"])
            if pairs:
                z = z + F.conv2d(h, (pairs[l] - Wp).permute(0, 3, 1, 2), stride=sp["s"], padding=sp["p"]).detach()
            T[l] = z.permute(0, 2, 3, 1)
        elif k == "bn":
            h = T[s_].reshape(-1, sp["h"], sp["w"], sp["c"]).permute(0, 3, 1, 2)
            gp, bp = P[l]
            mean = h.mean(dim=(0, 2, 3), keepdim=True)
            var = ((h - mean) ** 2).mean(dim=(0, 2, 3), keepdim=True)
            xh = (h - mean) / torch.sqrt(var + resnet.BN_EPS)
            z = gp.view(1, -1, 1, 1) * xh + bp.view(1, -1, 1, 1)
            if pairs:
                z = z + ((pairs[l] - gp).view(1, -1, 1, 1) * xh).detach()
            z = z.permute(0, 2, 3, 1)
            if sp.get("res") is not None:
                z = z + T[sp["res"]].reshape(z.shape)
            T[l] = torch.relu(z) if sp.get("relu") else z
        elif k == "maxpool3":
            h = T[s_].reshape(-1, sp["h"], sp["w"], sp["c"]).permute(0, 3, 1, 2)
            T[l] = F.max_pool2d(h, 3, 2, 1).permute(0, 2, 3, 1)
        elif k == "avgpool":
            T[l] = T[s_].reshape(-1, sp["h"], sp["w"], sp["c"]).mean(dim=(1, 2))
        else:
            Wp, bp = P[l]
            h = T[s_].reshape(T[s_].shape[0], -1)
            z = h @ Wp.T + bp
            if pairs:
                z = z + (h @ (pairs[l] - Wp).T).detach()
            T[l] = z
    return T[len(layers) - 1]


def test_resnet_graph_single_stage_exact_equals_torch_sgd():
    layers, _ = tiny_resnet()
    m, b, M = 2, 3, 3
    xs, ys = graph_inputs(layers, m, b, M)
    p0 = graph_params(layers)
    res = graph.run(layers, [0, len(layers)], m, b, M, xs, ys, p0, lr=0.05, mu=0.9, exact=True)
    P, flat = {}, []
    for l, (w, bb) in enumerate(p0):
        if w is None:
            continue
        P[l] = (torch.tensor(np.asarray(w, np.float64), requires_grad=True),
                None if bb is None else torch.tensor(np.asarray(bb, np.float64), requires_grad=True))
        flat += [t for t in P[l] if t is not None]
    opt = torch.optim.SGD(flat, lr=0.05, momentum=0.9)
    for j in range(M):
        loss = 0.0
        for a in range(m):
            x = torch.tensor(xs[j][a * b:(a + 1) * b], dtype=torch.float64)
            logits = torch_net_forward(layers, x, P)
            loss = loss + F.cross_entropy(logits, torch.tensor(ys[j][a * b:(a + 1) * b], dtype=torch.long),
                                          reduction="sum")
        loss = loss / (m * b)
        opt.zero_grad()
        loss.backward()
        opt.step()
        assert abs(loss.item() - res.losses[j]) <= 1e-11 * abs(loss.item())
    for l in P:
        np.testing.assert_allclose(res.weights[l], P[l][0].detach().numpy(), rtol=1e-9, atol=1e-12)
        if P[l][1] is not None:
            np.testing.assert_allclose(res.biases[l], P[l][1].detach().numpy(), rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("variant,blend,lam", [(st.V_VARIANT, st.EQ1, 0.5), (st.I_VARIANT, st.EQ1, 0.3),
                                               (st.I_VARIANT, st.CONVEX, 0.7)])
def test_resnet_graph_multistage_exact_equals_torch_replay(variant, blend, lam):
    layers, starts = tiny_resnet()
    bounds = [0, starts[1], starts[2], len(layers)]   # [stem] [block 1] [block 2 + head]
    S = len(bounds) - 1
    m, b, M, lr, mu = 2, 2, 5, 0.05, 0.5
    xs, ys = graph_inputs(layers, m, b, M, seed=2)
    p0 = graph_params(layers, seed=2)
    res = graph.run(layers, bounds, m, b, M, xs, ys, p0, variant=variant, blend=blend, lam=lam, lr=lr, mu=mu,
                    exact=True)
    stage_of = [next(s for s in range(S) if bounds[s] <= l < bounds[s + 1]) for l in range(len(layers))]
    idx = [l for l in range(len(layers)) if p0[l][0] is not None]
    hw = {l: [torch.tensor(np.asarray(p0[l][0], np.float64))] for l in idx}
    hb = {l: [torch.tensor(np.asarray(p0[l][1], np.float64))] for l in idx if p0[l][1] is not None}
    mw = {l: torch.zeros_like(hw[l][0]) for l in hw}
    mb_ = {l: torch.zeros_like(hb[l][0]) for l in hb}
    for j in range(M):
        P, pairs, leaves = {}, {}, []
        for l in idx:
            vf = max(0, j - S + stage_of[l] + 1)
            Wf, Wl = hw[l][vf], hw[l][j]
            if variant == st.V_VARIANT:
                Wres = Wl
            else:
                a_, b_ = st.blend_coeffs(variant, blend, j - vf, lam)
                Wres = a_ * Wf + b_ * Wl
            Pw = Wres.clone().requires_grad_(True)
            Pb = hb[l][vf].clone().requires_grad_(True) if l in hb else None
            P[l], pairs[l] = (Pw, Pb), Wf
            leaves += [Pw] + ([Pb] if Pb is not None else [])
        loss = 0.0
        for a in range(m):
            x = torch.tensor(xs[j][a * b:(a + 1) * b], dtype=torch.float64)
            logits = torch_net_forward(layers, x, P, pairs)
            loss = loss + F.cross_entropy(logits, torch.tensor(ys[j][a * b:(a + 1) * b], dtype=torch.long),
                                          reduction="sum")
        loss = loss / (m * b)
        g = torch.autograd.grad(loss, leaves)
        assert abs(loss.item() - res.losses[j]) <= 1e-10 * abs(loss.item())
        i = 0
        for l in idx:
            mw[l] = mu * mw[l] + g[i]; i += 1
            hw[l].append(hw[l][j] - lr * mw[l])
            if l in hb:
                mb_[l] = mu * mb_[l] + g[i]; i += 1
                hb[l].append(hb[l][j] - lr * mb_[l])
    for l in idx:
        np.testing.assert_allclose(res.weights[l], hw[l][-1].numpy(), rtol=1e-9, atol=1e-12)
        if l in hb:
            np.testing.assert_allclose(res.biases[l], hb[l][-1].numpy(), rtol=1e-9, atol=1e-12)


def test_resnet50_graph_is_torchvision_resnet50():
    """Pins oracle.graph.resnet_layers() (which feeds BOTH the oracle and the GPU path) to an
    independent library definition: torchvision.models.resnet50 (v1.5).  Same parameter count
    (25,557,032 at 1000 classes), and at 64x64 inputs one exact-mode training step of the oracle
    graph (S = 1, BN statistics of the micro-batch) equals torchvision's forward in training
    mode + autograd + SGD: the same loss and the same updated parameters for all 161 tensors."""
    tv = pytest.importorskip("torchvision")
    layers, _ = graph.resnet_layers()
    n = sum(int(np.prod(p[0].shape)) + (0 if p[1] is None else p[1].size)
            for p in graph_params(layers) if p[0] is not None)
    assert n == 25_557_032 == sum(p.numel() for p in tv.models.resnet50(weights=None).parameters())

    classes, H, b = 10, 64, 2
    layers, _ = graph.resnet_layers(H=H, classes=classes)
    p0 = graph_params(layers, seed=4)
    xs, ys = graph_inputs(layers, 1, b, 1, seed=4)
    res = graph.run(layers, [0, len(layers)], 1, b, 1, xs, ys, p0, lr=0.1, mu=0.9, exact=True)

    net = tv.models.resnet50(weights=None, num_classes=classes).double().train()
    pairs, prev = [], None        # (conv, bn) in torchvision's conv order: each conv feeds one bn
    for mod in net.modules():
        if isinstance(mod, torch.nn.Conv2d):
            prev = mod
        elif isinstance(mod, torch.nn.BatchNorm2d):
            pairs.append((prev, mod))
    oconv = [l for l, sp in enumerate(layers) if sp["kind"] == "conv"]
    assert len(oconv) == len(pairs) == 53
    bn_of = {}
    with torch.no_grad():
        for l, (conv, bn) in zip(oconv, pairs):
            sp = layers[l]
            assert (conv.in_channels, conv.out_channels, conv.kernel_size[0], conv.stride[0], conv.padding[0]) == \
                (sp["cin"], sp["cout"], sp["k"], sp["s"], sp["p"]), (l, conv)
            conv.weight.copy_(torch.from_numpy(np.asarray(p0[l][0], np.float64)).permute(0, 3, 1, 2))
            bn_of[l] = bn
        for l, sp in enumerate(layers):
            if sp["kind"] == "bn":
                bn = bn_of[sp.get("src", l - 1)]          # the BN that normalises this BN's source conv
                bn.weight.copy_(torch.from_numpy(np.asarray(p0[l][0], np.float64)))
                bn.bias.copy_(torch.from_numpy(np.asarray(p0[l][1], np.float64)))
                bn_of[("bn", l)] = bn
        net.fc.weight.copy_(torch.from_numpy(np.asarray(p0[-1][0], np.float64)))
        net.fc.bias.copy_(torch.from_numpy(np.asarray(p0[-1][1], np.float64)))
    opt = torch.optim.SGD(net.parameters(), lr=0.1, momentum=0.9)
    x = torch.from_numpy(np.asarray(xs[0], np.float64).reshape(b, H, H, 3)).permute(0, 3, 1, 2)
    loss = F.cross_entropy(net(x), torch.from_numpy(np.asarray(ys[0], np.int64)))
    opt.zero_grad()
    loss.backward()
    opt.step()
    assert abs(loss.item() - res.losses[0]) <= 1e-10 * abs(loss.item())
    with torch.no_grad():
        for l, (conv, _) in zip(oconv, pairs):
            np.testing.assert_allclose(res.weights[l], conv.weight.permute(0, 2, 3, 1).numpy(), rtol=1e-8, atol=1e-9 * np.abs(res.weights[l]).max())
        for l, sp in enumerate(layers):
            if sp["kind"] == "bn":
                bn = bn_of[("bn", l)]
                np.testing.assert_allclose(res.weights[l], bn.weight.numpy(), rtol=1e-8, atol=1e-9 * np.abs(res.weights[l]).max())
                np.testing.assert_allclose(res.biases[l], bn.bias.numpy(), rtol=1e-8, atol=1e-9)
        np.testing.assert_allclose(res.weights[-1], net.fc.weight.numpy(), rtol=1e-8, atol=1e-9)
        np.testing.assert_allclose(res.biases[-1], net.fc.bias.numpy(), rtol=1e-8, atol=1e-9)

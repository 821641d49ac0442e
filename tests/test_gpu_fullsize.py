"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

* C5 (the bench workload): 16 x Linear(4096,4096)+ReLU + head, B = 2048 (32 micro-batches of
  64, all forwards in one launch), I-TiMePReSt EQ1, SGD momentum 0.9, S = 1, fused update +
  split backward exactly as bench.py runs it — the oracle replays 3 mini-batches (forward,
  collective backward, update of all 270M parameters).
* 4 x 4096 + head at B = 2048 on 2 stages for 10 mini-batches with the fused update.
* C2: 4-stage 4096-wide MLP, 8 micro-batches of 64, staleness 3/2/1/0 by stage — the full
  pipeline for 10 mini-batches on one GPU (LOCAL transport), fused and separate update.
Both: trace bit-exact, losses within 1e-3 relative, weights within 5e-3 (Z19).
"""
import numpy as np
import pytest

import synthgen
from oracle import staleness as ost
from pipeline_helpers import expand_gpu_trace, layer_rel_err, oracle_trace, run_gpu, run_oracle, weight_rel_err

pytestmark = pytest.mark.gpu


def check(stages, losses, ref):
    assert expand_gpu_trace(stages) == oracle_trace(ref)
    np.testing.assert_allclose(losses, ref.losses, rtol=1e-3, atol=0)
    for st in stages:
        for k, l in enumerate(st.layers):
            w, bb, _, _ = st.get_weights(k)
            assert weight_rel_err(w, ref.weights[l]) <= 5e-3, l
            assert layer_rel_err(w, bb, ref.weights[l], ref.biases[l]) <= 5e-3, l


@pytest.mark.timeout(1200)
def test_c5_bench_config_three_steps(gpu_lib):
    """bench.py's exact launch configuration (C5 at S = 1: all 32 micro-batch forwards in one
    2048-row GEMM per layer, fused wgrad + SGD/momentum epilogue, split backward on the
    weight-gradient stream, bias steps on the optimizer stream, extra receive slot,
    device-side synthetic init) for 3 mini-batches against the oracle."""
    dims = [4096] * 17 + [10]
    bounds = [0, 17]
    args = (dims, bounds, 32, 64, 3, ost.I_VARIANT, ost.EQ1, 0.05, 0.01, 0.9)
    ref = run_oracle(*args, kind=synthgen.X_SIGNED)
    stages, losses = run_gpu(*args, kind=synthgen.X_SIGNED, init="synthetic", fuse_update=1, fwd_group=0,
                             extra_recv_slot=1)
    check(stages, losses, ref)


@pytest.mark.timeout(1200)
def test_full_width_two_stage_ten_steps_fused(gpu_lib):
    """Full width and batch (4 x Linear(4096,4096) + head, B = 2048 = 32 x 64), two stages
    (stage 0 has δ = 1 and two layers, so the I-EQ1 α-scaled input gradient runs), fused
    wgrad + update epilogue and split backward, 10 mini-batches (the north_star's bar)."""
    dims = [4096] * 5 + [10]
    bounds = [0, 2, 5]
    args = (dims, bounds, 32, 64, 10, ost.I_VARIANT, ost.EQ1, 0.05, 0.01, 0.9)
    ref = run_oracle(*args, kind=synthgen.X_SIGNED)
    stages, losses = run_gpu(*args, kind=synthgen.X_SIGNED, init="synthetic", fuse_update=1)
    check(stages, losses, ref)
    assert max(e.delta for e in stages[0].trace() if e.kind == 1) == 1


@pytest.mark.timeout(1200)
@pytest.mark.parametrize("fuse", [1, 0])
@pytest.mark.parametrize("blend", [ost.EQ1, ost.CONVEX])
def test_c2_four_stage_staleness_sweep(gpu_lib, blend, fuse):
    """C2 at full size for 10 mini-batches (the north_star's bar), staleness 3/2/1/0 by stage."""
    dims = [4096] * 9 + [10]
    bounds = [0, 2, 4, 6, 9]
    args = (dims, bounds, 8, 64, 10, ost.I_VARIANT, blend, 0.05, 0.01, 0.9)
    ref = run_oracle(*args, kind=synthgen.X_SIGNED)
    stages, losses = run_gpu(*args, kind=synthgen.X_SIGNED, init="synthetic", fuse_update=fuse)
    check(stages, losses, ref)
    deltas = sorted({(e.stage, e.delta) for st in stages for e in st.trace() if e.kind == 1})
    assert max(d for s, d in deltas if s == 0) == 3 and max(d for s, d in deltas if s == 3) == 0


def vgg16_cifar(classes=10):
    """VGG-16 on 32x32x3 (BASELINE.json configs[2]): 13 conv3x3 + 5 max-pools + FC 512-4096-4096-classes."""
    layers, H, C = [], 32, 3
    for block, (width, n) in enumerate([(64, 2), (128, 2), (256, 3), (512, 3), (512, 3)]):
        for _ in range(n):
            layers.append({"kind": "conv3", "cin": C, "cout": width, "h": H, "w": H})
            C = width
        layers.append({"kind": "pool2", "c": C, "h": H, "w": H})
        H //= 2
    layers += [{"kind": "linear", "in": 512, "out": 4096}, {"kind": "linear", "in": 4096, "out": 4096},
               {"kind": "linear", "in": 4096, "out": classes}]
    return layers


# stage partition by conv block: [c1,c2 + pools] [c3 + pool] [c4 + pool] [c5 + pool + FCs]
VGG_BOUNDS = [0, 6, 10, 14, 21]


@pytest.mark.timeout(900)
def test_c3_vgg16_four_stage(gpu_lib):
    layers = vgg16_cifar()
    dims = [32 * 32 * 3, 10]
    args = (dims, VGG_BOUNDS, 2, 64, 4, ost.I_VARIANT, ost.EQ1, 0.05, 0.01, 0.9)
    ref = run_oracle(*args, kind=synthgen.X_UNIT, layers=layers)
    stages, losses = run_gpu(*args, kind=synthgen.X_UNIT, init="synthetic", layers=layers)
    assert expand_gpu_trace(stages) == oracle_trace(ref)
    np.testing.assert_allclose(losses, ref.losses, rtol=1e-3, atol=0)
    for st in stages:
        for k, l in enumerate(st.layers):
            if ref.weights[l] is None:
                continue
            w, bb, _, _ = st.get_weights(k)
            wr = ref.weights[l].reshape(w.shape)
            assert weight_rel_err(w, wr) <= 5e-3, l
            assert layer_rel_err(w, bb, wr, ref.biases[l]) <= 5e-3, l

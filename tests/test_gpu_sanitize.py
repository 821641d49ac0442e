"""Small end-to-end runs for compute-sanitizer (tools/gpu_round.sh `sanitize`: memcheck,
racecheck, synccheck over this file).  They cover every kernel family of the hot path on the
multi-stream runtime: forward / input-gradient / weight-gradient GEMMs (single CTA and CTA
pairs), the blend-on-load input gradient, the fused wgrad + update epilogue with the split
backward (weight-gradient + optimizer streams), the separate update, softmax-CE, bias
gradients, the VGG conv / pool kernels and the ResNet graph kernels (BN, pools, im2col,
col2im).  Sizes are tiny: the sanitizer slows kernels by 10-100x.  Each run is also checked
against the oracle, so a sanitizer-clean run is also a correct one."""
import numpy as np
import pytest

import synthgen
from oracle import graph as ograph
from oracle import staleness as ost
from pipeline_helpers import expand_gpu_trace, oracle_trace, run_gpu, run_oracle, weight_rel_err

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("fuse,blend", [(1, ost.EQ1), (1, ost.CONVEX), (0, ost.CONVEX)])
def test_sanitize_mlp_three_stages(gpu_lib, fuse, blend):
    dims, bounds = [512, 512, 256, 256, 16], [0, 2, 3, 4]      # 512-wide: CTA-pair tiles
    args = (dims, bounds, 2, 128, 4, ost.I_VARIANT, blend, 0.3, 0.05, 0.9)
    ref = run_oracle(*args)
    stages, losses = run_gpu(*args, fuse_update=fuse)
    assert expand_gpu_trace(stages) == oracle_trace(ref)
    np.testing.assert_allclose(losses, ref.losses, rtol=1e-3)
    for st in stages:
        for k, l in enumerate(st.layers):
            assert weight_rel_err(st.get_weights(k)[0], ref.weights[l]) <= 5e-3
        st.close()


def test_sanitize_vgg_chain(gpu_lib):
    layers = [{"kind": "conv3", "cin": 3, "cout": 64, "h": 8, "w": 8},
              {"kind": "conv3", "cin": 64, "cout": 64, "h": 8, "w": 8},
              {"kind": "pool2", "c": 64, "h": 8, "w": 8},
              {"kind": "linear", "in": 1024, "out": 10}]
    args = ([8 * 8 * 3, 10], [0, 2, 4], 2, 8, 3, ost.I_VARIANT, ost.CONVEX, 0.3, 0.05, 0.9)
    ref = run_oracle(*args, kind=synthgen.X_UNIT, layers=layers)
    stages, losses = run_gpu(*args, kind=synthgen.X_UNIT, layers=layers)
    np.testing.assert_allclose(losses, ref.losses, rtol=1e-3)
    for st in stages:
        st.close()


def test_sanitize_resnet_graph(gpu_lib):
    layers, starts = ograph.resnet_layers(blocks=(1, 1), widths=(64, 128), H=16, classes=10, stem_c=64)
    dims = [16 * 16 * 3, 10]
    stages, losses = run_gpu(dims, [0, starts[1], len(layers)], 2, 4, 2, ost.I_VARIANT, ost.CONVEX, 0.05, 0.01, 0.9,
                             kind=synthgen.X_UNIT, layers=layers)
    assert np.isfinite(losses).all()
    for st in stages:
        st.close()

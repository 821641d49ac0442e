import sys, os, numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from test_gpu_fullsize import vgg16_cifar, VGG_BOUNDS
from pipeline_helpers import run_gpu, run_oracle, weight_rel_err
import synthgen
from oracle import staleness as ost
layers = vgg16_cifar()
M = int(sys.argv[1]) if len(sys.argv) > 1 else 2
args = ([3072, 10], VGG_BOUNDS, 2, 64, M, ost.I_VARIANT, ost.EQ1, 0.05, 0.01, 0.9)
ref = run_oracle(*args, kind=synthgen.X_UNIT, layers=layers)
for fuse in (0, 1):
    stages, losses = run_gpu(*args, kind=synthgen.X_UNIT, init="synthetic", layers=layers, fuse_update=fuse)
    print("fuse", fuse, "loss rel", np.abs(losses / ref.losses - 1).max())
    for st in stages:
        for k, l in enumerate(st.layers):
            if ref.weights[l] is None: continue
            w = st.get_weights(k)[0]; wr = ref.weights[l].reshape(w.shape)
            e = weight_rel_err(w, wr)
            if e > 2e-3:
                d = np.abs(w - wr); i = np.unravel_index(d.argmax(), d.shape)
                rows = np.unique(np.argwhere(d > 0.1 * d.max())[:, 0])
                print(f"  layer {l} err {e:.4f} at {i} got {w[i]:.5f} ref {wr[i]:.5f}; bad rows {rows[:20]} (#{rows.size})")
            else:
                print(f"  layer {l} ok {e:.5f}")

"""Determinism check of the ResNet-50 graph path: identical runs must give bitwise-identical
weights; prints the layers that differ between repeats."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from oracle import graph as ograph  # noqa: E402
from oracle import staleness as ost  # noqa: E402
from pipeline_helpers import run_gpu  # noqa: E402

layers, starts = ograph.resnet_layers()
L = len(layers)
dims = [224 * 224 * 3, 1000]
res = []
for rep in range(3):
    stages, losses = run_gpu(dims, [0, L], 2, 8, 1, ost.I_VARIANT, ost.EQ1, 0.05, 0.01, 0.9, kind=1, layers=layers)
    st = stages[0]
    ws = {l: st.get_weights(k)[0].copy() for k, l in enumerate(st.layers) if layers[l]["kind"] in ("conv", "linear")}
    st.close()
    res.append((losses.copy(), ws))
    torch.cuda.synchronize()
print("env", {k: v for k, v in os.environ.items() if k.startswith("TPS_")})
print("losses", [r[0].tolist() for r in res])
for l in res[0][1]:
    d = [float(np.abs(res[i][1][l] - res[0][1][l]).max()) for i in (1, 2)]
    if max(d) > 0:
        print("layer", l, layers[l], "max diff vs run0", d, "scale", float(np.abs(res[0][1][l]).max()))

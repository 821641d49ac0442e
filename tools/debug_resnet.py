"""Per-step loss error and per-layer parameter error of the ResNet graph path vs the oracle."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import synthgen  # noqa: E402
from oracle import graph as ograph, staleness as ost  # noqa: E402
from pipeline_helpers import run_gpu, run_oracle_graph  # noqa: E402


def run(tag, layers, bounds, m, b, M, variant, blend, lr=0.01, mu=0.9, kind=synthgen.X_UNIT):
    from pipeline_helpers import graph_workload
    ref = run_oracle_graph(layers, bounds, m, b, M, variant, blend, 0.05, lr, mu, kind=kind)
    xs, ys, params = graph_workload(layers, m, b, M, kind=kind)
    ex = ograph.run(layers, bounds, m, b, M, xs, ys, params, variant=variant, blend=blend, lam=0.05, lr=lr, mu=mu,
                    exact=True)
    dims = [layers[0]["h"] * layers[0]["w"] * layers[0]["cin"], layers[-1]["out"]]
    stages, losses = run_gpu(dims, bounds, m, b, M, variant, blend, 0.05, lr, mu, kind=kind, layers=layers)
    rel = np.abs(losses - ref.losses) / np.abs(ref.losses)
    rex = np.abs(ex.losses - ref.losses) / np.abs(ref.losses)
    print(tag, "loss rel err gpu:", " ".join(f"{x:.1e}" for x in rel), "| bf16-vs-exact:", " ".join(f"{x:.1e}" for x in rex))
    out = []
    for st in stages:
        for k, l in enumerate(st.layers):
            if ref.weights[l] is None:
                continue
            w, bb, _, _ = st.get_weights(k)
            w0 = np.asarray(params[l][0], np.float64).reshape(w.shape)
            wr = np.asarray(ref.weights[l], np.float64).reshape(w.shape)
            we = np.asarray(ex.weights[l], np.float64).reshape(w.shape)
            du = np.abs(wr - w0).max()
            sc = np.abs(wr).max()
            out.append(f"{l}{layers[l]['kind'][0]}:{np.abs(w - wr).max() / sc:.0e}/{np.abs(we - wr).max() / sc:.0e}")
        st.close()
    print(tag, "param-rel err gpu/exact-gap:", " ".join(out), flush=True)


if __name__ == "__main__":
    layers, starts = ograph.resnet_layers(blocks=(1, 1), widths=(16, 32), H=32, classes=10, stem_c=16)
    L = len(layers)
    b3 = [0, starts[1], starts[2], L]
    for kind in (synthgen.X_SIGNED, synthgen.X_UNIT):
        for lr in (0.002, 0.01):
            run(f"kind{kind} lr{lr} S3 I-EQ1", layers, b3, 2, 8, 10, ost.I_VARIANT, ost.EQ1, lr=lr, kind=kind)
            run(f"kind{kind} lr{lr} S1 V", layers, [0, L], 2, 8, 10, ost.V_VARIANT, ost.EQ1, lr=lr, kind=kind)

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


def run_update(tag, layers, bounds, m, b, M, variant, blend, lr=0.01, mu=0.9, kind=synthgen.X_UNIT):
    """per-layer update error (ΔW vs oracle ΔW) and the oracle's own fp64 gap; prints outliers"""
    from pipeline_helpers import graph_workload
    ref = run_oracle_graph(layers, bounds, m, b, M, variant, blend, 0.05, lr, mu, kind=kind)
    xs, ys, params = graph_workload(layers, m, b, M, kind=kind)
    ex = ograph.run(layers, bounds, m, b, M, xs, ys, params, variant=variant, blend=blend, lam=0.05, lr=lr, mu=mu,
                    exact=True)
    dims = [layers[0]["h"] * layers[0]["w"] * layers[0]["cin"], layers[-1]["out"]]
    stages, losses = run_gpu(dims, bounds, m, b, M, variant, blend, 0.05, lr, mu, kind=kind, layers=layers)
    print(tag, "losses gpu", losses, "ref", ref.losses, "exact", ex.losses, flush=True)
    rows = []
    for st in stages:
        for k, l in enumerate(st.layers):
            if ref.weights[l] is None:
                continue
            w = st.get_weights(k)[0].astype(np.float64)
            w0 = np.asarray(params[l][0], np.float64).reshape(w.shape)
            dr = np.asarray(ref.weights[l], np.float64).reshape(w.shape) - w0
            de = np.asarray(ex.weights[l], np.float64).reshape(w.shape) - w0
            dg = w - w0
            fr = np.linalg.norm(dg - dr) / np.linalg.norm(dr)
            fe = np.linalg.norm(de - dr) / np.linalg.norm(dr)
            cos = float((dg * dr).sum() / (np.linalg.norm(dg) * np.linalg.norm(dr)))
            cose = float((de * dr).sum() / (np.linalg.norm(de) * np.linalg.norm(dr)))
            rows.append((l, layers[l]["kind"], fr, fe, cos, cose))
    for r in rows:
        print(f"  F {r[0]} {r[1]} relF gpu {r[2]:.3f} exact-gap {r[3]:.3f} cos gpu {r[4]:.4f} cos exact {r[5]:.4f}")
    for st in stages:
        for k, l in enumerate(st.layers):
            if ref.weights[l] is None:
                continue
            w, bb, _, _ = st.get_weights(k)
            w0 = np.asarray(params[l][0], np.float64).reshape(w.shape)
            wr = np.asarray(ref.weights[l], np.float64).reshape(w.shape)
            du = np.abs(wr - w0).max()
            e = np.abs(w - wr).max() / du
            if e > 0.3 or l in (0, 91, 99):
                sp = layers[l]
                print(f"  {l} {sp['kind']} {sp.get('cin', sp.get('c'))}->{sp.get('cout', '')} k{sp.get('k', '')}"
                      f" s{sp.get('s', '')} h{sp.get('h', '')} upd_err {e:.3f} |dW_gpu| {np.abs(w - w0).max():.3e}"
                      f" |dW_ref| {du:.3e}", flush=True)
        st.close()


if __name__ == "__main__":
    import sys as _s
    layers, starts = ograph.resnet_layers()
    L = len(layers)
    b8 = [0, starts[3], starts[5], starts[7], starts[9], starts[11], starts[14], starts[15], L]
    which = _s.argv[1] if len(_s.argv) > 1 else "s1"
    if which == "s1":
        run_update("R50 S1 M1", layers, [0, L], 2, 8, 1, ost.I_VARIANT, ost.EQ1)
    else:
        run_update("R50 S8 M1", layers, b8, 2, 8, 1, ost.I_VARIANT, ost.EQ1)

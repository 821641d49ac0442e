"""Pipeline x data parallelism ("distributing the network layers
across multiple machines ... working together with data parallelism").

R replicas of the S-stage pipeline, one process per (replica, stage), all on the test box's
one GPU; replica r takes rows [r·B, (r+1)·B) of every pool entry; stage s of every replica
averages the R weight / bias gradients in replica order inside one fused reduce + SGD kernel
that reads the peers' buffers through IPC mappings (NVLink peer memory on a multi-GPU box).
With equal replica batches the averaged gradient is the gradient of the mean loss over the
merged R·B rows, so the oracle is the SAME pipeline replay with m' = R·m micro-batches: no new
oracle code (and its bf16 storage points coincide: 1/(R·B) = (1/B)/R is a power-of-2 rescale
for R = 2, 4).

Checks: replicas bitwise identical; versions / staleness of every backward bit-exact vs the
oracle; mean replica loss within 1e-3 of the merged loss; weights within 5e-3 (Z19).
"""
import numpy as np
import pytest

import synthgen
from oracle import staleness as ost
from paper_2509_23241_b200 import tps
from pipeline_helpers import layer_rel_err, run_oracle, weight_rel_err
from test_gpu_ipc import run_ipc

pytestmark = pytest.mark.gpu

CASES = {
    # name: dims, bounds, m, b, M, R, variant, blend, lam, lr, mu
    "S2xR2-I-CONVEX": ([256, 192, 192, 128, 10], [0, 2, 4], 2, 32, 8, 2, 1, 1, 0.3, 0.05, 0.9),
    "S3xR2-I-EQ1": ([256, 192, 192, 128, 10], [0, 1, 3, 4], 2, 32, 8, 2, 1, 0, 0.3, 0.05, 0.9),
    "S1xR4-V": ([256, 192, 128, 10], [0, 3], 2, 16, 6, 4, 0, 0, 0.05, 0.05, 0.0),
    "S1xR2-I": ([512, 256, 10], [0, 2], 4, 32, 6, 2, 1, 0, 0.05, 0.05, 0.9),
}


@pytest.mark.timeout(900, method="thread")
@pytest.mark.parametrize("name", list(CASES))
def test_dp_replicas_match_merged_oracle(gpu_lib, name):
    dims, bounds, m, b, M, R, var, blend, lam, lr, mu = CASES[name]
    S = len(bounds) - 1
    case = {"dims": dims, "bounds": bounds, "m": m, "b": b, "M": M, "variant": var, "blend": blend, "lam": lam,
            "lr": lr, "mu": mu, "kind": synthgen.X_SIGNED}
    res = run_ipc(case, dp=R)
    ov = ost.V_VARIANT if var == 0 else ost.I_VARIANT
    ob = ost.EQ1 if blend == 0 else ost.CONVEX
    ref = run_oracle(dims, bounds, R * m, b, M, ov, ob, lam, lr, mu, kind=synthgen.X_SIGNED)
    want = sorted((r.stage, r.mb, r.v_used, r.v_latest, r.delta, float(r.alpha), float(r.beta))
                  for r in ref.trace if r.kind == "B")
    by = {(pr["replica"], pr["stage"]): pr for pr in res}
    for rep in range(R):
        got = sorted((s_, mb, vu, vl, d, a, b_) for s in range(S)
                     for (s_, kind, _, _, mb, vu, vl, d, a, b_) in by[(rep, s)]["trace"] if kind == 1)
        assert got == want
    losses = np.mean([by[(rep, S - 1)]["losses"] for rep in range(R)], axis=0)
    np.testing.assert_allclose(losses, ref.losses, rtol=1e-3, atol=0)
    for s in range(S):
        pr0 = by[(0, s)]
        for k, l in enumerate(pr0["layers"]):
            w, bb, mw, mb_ = pr0["weights"][k]
            assert weight_rel_err(w, ref.weights[l]) <= 5e-3, l
            assert layer_rel_err(w, bb, ref.weights[l], ref.biases[l]) <= 5e-3, l
            for rep in range(1, R):      # replicas stay bitwise identical
                for x, y in zip(by[(rep, s)]["weights"][k], (w, bb, mw, mb_)):
                    np.testing.assert_array_equal(x, y)


def test_dp_config_errors(gpu_lib):
    with pytest.raises(tps.TpsError):
        tps.Pipeline(tps.StageSpec([64, 64, 10], [0, 2], 0, 2, 8, dp_size=2, dp_rank=2))
    with pytest.raises(tps.TpsError):      # replicas of a multi-stage pipeline: IPC transport only
        tps.Pipeline(tps.StageSpec([64, 64, 10], [0, 1, 2], 0, 2, 8, transport=tps.TPS_TRANSPORT_LOCAL, dp_size=2))
    st = tps.Pipeline(tps.StageSpec([64, 64, 10], [0, 2], 0, 2, 8, dp_size=2, dp_rank=0))
    with pytest.raises(tps.TpsError) as ei:       # not connected to its replica yet
        st.begin_run(0, 1)
    assert ei.value.status == 9
    st.close()

"""Multi-process execution of the product runtime: one process per stage, IPC transport
(include/tps.h TPS_TRANSPORT_IPC), all processes sharing the one GPU of the test box.

This is the paper's setting (one stage per node, one-to-one exchanges: P:134) run by
the same per-rank walker (tps_run_schedule) the multi-GPU bench uses; only the placement
differs (the processes share a GPU instead of owning one each, so the IPC mappings resolve to
the same HBM instead of NVLink peer memory).  Checks:
  * IPC run == LOCAL-transport run of the same pipeline in one process, BIT FOR BIT (losses,
    every parameter, the trace): the kernels and their order are identical, only the
    exchange differs — fused compute + send (the producing GEMM stores into the neighbour's
    buffer) for chain networks, and the copy path (graph networks / TPS_IPC_DIRECT=0);
  * trace bit-exact and losses / weights within the north_star tolerance vs the oracle.
"""
import json
import os
import pickle
import subprocess
import sys
import tempfile
import time

import numpy as np
import pytest

import synthgen
from oracle import graph as ograph
from oracle import staleness as ost
from pipeline_helpers import layer_rel_err, oracle_trace, run_gpu, run_oracle, weight_rel_err

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def run_ipc(case, env_extra=None, timeout=300, dp=1):
    S = len(case["bounds"]) - 1 if dp == 1 else (len(case["bounds"]) - 1) * dp
    with tempfile.TemporaryDirectory() as store, tempfile.TemporaryDirectory() as out:
        env = dict(os.environ)
        env.update(env_extra or {})
        procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "ipc_worker.py"), "--rank", str(r), "--world",
                                   str(S), "--store", store, "--case", json.dumps(case), "--out", out,
                                   "--dp", str(dp)],
                                  env=env, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
                 for r in range(S)]
        deadline = time.time() + timeout
        logs = []
        try:
            for pr in procs:
                rem = max(1.0, deadline - time.time())
                o, _ = pr.communicate(timeout=rem)
                logs.append(o)
        except subprocess.TimeoutExpired:
            for pr in procs:
                pr.kill()
            raise AssertionError("IPC pipeline timed out:\n" + "\n".join(logs))
        for r, pr in enumerate(procs):
            assert pr.returncode == 0, f"rank {r} failed:\n{logs[r][-3000:]}"
        res = []
        for r in range(S):
            with open(os.path.join(out, f"stage{r}.pkl"), "rb") as fh:
                res.append(pickle.load(fh))
        return res


def trace_rows(res):
    rows = []
    for st in res:
        for (stage, kind, micro, cnt, mb, vu, vl, d, a, b) in st["trace"]:
            if kind == 0:
                for x in range(micro, micro + cnt):
                    rows.append((stage, "F", mb, x, vu, vl, d, 1.0, 0.0))
            elif kind == 1:
                rows.append((stage, "B", mb, -1, vu, vl, d, a, b))
            else:
                rows.append((stage, "U", mb, -1, vu, vl, 0, 1.0, 0.0))
    return sorted(rows)


MLP = {
    "dims": [256, 192, 192, 128, 128, 10], "bounds": [0, 2, 3, 5], "m": 2, "b": 32, "M": 8,
    "variant": 1, "blend": 1, "lam": 0.3, "lr": 0.05, "mu": 0.9, "kind": synthgen.X_SIGNED,
}


def local_reference(case):
    var = ost.V_VARIANT if case["variant"] == 0 else ost.I_VARIANT
    blend = ost.EQ1 if case["blend"] == 0 else ost.CONVEX
    stages, losses = run_gpu(case["dims"], case["bounds"], case["m"], case["b"], case["M"], var, blend, case["lam"],
                             case["lr"], case["mu"], kind=case["kind"], layers=case.get("layers"),
                             fuse_update=case.get("fuse", 1), dtype=case.get("dtype", 0))
    w = [[st.get_weights(k) if st.shapes[k] is not None else None for k in range(len(st.layers))] for st in stages]
    for st in stages:
        st.close()
    return losses, w, (var, blend)


def assert_same_as_local(res, case):
    losses, w, _ = local_reference(case)
    np.testing.assert_array_equal(res[-1]["losses"], losses)
    for s, st in enumerate(res):
        for k, got in enumerate(st["weights"]):
            if got is None:
                continue
            for a, b in zip(got, w[s][k]):
                np.testing.assert_array_equal(a, b)


@pytest.mark.timeout(900, method="thread")
@pytest.mark.parametrize("direct", ["1", "0"])
@pytest.mark.parametrize("variant,blend", [(1, 1), (1, 0), (0, 0)])
def test_ipc_mlp_three_processes(gpu_lib, direct, variant, blend):
    case = dict(MLP, variant=variant, blend=blend)
    res = run_ipc(case, {"TPS_IPC_DIRECT": direct})
    assert_same_as_local(res, case)
    assert all(st["contiguity"] == 3 for st in res)      # TPS_E_ORDER
    var = ost.V_VARIANT if variant == 0 else ost.I_VARIANT
    bl = ost.EQ1 if blend == 0 else ost.CONVEX
    ref = run_oracle(case["dims"], case["bounds"], case["m"], case["b"], case["M"], var, bl, case["lam"], case["lr"],
                     case["mu"], kind=case["kind"])
    assert trace_rows(res) == oracle_trace(ref)
    np.testing.assert_allclose(res[-1]["losses"], ref.losses, rtol=1e-3, atol=0)
    for st in res:
        for k, l in enumerate(st["layers"]):
            w, bb, _, _ = st["weights"][k]
            assert weight_rel_err(w, ref.weights[l]) <= 5e-3
            assert layer_rel_err(w, bb, ref.weights[l], ref.biases[l]) <= 5e-3


@pytest.mark.timeout(900, method="thread")
def test_ipc_tf32_three_processes(gpu_lib):
    """tf32 storage (reading Z28) over the IPC transport: 4-byte elements in every exchanged
    buffer and offset (fused compute + send); bitwise equal to the LOCAL run, and the tf32 oracle's
    trace / tolerances."""
    case = dict(MLP, variant=1, blend=1, dtype=1)
    res = run_ipc(case)
    assert_same_as_local(res, case)
    ref = run_oracle(case["dims"], case["bounds"], case["m"], case["b"], case["M"], ost.I_VARIANT, ost.CONVEX,
                     case["lam"], case["lr"], case["mu"], kind=case["kind"], dtype="tf32")
    assert trace_rows(res) == oracle_trace(ref)
    np.testing.assert_allclose(res[-1]["losses"], ref.losses, rtol=1e-3, atol=0)
    for st in res:
        for k, l in enumerate(st["layers"]):
            w, bb, _, _ = st["weights"][k]
            assert weight_rel_err(w, ref.weights[l]) <= 5e-3


@pytest.mark.timeout(900, method="thread")
def test_ipc_four_processes_full_width(gpu_lib):
    """C2-shaped (4096 wide, staleness 3/2/1/0) with the fused wgrad + update epilogue."""
    case = {"dims": [4096] * 5 + [10], "bounds": [0, 1, 2, 3, 5], "m": 4, "b": 64, "M": 6, "variant": 1,
            "blend": 0, "lam": 0.05, "lr": 0.01, "mu": 0.9, "kind": synthgen.X_SIGNED}
    res = run_ipc(case)
    assert_same_as_local(res, case)


@pytest.mark.timeout(900, method="thread")
def test_ipc_resnet_graph_three_processes(gpu_lib):
    """Graph network (tiny ResNet, block inputs crossing the stage boundaries): copy path."""
    layers, starts = ograph.resnet_layers(blocks=(1, 1), widths=(16, 32), H=32, classes=10, stem_c=16)
    case = {"dims": [32 * 32 * 3, 10], "bounds": [0, starts[1], starts[2], len(layers)], "m": 2, "b": 8, "M": 5,
            "variant": 1, "blend": 1, "lam": 0.05, "lr": 0.01, "mu": 0.9, "kind": synthgen.X_UNIT, "layers": layers}
    res = run_ipc(case)
    assert_same_as_local(res, case)

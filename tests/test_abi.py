"""C-ABI library checks that need no GPU: it loads, exports every symbol include/tps.h
declares, and its host-only entry points (static schedule, blend coefficients,
config validation) agree with the oracle.  No compute call runs here."""
import math
import os
import re
import subprocess

import pytest

from oracle import schedule as osched
from oracle import staleness as ost
from paper_2509_23241_b200 import tps

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "tps.h")).read()
    return sorted(set(re.findall(r"^(?:tps_status|int32_t|const char\*)\s+(tps_[a-z_0-9]+)\(", hdr, re.M)))


def test_header_and_binding_agree():
    assert declared_symbols() == sorted(tps.EXPORTS)


def test_library_exports_every_declared_symbol():
    tps.lib()
    out = subprocess.run(["nm", "-D", "--defined-only", tps.LIB_PATH], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (tps_[a-z_0-9]+)", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    assert tps.lib().tps_abi_version() == 4


@pytest.mark.parametrize("S", [1, 2, 4, 8])
@pytest.mark.parametrize("m,g", [(1, 1), (4, 1), (4, 2), (4, 4), (32, 8)])
def test_static_schedule_matches_oracle(S, m, g):
    for M in (1, 3, 11):
        for s in range(S):
            got = [(e.kind, e.mb, e.micro, e.micro_count) for e in tps.schedule_events(S, s, m, g, M)]
            ref = []
            for e in osched.stage_order(S, s, m, M):
                if e.kind == "F":
                    if e.micro % g == 0:
                        ref.append((0, e.mb, e.micro, g))
                else:
                    ref.append(({"B": 1, "U": 2}[e.kind], e.mb, -1 if True else 0, 0))
            got = [(k, j, a if k == 0 else -1, c if k == 0 else 0) for k, j, a, c in got]
            assert got == ref


@pytest.mark.parametrize("lam", [0.05, 0.3, math.log(2), 2.0])
def test_blend_coeffs_match_oracle_bit_exact(lam):
    for d in range(9):
        for bl, obl in [(tps.TPS_BLEND_EQ1, ost.EQ1), (tps.TPS_BLEND_CONVEX, ost.CONVEX)]:
            assert tps.blend_coeffs(tps.TPS_I, bl, d, lam) == ost.blend_coeffs(ost.I_VARIANT, obl, d, lam)
        assert tps.blend_coeffs(tps.TPS_V, 0, d, lam) == (1.0, 0.0)


def test_blend_coeffs_errors():
    with pytest.raises(tps.TpsError) as e:
        tps.blend_coeffs(tps.TPS_I, 0, 1, 0.0)
    assert e.value.status == 2          # TPS_E_CONFIG: λ > 0
    with pytest.raises(tps.TpsError):
        tps.blend_coeffs(tps.TPS_I, 0, -1, 0.5)


def test_config_validation_errors_without_gpu():
    bad = [
        tps.StageSpec([8, 8, 4], [0, 1], 0, 2, 4),                              # bounds don't end at L
        tps.StageSpec([8, 8, 4], [0, 2], 0, 0, 4),                              # m < 1
        tps.StageSpec([8, 8, 4], [0, 2], 0, 4, 4, fwd_group=3),                 # group must divide m
        tps.StageSpec([8, 8, 4], [0, 2], 0, 2, 4, variant=tps.TPS_I, lam=0.0),  # λ <= 0
        tps.StageSpec([8, 8, 4], [0, 1, 2], 0, 2, 4),                           # S > 1 needs a transport
        tps.StageSpec([8, 8, 4], [0, 0, 2], 0, 2, 4, transport=1),              # empty stage
    ]
    for spec in bad:
        with pytest.raises(tps.TpsError) as e:
            tps.Pipeline(spec)
        assert e.value.status == 2, spec


def test_dtype_validation_without_gpu():
    """tps_config.dtype (reading Z28): an unknown value is TPS_E_CONFIG; tf32 storage on an
    image network or with data parallelism is TPS_E_UNSUPPORTED; both before the device check."""
    with pytest.raises(tps.TpsError) as e:
        tps.Pipeline(tps.StageSpec([8, 8, 4], [0, 2], 0, 2, 4, dtype=7))
    assert e.value.status == 2
    layers = [{"kind": "conv3", "cin": 3, "cout": 64, "h": 8, "w": 8}, {"kind": "linear", "in": 4096, "out": 10}]
    for spec in (tps.StageSpec([192, 10], [0, 2], 0, 2, 4, layers=layers, dtype=tps.TPS_TF32),
                 tps.StageSpec([8, 8, 4], [0, 2], 0, 2, 4, dp_size=2, dp_rank=0, dtype=tps.TPS_TF32)):
        with pytest.raises(tps.TpsError) as e:
            tps.Pipeline(spec)
        assert e.value.status == 10, tps.last_error() if hasattr(tps, "last_error") else spec


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(tps.TpsError) as e:
        tps.Pipeline(tps.StageSpec([8, 8, 4], [0, 2], 0, 2, 4))
    assert e.value.status == 8          # TPS_E_ARCH


def _resnet(**kw):
    from oracle import graph
    return graph.resnet_layers(blocks=(1, 1), widths=(16, 32), H=32, classes=10, stem_c=16, **kw)


def test_graph_config_validation_errors_without_gpu():
    """ResNet-style layer graphs: shape, residual, stage-crossing and head checks run before
    the device check, so each bad config fails with TPS_E_CONFIG on a CPU-only host."""
    import copy
    layers, starts = _resnet()
    L = len(layers)
    dims = [32 * 32 * 3, 10]

    def spec(ls, bounds, sid=0):
        return tps.StageSpec(dims, bounds, sid, 2, 4, layers=ls, transport=1 if len(bounds) > 2 else 0)

    bad = []
    x = copy.deepcopy(layers)
    x[3]["cin"] = 32                                   # conv input channels != its source's
    bad.append(spec(x, [0, L]))
    x = copy.deepcopy(layers)
    x[10]["res"] = 4                                   # residual of a different shape
    bad.append(spec(x, [0, L]))
    x = copy.deepcopy(layers)
    x[0]["cout"] = 12                                  # conv out_c % 16
    x[1]["c"] = 12
    bad.append(spec(x, [0, L]))
    x = copy.deepcopy(layers)
    x.insert(L - 1, {"kind": "linear", "in": 128, "out": 128, "src": L - 2})   # LINEAR not last
    bad.append(spec(x, [0, L + 1]))
    # a stage boundary inside a bottleneck: bn3 would read the block input across the boundary
    bad.append(spec(layers, [0, starts[1] + 2, L], sid=1))
    for sp in bad:
        with pytest.raises(tps.TpsError) as e:
            tps.Pipeline(sp)
        assert e.value.status == 2, tps.last_error() if hasattr(tps, "last_error") else sp
    # the valid graph passes validation and stops at the device check (no GPU here)
    import torch
    if not torch.cuda.is_available():
        with pytest.raises(tps.TpsError) as e:
            tps.Pipeline(spec(layers, [0, starts[1], L], sid=1))
        assert e.value.status == 8

"""CUDA-graph capture / replay of whole runs (include/tps.h tps_graph_*).

The static nF1B order (reading Z7) makes every run of n_mb mini-batches issue the same device
work up to slot indices; with n_mb a multiple of the schedule period those repeat too, so one
captured graph replays every later run.  Checks: capture + replays == walking the same runs,
BIT FOR BIT (losses, all parameters, momentum, the trace with its versions and staleness), for
a multi-stage LOCAL pipeline (I-CONVEX blend on load, fused update, split backward) and a
single stage; the period and state checks."""
import numpy as np
import pytest
import torch

import synthgen
from paper_2509_23241_b200 import tps

pytestmark = pytest.mark.gpu


def make(dims, bounds, m, b, variant, blend, fuse=1, dtype=tps.TPS_BF16):
    S = len(bounds) - 1
    st = [tps.Pipeline(tps.StageSpec(dims=dims, stage_bounds=bounds, stage_id=s, micro_batches=m, micro_batch_size=b,
                                     variant=variant, blend=blend, lam=0.3, lr=0.05, momentum=0.9, seed=3,
                                     transport=tps.TPS_TRANSPORT_LOCAL if S > 1 else tps.TPS_TRANSPORT_NONE,
                                     fuse_update=fuse, dtype=dtype))
          for s in range(S)]
    for h in st:
        h.init_weights_synthetic()
    if S > 1:
        tps.local_link(st)
    return st


def pools(dims, m, b, pool, dtype=tps.TPS_BF16):
    B = m * b
    xdt = torch.float32 if dtype == tps.TPS_TF32 else torch.bfloat16
    x = torch.from_numpy(np.stack([synthgen.inputs(3, j, B, dims[0]) for j in range(pool)])).to(xdt).cuda()
    y = torch.from_numpy(np.stack([synthgen.labels(3, j, B, dims[-1]) for j in range(pool)])).cuda()
    return x, y


def state(st):
    out = [st[-1].losses()]
    for h in st:
        for k in range(len(h.layers)):
            out += list(h.get_weights(k))
    trace = [[(e.kind, e.mb, e.micro, e.v_used, e.v_latest, e.delta, e.alpha, e.beta) for e in h.trace()] for h in st]
    return out, trace


@pytest.mark.parametrize("dims,bounds,m,b,pool,n,variant,blend,fuse,dtype", [
    ([256, 256, 192, 128, 10], [0, 2, 4], 2, 32, 6, 12, tps.TPS_I, tps.TPS_BLEND_CONVEX, 1, tps.TPS_BF16),   # period 6
    ([256, 256, 192, 128, 10], [0, 1, 2, 4], 2, 32, 8, 24, tps.TPS_I, tps.TPS_BLEND_EQ1, 0, tps.TPS_BF16),   # period 24
    ([512, 512, 512, 10], [0, 3], 4, 64, 4, 8, tps.TPS_I, tps.TPS_BLEND_EQ1, 1, tps.TPS_BF16),              # one stage
    ([256, 256, 10], [0, 1, 2], 2, 16, 6, 6, tps.TPS_V, tps.TPS_BLEND_EQ1, 1, tps.TPS_BF16),
    ([256, 256, 192, 128, 10], [0, 2, 4], 2, 32, 6, 12, tps.TPS_I, tps.TPS_BLEND_CONVEX, 1, tps.TPS_TF32),   # tf32 (Z28)
])
def test_graph_replay_equals_walk_bitwise(gpu_lib, dims, bounds, m, b, pool, n, variant, blend, fuse, dtype):
    x, y = pools(dims, m, b, pool, dtype)
    stream = torch.cuda.Stream()
    runs = 3
    walked = make(dims, bounds, m, b, variant, blend, fuse, dtype)
    for r in range(runs):
        tps.run_schedule_local(walked, r * n, n, x, y, pool)
    for h in walked:
        h.synchronize()
    graphed = make(dims, bounds, m, b, variant, blend, fuse, dtype)
    g = tps.Graph(graphed, 0, n, x, y, pool, stream.cuda_stream)
    for _ in range(runs - 1):
        g.replay()
    stream.synchronize()
    for h in graphed:
        h.synchronize()
    (sa, ta), (sb, tb) = state(walked), state(graphed)
    assert ta == tb
    assert len(sa[0]) == runs * n
    for a, b_ in zip(sa, sb):
        np.testing.assert_array_equal(a, b_)
    g.close()
    for h in walked + graphed:
        h.close()


def test_graph_period_and_state_checks(gpu_lib):
    dims, bounds = [256, 256, 192, 128, 10], [0, 2, 4]
    x, y = pools(dims, 2, 32, 6)
    stream = torch.cuda.Stream()
    st = make(dims, bounds, 2, 32, tps.TPS_I, tps.TPS_BLEND_EQ1)
    with pytest.raises(tps.TpsError) as ei:          # 8 is not a multiple of the period (6)
        tps.Graph(st, 0, 8, x, y, 6, stream.cuda_stream)
    assert ei.value.status == 2
    with pytest.raises(tps.TpsError):                # the legacy default stream cannot be captured
        tps.Graph(st, 0, 6, x, y, 6, 0)
    g = tps.Graph(st, 0, 6, x, y, 6, stream.cuda_stream)
    tps.run_schedule_local(st, 6, 6, x, y, 6)        # the handles moved on without the graph
    with pytest.raises(tps.TpsError) as ei:
        g.replay()
    assert ei.value.status == 9
    g.close()
    for h in st:
        h.close()

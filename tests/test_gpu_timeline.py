"""Per-event device timeline (include/tps.h tps_set_timeline / tps_get_timeline) and its
Chrome-trace export (tools/chrome_trace.py).  Checks: one record per trace event, in the trace's
order and with the same contents; brackets ordered (t0 <= t1) and serial on each stage's
compute stream; a shared origin puts stage s's forward of a mini-batch after stage s-1's;
graph capture is refused while the timeline is on; disabling clears it."""
import json
import os
import sys

import numpy as np
import pytest
import torch

import synthgen
from paper_2509_23241_b200 import tps

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
import chrome_trace  # noqa: E402

pytestmark = pytest.mark.gpu


def make(dims, bounds, m, b, variant):
    S = len(bounds) - 1
    st = [tps.Pipeline(tps.StageSpec(dims=dims, stage_bounds=bounds, stage_id=s, micro_batches=m, micro_batch_size=b,
                                     variant=variant, blend=tps.TPS_BLEND_EQ1, lam=0.3, lr=0.05, seed=3,
                                     transport=tps.TPS_TRANSPORT_LOCAL))
          for s in range(S)]
    for h in st:
        h.init_weights_synthetic()
    tps.local_link(st)
    return st


@pytest.mark.parametrize("variant", [tps.TPS_V, tps.TPS_I])
def test_timeline_matches_trace(gpu_lib, tmp_path, variant):
    dims, bounds, m, b, pool = [256, 256, 192, 128, 10], [0, 1, 2, 4], 2, 32, 4
    B = m * b
    x = torch.from_numpy(np.stack([synthgen.inputs(3, j, B, dims[0]) for j in range(pool)])).to(torch.bfloat16).cuda()
    y = torch.from_numpy(np.stack([synthgen.labels(3, j, B, dims[-1]) for j in range(pool)])).cuda()
    st = make(dims, bounds, m, b, variant)
    origin = torch.cuda.Event(enable_timing=True)
    origin.record()
    for h in st:
        h.set_timeline(True, origin.cuda_event)
    n = 8
    tps.run_schedule_local(st, 0, n, x, y, pool)
    recs = [h.timeline() for h in st]
    for h, r in zip(st, recs):
        tr = h.trace()
        assert len(r) == len(tr) > 0
        for a, e in zip(r, tr):
            assert (a.ev.kind, a.ev.mb, a.ev.micro, a.ev.v_used, a.ev.v_latest, a.ev.delta) == \
                   (e.kind, e.mb, e.micro, e.v_used, e.v_latest, e.delta)
            assert 0.0 <= a.t0_ms <= a.t1_ms
        for p_, q in zip(r, r[1:]):                 # one compute stream: brackets are serial
            assert q.t0_ms >= p_.t1_ms - 1e-3
    # mini-batch j's forward enters stage s only after stage s-1 sent it
    for s in range(1, len(st)):
        f_prev = {(a.ev.mb, a.ev.micro): a for a in recs[s - 1] if a.ev.kind == tps.TPS_EV_F}
        for a in recs[s]:
            if a.ev.kind == tps.TPS_EV_F and (a.ev.mb, a.ev.micro) in f_prev:
                assert a.t1_ms >= f_prev[(a.ev.mb, a.ev.micro)].t0_ms
    doc = chrome_trace.to_chrome(recs)
    path = tmp_path / "t.json"
    path.write_text(json.dumps(doc))
    xs = [e for e in json.loads(path.read_text())["traceEvents"] if e["ph"] == "X"]
    assert len(xs) == sum(len(r) for r in recs)
    stream = torch.cuda.Stream()
    with pytest.raises(tps.TpsError) as ei:
        tps.Graph(st, n, 24, x, y, pool, stream.cuda_stream)
    assert ei.value.status == 9
    for h in st:
        h.set_timeline(False)
        assert h.timeline() == []
    for h in st:
        h.close()

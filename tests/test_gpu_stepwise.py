"""The step-wise boundary (include/tps.h): tps_begin_run, tps_stage_forward,
tps_stage_backward(mb, δ) and tps_stage_update called one by one from the host, against
the oracle, plus every error path the header promises.

* An S = 3 LOCAL pipeline is driven event by event in a dependency-respecting host order
  (the same rule as tps_run_schedule_local, re-implemented here), passing each backward the
  EXPLICIT staleness δ the oracle logged for it (W_2(1|3) has δ = 2).  Trace
  bit-exact, losses 1e-3, weights 5e-3 (reading Z19).
* Error paths: TPS_E_ORDER for a call that is not the stage's next static event (P:134,
  reading Z7); TPS_E_STALENESS for an explicit δ != the logged one, for V with δ > 0 (V has
  no stash) and for a version no longer in the ring (microbenchmark mode).  A rejected
  call enqueues nothing, so the run continues and still matches the oracle.
* max_inflight (S = 1, K in flight; the one-GPU staleness sweep of BASELINE configs[1]) vs the
  oracle with the same override; the microbenchmark staleness mode; V vs I stash accounting;
  the torch allocator hook (per-GPU memory visible to torch.cuda.max_memory_allocated).
"""
import numpy as np
import pytest
import torch

import synthgen
from oracle import staleness as ost
from paper_2509_23241_b200 import tps
from pipeline_helpers import expand_gpu_trace, layer_rel_err, oracle_trace, run_gpu, run_oracle, weight_rel_err

pytestmark = pytest.mark.gpu

E_ORDER, E_STALENESS, E_CONFIG = 3, 4, 2


def expect_status(code, fn, *a):
    with pytest.raises(tps.TpsError) as ei:
        fn(*a)
    assert ei.value.status == code, str(ei.value)


def check_parity(stages, losses, ref):
    assert expand_gpu_trace(stages) == oracle_trace(ref)
    np.testing.assert_allclose(losses, ref.losses, rtol=1e-3, atol=0)
    for st in stages:
        for k, l in enumerate(st.layers):
            w, bb, _, _ = st.get_weights(k)
            assert weight_rel_err(w, ref.weights[l]) <= 5e-3, l
            assert layer_rel_err(w, bb, ref.weights[l], ref.biases[l]) <= 5e-3, l


def stepwise_driver(ref, b, probe_errors, v_probe=False):
    """Returns drive(stages, x_pool, y_pool, M) issuing every event with tps_stage_*."""
    logged = {(r.stage, r.mb): r.delta for r in ref.trace if r.kind == "B"}

    def drive(stages, x_pool, y_pool, M):
        S = len(stages)
        m = stages[0].spec.micro_batches
        orders = [tps.schedule_events(S, s, m, 0, M) for s in range(S)]
        for st in stages:
            st.begin_run(0, M)
        if probe_errors:
            # the first static event of every stage is F(0, group 0)
            expect_status(E_ORDER, stages[0].stage_backward, 0, -1)
            expect_status(E_ORDER, stages[0].stage_update, 0)
            expect_status(E_ORDER, stages[0].stage_forward, 1, 0, m, x_pool[1], None)
            # stage 1 has not received mini-batch 0 yet: the LOCAL mailbox is empty
            expect_status(E_ORDER, stages[1].stage_forward, 0, 0, m, None, None)
        pos = [0] * S
        fcount, bcount = [0] * S, [0] * S
        probed = set()
        while any(pos[s] < len(orders[s]) for s in range(S)):
            progress = False
            for s in range(S):
                if pos[s] >= len(orders[s]):
                    continue
                e = orders[s][pos[s]]
                j = e.mb
                if e.kind == tps.TPS_EV_F:
                    if s > 0 and fcount[s - 1] <= j:
                        continue
                    if s < S - 1 and j >= 2 and fcount[s + 1] <= j - 2:
                        continue
                    rows = slice(e.micro * b, (e.micro + e.micro_count) * b)
                    x = x_pool[j % len(x_pool)][rows] if s == 0 else None
                    y = y_pool[j % len(y_pool)][rows] if s == S - 1 else None
                    stages[s].stage_forward(j, e.micro, e.micro_count, x, y)
                    fcount[s] += 1
                elif e.kind == tps.TPS_EV_B:
                    if s < S - 1 and bcount[s + 1] <= j:
                        continue
                    if s > 0 and j >= 2 and bcount[s - 1] <= j - 2:
                        continue
                    d = logged[(s, j)]
                    if v_probe and s not in probed:
                        probed.add(s)
                        expect_status(E_STALENESS, stages[s].stage_backward, j, 1)   # V has no stash
                    if probe_errors and d > 0 and s not in probed:
                        probed.add(s)
                        expect_status(E_STALENESS, stages[s].stage_backward, j, d + 1)
                        expect_status(E_STALENESS, stages[s].stage_backward, j, d - 1)
                        expect_status(E_ORDER, stages[s].stage_update, j)
                    stages[s].stage_backward(j, d)
                    bcount[s] += 1
                else:
                    stages[s].stage_update(j)
                pos[s] += 1
                progress = True
            assert progress, "host order deadlocked"
        if probe_errors:
            expect_status(E_ORDER, stages[0].stage_forward, M, 0, m, x_pool[0], None)   # run complete
    return drive


@pytest.mark.parametrize("blend", [ost.EQ1, ost.CONVEX])
@pytest.mark.parametrize("fuse", [1, 0])
def test_stepwise_three_stages_explicit_staleness(gpu_lib, blend, fuse):
    dims, bounds = [192, 128, 128, 128, 128, 10], [0, 2, 4, 5]
    m, b, M = 2, 16, 8
    args = (dims, bounds, m, b, M, ost.I_VARIANT, blend, 0.3, 0.05, 0.9)
    ref = run_oracle(*args)
    assert max(r.delta for r in ref.trace if r.kind == "B") == 2          # stage 0: δ up to S-1
    stages, losses = run_gpu(*args, fuse_update=fuse, drive=stepwise_driver(ref, b, probe_errors=True))
    check_parity(stages, losses, ref)
    for st in stages:
        st.close()


def test_stepwise_equals_run_schedule_bitwise(gpu_lib):
    """The walker (tps_run_schedule_local) and the host-driven step-wise calls issue the same
    kernels: identical losses and weights bit for bit."""
    dims, bounds = [128, 128, 128, 64, 10], [0, 2, 3, 4]
    args = (dims, bounds, 2, 16, 6, ost.I_VARIANT, ost.EQ1, 0.3, 0.05, 0.9)
    ref = run_oracle(*args)
    st_a, l_a = run_gpu(*args)
    st_b, l_b = run_gpu(*args, drive=stepwise_driver(ref, 16, probe_errors=False))
    np.testing.assert_array_equal(l_a, l_b)
    for sa, sb in zip(st_a, st_b):
        for k in range(len(sa.layers)):
            for x, y in zip(sa.get_weights(k), sb.get_weights(k)):
                np.testing.assert_array_equal(x, y)


def test_v_rejects_positive_staleness(gpu_lib):
    dims, bounds = [128, 128, 128, 10], [0, 1, 2, 3]
    args = (dims, bounds, 2, 8, 5, ost.V_VARIANT, ost.EQ1, 0.05, 0.05, 0.0)
    ref = run_oracle(*args)
    assert all(r.delta == 0 for r in ref.trace)                          # V: zero staleness
    stages, losses = run_gpu(*args, drive=stepwise_driver(ref, 8, probe_errors=True, v_probe=True))
    check_parity(stages, losses, ref)
    for st in stages:
        assert st.stash_info()[0] == 1 and st.stash_info()[2] == 0      # V holds one version
        st.close()


@pytest.mark.parametrize("K", [2, 4])
@pytest.mark.parametrize("blend", [ost.EQ1, ost.CONVEX])
def test_max_inflight_one_stage_matches_oracle(gpu_lib, K, blend):
    """S = 1 keeping K mini-batches in flight: δ = min(j, K-1) (the staleness a stage at depth K
    sees), I-TiMePReSt backward on the blended stash, against the oracle with the same K."""
    dims, bounds = [256, 256, 256, 10], [0, 3]
    args = (dims, bounds, 2, 32, 10, ost.I_VARIANT, blend, 0.3, 0.05, 0.9)
    ref = run_oracle(*args, max_inflight=K)
    stages, losses = run_gpu(*args, max_inflight=K)
    deltas = [e.delta for e in stages[0].trace() if e.kind == 1]
    assert deltas == [min(j, K - 1) for j in range(10)]
    check_parity(stages, losses, ref)
    lv, stash, peak = stages[0].stash_info()
    assert peak == (K - 1) * sum(2 * ((o + 15) // 16 * 16) * ((i + 15) // 16 * 16)
                                 for o, i in stages[0].shapes)
    stages[0].close()


def test_max_inflight_config_errors(gpu_lib):
    with pytest.raises(tps.TpsError) as ei:
        tps.Pipeline(tps.StageSpec([64, 64, 10], [0, 1, 2], 0, 2, 8, transport=tps.TPS_TRANSPORT_LOCAL,
                                   max_inflight=3))
    assert ei.value.status == E_CONFIG


def test_microbenchmark_staleness_mode(gpu_lib):
    """staleness_mode = 1: an explicit δ other than the logged one is used as given while its
    version is in the ring (here R = K = 4: δ <= min(3, latest)); beyond it TPS_E_STALENESS."""
    dims = [256, 256, 10]
    spec = tps.StageSpec(dims, [0, 2], 0, 2, 32, variant=tps.TPS_I, blend=tps.TPS_BLEND_CONVEX, lam=0.2,
                         max_inflight=4, staleness_mode=1)
    st = tps.Pipeline(spec)
    st.init_weights_synthetic()
    x = torch.empty(8, 64, 256, dtype=torch.bfloat16, device="cuda")
    y = torch.empty(8, 64, dtype=torch.int32, device="cuda")
    for j in range(8):
        tps.fill_synthetic(0, 0, synthgen.TID_X + j, 64, 256, 0, x[j])
        tps.fill_synthetic(2, 0, synthgen.TID_Y + j, 64, 1, 10, y[j])
    torch.cuda.synchronize()
    st.begin_run(0, 8)
    for j in range(4):
        st.stage_forward(j, 0, 2, x[j], y[j])
    for j in range(8):
        latest = j
        if j >= 1:
            expect_status(E_STALENESS, st.stage_backward, j, latest + 1)   # version -1 never existed
        if j >= 4:
            expect_status(E_STALENESS, st.stage_backward, j, 4)            # evicted from the R = 4 ring
        want = min(j, 2)                                                   # != logged min(j, 3) for j >= 3
        st.stage_backward(j, want)
        st.stage_update(j)
        if j + 4 < 8:
            st.stage_forward(j + 4, 0, 2, x[j + 4], y[j + 4])
    st.synchronize()
    bs = [e for e in st.trace() if e.kind == 1]
    assert [e.delta for e in bs] == [min(j, 2) for j in range(8)]
    for e in bs:
        assert (e.alpha, e.beta) == tps.blend_coeffs(tps.TPS_I, tps.TPS_BLEND_CONVEX, e.delta, 0.2)
        assert e.v_used == e.v_latest - e.delta
    assert np.isfinite(st.losses()).all()
    st.close()


def test_stash_info_v_vs_i(gpu_lib):
    """Live versions / stash bytes during a run: I holds S - s versions at stage s once the
    pipeline is full, V always one and zero stash."""
    dims, bounds = [256, 256, 256, 256, 10], [0, 2, 3, 4]
    peaks = {}
    for var in (ost.V_VARIANT, ost.I_VARIANT):
        stages, _ = run_gpu(dims, bounds, 2, 16, 8, var, ost.EQ1, 0.05, 0.05, 0.0)
        peaks[var] = [st.stash_info()[2] for st in stages]
        for st in stages:
            st.close()
    ver = [2 * 256 * 256 * 2, 2 * 256 * 256, 2 * 256 * 16]   # bf16 bytes of one version per stage
    assert peaks[ost.V_VARIANT] == [0, 0, 0]
    assert peaks[ost.I_VARIANT] == [(3 - s - 1) * ver[s] for s in range(3)]


def test_torch_allocator_hook(gpu_lib):
    """dev_alloc / dev_free through PyTorch's caching allocator: the handle's buffers appear in
    torch.cuda.memory_allocated (the per-GPU peak memory the bench reports) and are returned
    on destroy; the run is bitwise identical to one on cudaMalloc."""
    dims, bounds = [256, 256, 256, 10], [0, 2, 3]
    args = (dims, bounds, 2, 16, 5, ost.I_VARIANT, ost.CONVEX, 0.3, 0.05, 0.9)
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated()
    st_t, l_t = run_gpu(*args, torch_alloc=True)
    held = torch.cuda.memory_allocated() - base
    lib_bytes = sum(st.memory_stats()["peak"] for st in st_t)
    assert held >= lib_bytes > 0
    st_c, l_c = run_gpu(*args)
    np.testing.assert_array_equal(l_t, l_c)
    for a, c in zip(st_t, st_c):
        np.testing.assert_array_equal(a.get_weights(0)[0], c.get_weights(0)[0])
        # cudaMalloc path: the device's free memory dropped by about the library's own count
        # (2 MiB pages: small allocations share pages with earlier ones)
        assert abs(c.memory_observed() - c.memory_stats()["peak"]) <= 4 * 2 ** 20 + c.memory_stats()["peak"] // 10
    for st in st_t + st_c:
        st.close()
    torch.cuda.synchronize()
    assert torch.cuda.memory_allocated() - base < held

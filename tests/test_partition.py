"""NEXT-4 partitioner (tps_partition, host-only C++): exact min-max over consecutive splits,
checked against brute-force enumeration of every partition; memory model of DESIGN.md."""
import itertools
import math

import numpy as np
import pytest

from paper_2509_23241_b200 import tps


def stage_mem(pb, ab, i, j, s, S, variant, mom):
    K = S - s
    R = K if variant == tps.TPS_I else 1
    return sum(pb[i:j]) * (1 + (1 if mom else 0) + 0.5 * R) + K * sum(ab[i:j])


def brute(pb, ab, fl, S, variant, mom, objective):
    L = len(pb)
    best, arg = math.inf, None
    for cuts in itertools.combinations(range(1, L), S - 1):
        b = [0, *cuts, L]
        costs = [(sum(fl[b[s]:b[s + 1]]) if objective == 1 else stage_mem(pb, ab, b[s], b[s + 1], s, S, variant, mom))
                 for s in range(S)]
        if max(costs) < best:
            best, arg = max(costs), b
    return best, arg


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("S", [1, 2, 3, 4])
@pytest.mark.parametrize("variant", [tps.TPS_V, tps.TPS_I])
@pytest.mark.parametrize("objective", [0, 1])
def test_partition_is_optimal(seed, S, variant, objective):
    rng = np.random.default_rng(seed)
    L = 9
    pb, ab, fl = rng.integers(1, 100, L) * 1e6, rng.integers(1, 50, L) * 1e6, rng.integers(1, 100, L) * 1e9
    bounds, cost = tps.partition(pb, ab, fl, S, variant, True, objective)
    ref, _ = brute(list(pb), list(ab), list(fl), S, variant, True, objective)
    assert bounds[0] == 0 and bounds[-1] == L and all(b2 > b1 for b1, b2 in zip(bounds, bounds[1:]))
    assert max(cost) == pytest.approx(ref, rel=1e-12)


def test_i_stash_shifts_layers_away_from_early_stages():
    # equal layers: I's stash (K_s copies at stage s) makes early stages costlier, so the
    # memory-balanced I partition gives stage 0 no more layers than the V partition does
    L, S = 16, 4
    pb, ab = np.full(L, 64e6), np.full(L, 16e6)
    bv, _ = tps.partition(pb, ab, None, S, tps.TPS_V, True, 0)
    bi, ci = tps.partition(pb, ab, None, S, tps.TPS_I, True, 0)
    assert bi[1] - bi[0] <= bv[1] - bv[0]
    assert bi[-1] - bi[-2] >= bv[-1] - bv[-2]

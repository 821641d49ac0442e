"""NEXT-3 harness smoke: the statistical-efficiency tool runs every variant over
several seeds on the GPU path and the synthetic teacher-student task is learnable (every
variant's epoch loss falls below its first epoch's for every seed).  It reports, it does not
assert which variant converges faster: that is the paper's empirical claim, measured by
tools/stat_efficiency.py and recorded under profiles/."""
import os
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.timeout(600)
def test_stat_efficiency_harness_runs_and_learns(gpu_lib, monkeypatch):
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import stat_efficiency
    monkeypatch.setattr(sys, "argv", ["stat_efficiency.py", "--stages", "2", "--depth", "4", "--width", "256",
                                      "--epochs", "4", "--batches", "8", "--seeds", "0,1", "--quick", "--lr", "0.05"])
    rep = stat_efficiency.main()
    assert set(rep["results"]) == {"V", "I-EQ1 λ=0.05", "I-CONVEX λ=0.5"}
    for name, r in rep["results"].items():
        assert len(r["epoch_mean_loss_per_seed"]) == 2
        for curve in r["epoch_mean_loss_per_seed"]:
            assert curve[-1] < curve[0], (name, curve)

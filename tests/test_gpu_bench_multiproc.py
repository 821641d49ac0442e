"""bench.py's N > 1 path on the one-GPU test box: `torch.distributed.run --nproc-per-node 2
bench.py --gpus 2 --same-device` (one process per pipeline stage, IPC transport with the fused
compute + send, gloo process group for the rendezvous, max-over-ranks device timing, memory
gather).  Checks that rank 0 prints one well-formed JSON line for the 2-stage run."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.timeout(600, method="thread")
def test_bench_two_stages_two_processes(gpu_lib):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", "29541", os.path.join(ROOT, "bench.py"), "--gpus", "2", "--same-device",
           "--steps", "2", "--warmup", "3", "--epoch-mb", "8", "--no-v"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=540, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["parallelism"] == "pp2" and d["config"]["stages"] == 2
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
    assert len(d["memory_per_gpu"]) == 2
    assert d["losses_first_last"] is None or all(x == x for x in d["losses_first_last"])

"""Microbenchmark of the stage GEMM modes at the bench shapes (C5: B=2048, d=4096),
CUDA-event timed, with cuBLAS (torch.matmul) beside it for context."""
import argparse
import os
import statistics
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_23241_b200 import tps  # noqa: E402


class Nvml:
    """pynvml sampling (SM clock MHz, board power W) in a thread while a mode runs, so a
    number can be read against the clock it ran at (this pool's B200s are power-capped)."""

    def __init__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
        except Exception:
            self.nv = None
        self.rows = []

    def __enter__(self):
        import threading
        self.rows, self.stop = [], False

        def run():
            while not self.stop and self.nv:
                try:
                    self.rows.append((self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM),
                                      self.nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0))
                except Exception:
                    break
                time.sleep(0.005)
        self.t = threading.Thread(target=run, daemon=True)
        self.t.start()
        return self

    def __exit__(self, *a):
        self.stop = True
        self.t.join()

    def summary(self):
        if not self.rows:
            return ""
        rows = self.rows[len(self.rows) // 4:]          # skip the ramp
        mhz = statistics.median(r[0] for r in rows)
        w = statistics.median(r[1] for r in rows)
        return f"  [{mhz:.0f} MHz, {w:.0f} W]"


def timeit(fn, iters=20, warm=5, seconds=0.0):
    if seconds > 0:            # steady state under the power cap: run ~seconds before timing
        t0 = time.time()
        while time.time() - t0 < seconds:
            for _ in range(20):
                fn()
            torch.cuda.synchronize()
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--M", type=int, default=2048)
    ap.add_argument("--N", type=int, default=4096)
    ap.add_argument("--K", type=int, default=4096)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--modes", default="0,1,2,3,4")
    ap.add_argument("--seconds", type=float, default=0.0,
                    help="run each mode this long first and sample SM clock / power while timing")
    a = ap.parse_args()
    M, N, K = a.M, a.N, a.K
    X = torch.randn(M, K, device="cuda").to(torch.bfloat16)          # fwd A / dgrad A (G)
    W = (torch.randn(N, K, device="cuda") * K ** -0.5).to(torch.bfloat16)
    Wt = (torch.randn(K, N, device="cuda") * K ** -0.5).to(torch.bfloat16)  # dgrad B stored [K, N]
    W2 = Wt.clone()
    Gk = torch.randn(K, M, device="cuda").to(torch.bfloat16)          # wgrad A stored [K, M]
    Xk = torch.randn(K, N, device="cuda").to(torch.bfloat16)          # wgrad B stored [K, N]
    mask = torch.randn(M, N, device="cuda").to(torch.bfloat16)
    bias = torch.zeros(N, device="cuda")
    ob = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    of = torch.empty(M, N, device="cuda", dtype=torch.float32)
    # fused wgrad + update at the pipeline's shape: dW [N, N] = Gᵀ·X over K = M rows
    G4 = torch.randn(M, N, device="cuda").to(torch.bfloat16)
    X4 = torch.randn(M, N, device="cuda").to(torch.bfloat16)
    wm = torch.randn(N, N, device="cuda")
    vm = torch.zeros(N, N, device="cuda")
    qm = torch.empty(N, N, device="cuda", dtype=torch.bfloat16)
    fl = 2.0 * M * N * K
    # dual: the fused wgrad + update above together with a dgrad of the same size (one launch)
    Gd = torch.randn(M, N, device="cuda").to(torch.bfloat16)
    Wd = (torch.randn(N, N, device="cuda") * N ** -0.5).to(torch.bfloat16)
    od = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    maskd = torch.randn(M, N, device="cuda").to(torch.bfloat16)

    Xf, Wf, Wtf, maskf, Gkf, Xkf = (t.float() for t in (X, W, Wt, mask, Gk, Xk))

    def sep():
        tps.gemm_wgrad_sgd(N, N, M, G4, N, X4, N, wm, vm, qm, N, 1e-9, 0.9)
        tps.gemm(1, M, N, N, Gd, N, Wd, N, od, N, 0, None, 0, 0.9, 0.0, maskd, N)

    runs = {
        0: ("fwd  (K-major A,B; bias+ReLU)", lambda: tps.gemm(0, M, N, K, X, K, W, K, ob, N, 0, bias, 1)),
        1: ("dgrad(MN-major B; α, mask)", lambda: tps.gemm(1, M, N, K, X, K, Wt, N, ob, N, 0, None, 0, 0.9, 0.0, mask, N)),
        2: ("wgrad(MN-major A,B; fp32)", lambda: tps.gemm(2, M, N, K, Gk, M, Xk, N, of, N, 1)),
        3: ("dgrad blend-on-load", lambda: tps.gemm(3, M, N, K, X, K, Wt, N, ob, N, 0, None, 0, 0.7, 0.3, mask, N, B2=W2)),
        4: ("wgrad + fused SGD/momentum update", lambda: tps.gemm_wgrad_sgd(N, N, M, G4, N, X4, N, wm, vm, qm, N,
                                                                           1e-9, 0.9)),
        5: ("dual: wgrad+update & dgrad, one launch", lambda: tps.gemm_bwd_dual(
            N, N, M, G4, N, X4, N, wm, vm, qm, N, 1e-9, 0.9, 0.0, M, N, N, Gd, N, Wd, N, od, N, 0.9, maskd, N)),
        6: ("the same two as separate launches", sep),
        # tf32 storage (reading Z28): kind::tf32 on fp32 containers (half the bf16 tensor rate)
        7: ("tf32 fwd", lambda: tps.gemm(tps.GEMM_FWD | tps.TPS_GEMM_TF32, M, N, K, Xf, K, Wf, K, of, N, 0, bias, 1)),
        8: ("tf32 dgrad", lambda: tps.gemm(tps.GEMM_DGRAD | tps.TPS_GEMM_TF32, M, N, K, Xf, K, Wtf, N, of, N, 0, None,
                                           0, 0.9, 0.0, maskf, N)),
        9: ("tf32 wgrad", lambda: tps.gemm(tps.GEMM_WGRAD | tps.TPS_GEMM_TF32, M, N, K, Gkf, M, Xkf, N, of, N, 1)),
    }
    for m in [int(x) for x in a.modes.split(",")]:
        name, fn = runs[m]
        nv = Nvml()
        with nv:
            ms = timeit(fn, a.iters if not a.seconds else max(a.iters, 200), seconds=a.seconds)
        extra = ""
        f = fl
        if m == 4:   # HBM roofline of the fused kernel: operands + 18 B per parameter (w, v r/w + bf16 version)
            by = 2.0 * (M * N + M * N) + 18.0 * N * N
            extra = f"  {by / ms / 1e6:7.1f} GB/s algorithmic ({by / 1e6:.1f} MB)"
        if m in (5, 6):
            f = 2.0 * M * N * N * 2
        print(f"mode {m} {name:34s} {M}x{N}x{K}: {ms*1e3:8.1f} us  {f/ms/1e9:7.1f} TFLOP/s{extra}{nv.summary()}",
              flush=True)
    nv = Nvml()
    with nv:
        ms = timeit(lambda: torch.matmul(X, W.T), a.iters if not a.seconds else max(a.iters, 200), seconds=a.seconds)
    print(f"cuBLAS torch.matmul bf16 {M}x{N}x{K}: {ms*1e3:8.1f} us  {fl/ms/1e9:7.1f} TFLOP/s{nv.summary()}")


if __name__ == "__main__":
    main()

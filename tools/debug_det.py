"""Bitwise determinism of the individual kernels at ResNet-50 shapes (3 repeats each)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2509_23241_b200 import tps  # noqa: E402

g = torch.Generator(device="cuda").manual_seed(0)


def rnd(*s, scale=1.0):
    return (torch.randn(*s, generator=g, device="cuda") * scale).to(torch.bfloat16)


def check(name, fn, out):
    res = []
    for _ in range(4):
        out.fill_(float("nan"))
        fn()
        torch.cuda.synchronize()
        res.append(out.clone())
    same = all(torch.equal(res[0], r) for r in res[1:])
    nan = torch.isnan(res[0].float()).any().item()
    print(f"{name:50s} deterministic={same} nan={nan}", flush=True)


N = 16
for (H, Ci, Co, k, s, p) in [(56, 64, 64, 3, 1, 1), (56, 128, 128, 3, 2, 1), (28, 128, 128, 3, 1, 1), (14, 256, 256, 3, 1, 1),
                             (7, 512, 512, 3, 1, 1), (56, 256, 512, 1, 2, 0)]:
    X = rnd(N, H, H, Ci)
    Wt = rnd(Co, k, k, Ci, scale=(k * k * Ci) ** -0.5)
    Ho = (H + 2 * p - k) // s + 1
    out = torch.empty(N * Ho * Ho, Co, device="cuda", dtype=torch.bfloat16)
    check(f"conv fwd H{H} {Ci}->{Co} k{k} s{s}", lambda: tps.conv2d_gemm(0, N, H, H, Ci, Co, k, s, p, X, Wt, out), out)
    dY = rnd(N, Ho, Ho, Co)
    dW = torch.empty(Co, k * k * Ci, device="cuda")
    check(f"conv wgrad H{H} {Ci}->{Co} k{k} s{s}", lambda: tps.conv2d_gemm(2, N, H, H, Ci, Co, k, s, p, dY, X, dW, 1), dW)
    if s == 1:
        dX = torch.empty(N * H * H, Ci, device="cuda", dtype=torch.bfloat16)
        check(f"conv dgrad H{H} {Ci}->{Co}", lambda: tps.conv2d_gemm(1, N, H, H, Ci, Co, 3, 1, 1, dY, Wt, dX), dX)
for (M, Nn, K) in [(50176, 256, 64), (3136, 1024, 256), (784, 2048, 512), (16, 1000, 2048)]:
    A = rnd(M, K)
    B = rnd(Nn, K, scale=K ** -0.5)
    o = torch.empty(M, Nn, device="cuda", dtype=torch.bfloat16)
    check(f"gemm fwd {M}x{Nn}x{K}", lambda: tps.gemm(0, M, Nn, K, A, K, B, K, o, Nn, 0), o)
    Gk = rnd(M, Nn)
    dW = torch.empty(Nn, K, device="cuda")
    check(f"gemm wgrad {Nn}x{K}x{M}", lambda: tps.gemm(2, Nn, K, M, Gk, Nn, A, K, dW, K, 1), dW)
segs, rows, C = 2, 8 * 56 * 56, 64
x = rnd(segs * rows, C)
y = torch.empty_like(x)
gam = torch.ones(C, device="cuda")
bet = torch.zeros(C, device="cuda")
mean = torch.empty(segs, C, device="cuda")
inv = torch.empty(segs, C, device="cuda")
check("bn forward", lambda: tps.bn_forward(x, None, y, gam, bet, mean, inv, segs, rows, C, 1), y)
X = rnd(16, 112, 112, 64)
Y = torch.empty(16, 56, 56, 64, device="cuda", dtype=torch.bfloat16)
check("maxpool3 fwd", lambda: tps.pool_op(0, X, None, Y, 16, 112, 112, 64), Y)
P = torch.empty(16 * 112 * 112, 160, device="cuda", dtype=torch.bfloat16)
X3 = rnd(16, 224, 224, 3)
check("im2col stem", lambda: tps.im2col(X3, P, 16, 224, 224, 3, 7, 2, 3, 160), P)

#!/usr/bin/env python
"""Benchmark: training samples/s of the TiMePReSt pipeline step at N B200 stages.

Workload (BASELINE.json configs[4], the stage-scaling sweep):
  deep MLP, 16 x Linear(4096,4096)+ReLU + head 4096->10, micro-batches of b = 64,
  m = 32 micro-batches per mini-batch (B = 2048), S = N stages (one per GPU, 16/S hidden
  layers each, head on the last), I-TiMePReSt EQ1 (λ = 0.05, staleness up to S-1 at
  stage 0: "I max staleness"), SGD momentum 0.9.  Synthetic bf16 inputs / random labels.

One "step" = one pipeline epoch of EPOCH_MB = 64 mini-batches (131072 samples), i.e. the
static nF1B order with fill, steady state and drain (reading Z17; "throughput" is
epochs per unit time in the paper).  value = samples / (max over ranks of the
device time of the K timed epochs).

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
       (N > 1: launched by torch.distributed.run, one rank = one stage = one GPU)
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HIDDEN, WIDTH, CLASSES = 16, 4096, 10
MICRO_B, MICRO_M = 64, 32
EPOCH_MB = 64
POOL = 8
LAM, LR, MU = 0.05, 0.01, 0.9
METRIC = "training samples/sec at 1/2/4/8 B200 stages; per-GPU peak memory V vs I"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--epoch-mb", type=int, default=EPOCH_MB)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-v", action="store_true")
    ap.add_argument("--fwd-group", type=int, default=0)
    ap.add_argument("--fuse-update", type=int, default=1, help="1: SGD update in the wgrad epilogue (TMA-fed)")
    ap.add_argument("--transport", default="ipc", choices=["ipc", "nccl"],
                    help="N > 1: ipc = neighbours' buffers mapped, the producing GEMM stores into them "
                         "(fused compute + send); nccl = ncclSend/ncclRecv per edge")
    ap.add_argument("--same-device", action="store_true",
                    help="N > 1 on ONE GPU: every rank uses cuda:0 (gloo process group); exercises the "
                         "multi-process path on a one-GPU box (throughput is then time-sliced)")
    ap.add_argument("--prio-stream", action="store_true",
                    help="enqueue on a high-priority compute stream (the weight-gradient / optimizer streams "
                         "stay at the default priority)")
    ap.add_argument("--no-torch-alloc", action="store_true", help="cudaMalloc instead of the torch allocator hook")
    ap.add_argument("--graph", type=int, default=1,
                    help="N = 1: capture one epoch as a CUDA graph (tps_graph_capture) and replay it for every "
                         "step (0 = walk the static order from the host every step)")
    ap.add_argument("--no-method", action="store_true", help="skip the C2 method leg (4 stages, V / I-EQ1 / "
                    "I-CONVEX, staleness sweep, measured memory)")
    return ap.parse_args()


def model(S):
    dims = [WIDTH] * (HIDDEN + 1) + [CLASSES]
    per = HIDDEN // S
    bounds = [s * per for s in range(S)] + [HIDDEN + 1]
    return dims, bounds


def flops_per_sample():
    # forward + dgrad + wgrad = 3 GEMMs of 2·d_in·d_out per sample and layer (layer 0 has no dgrad)
    d = [WIDTH] * (HIDDEN + 1) + [CLASSES]
    f = 0.0
    for l in range(len(d) - 1):
        g = 2.0 * d[l] * d[l + 1]
        f += g * (3 if l > 0 else 2)
    return f


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return p, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """nvidia-smi sampling during the timed region (clocks + throttle reasons)."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu):
        self.gpu = gpu
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        rows = [r.split(",") for r in out.strip().splitlines() if r.count(",") >= 6]
        sm = [float(r[0]) for r in rows if r[0].strip().replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if "Active" in r[3 + i] and "Not" not in r[3 + i]})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ------------------------------------------------------------------ oracle (CPU) legs
def oracle_sample(rows_m=4, seconds_hint=None):
    """Time the oracle on a bounded sample of the workload: ONE mini-batch of rows_m
    micro-batches of 64 rows through all 17 layers at S = 1 (forward, collective backward,
    update of all 16·4096² + head parameters).  Returns (samples/s, seconds, cores, desc)."""
    import numpy as np
    from threadpoolctl import threadpool_info

    import synthgen
    from oracle import pipeline as opipe
    from oracle import staleness as ost

    dims, _ = model(1)
    m, b = rows_m, MICRO_B
    B = m * b
    xs = [synthgen.inputs(0, 0, B, dims[0])]
    ys = [synthgen.labels(0, 0, B, CLASSES)]
    w0 = [synthgen.weights(0, l, dims[l + 1], dims[l]) for l in range(len(dims) - 1)]
    b0 = [np.zeros(dims[l + 1], np.float32) for l in range(len(dims) - 1)]
    cfg = opipe.Config(dims, [0, len(dims) - 1], m, b, 1, variant=ost.I_VARIANT, blend=ost.EQ1, lam=LAM, lr=LR,
                       momentum=MU)
    t0 = time.perf_counter()
    opipe.run(cfg, xs, ys, w0, b0)
    dt = time.perf_counter() - t0
    cores = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    desc = (f"oracle (numpy fp64 + bf16 emulation), S=1, one mini-batch of {B} rows "
            f"({m} micro-batches of {b}) through all {len(dims)-1} layers incl. the update; "
            f"samples/s = {B} / wall time")
    return B / dt, dt, cores, desc


def run_reference(args, rank, world):
    if rank != 0:
        return
    vals = []
    cores = desc = None
    for i in range(args.warmup + args.steps):
        v, dt, cores, desc = oracle_sample(rows_m=2)
        if i >= args.warmup:
            vals.append((v, dt))
    value = statistics.median(v for v, _ in vals)
    ms = statistics.median(dt for _, dt in vals) * 1e3
    dims, bounds = model(args.gpus)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(args),
        "cpu_baseline": {"value": value, "unit": "samples/s", "cores": cores, "kind": "oracle", "sample": desc},
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_dict(args):
    S = args.gpus
    return {"workload": "C5 deep-MLP stage-scaling sweep (BASELINE.json configs[4])",
            "layers": f"{HIDDEN} x Linear({WIDTH},{WIDTH})+ReLU + Linear({WIDTH},{CLASSES}) + softmax-CE",
            "stages": S, "micro_batch": MICRO_B, "micro_batches": MICRO_M, "global_batch": MICRO_B * MICRO_M,
            "variant": "I-TiMePReSt EQ1", "lambda": LAM, "optimizer": f"SGD lr={LR} momentum={MU}",
            "step": f"one pipeline epoch = {args.epoch_mb} mini-batches (fill+steady+drain)",
            "fused_update": bool(args.fuse_update), "parallelism": f"pp{S}",
            "issue": "CUDA graph of one epoch, replayed per step" if (args.graph and S == 1) else
                     "host walker (tps_run_schedule) per step", "l2": "inputs+weights per step >> 126 MB L2 (no flush needed)"}


# ------------------------------------------------------------------ method leg (C2 on one GPU)
def method_leg(torch, tps, windows=3, epoch=32, pool=4):
    """BASELINE.json configs[1]: 4-stage MLP, 8 x Linear(4096,4096) + head,
    m = 8 micro-batches of 64, all 4 stages as LOCAL handles on this GPU (so samples/s is the
    one-GPU cost of the whole pipeline), staleness 3/2/1/0 by stage; V, I-EQ1 and I-CONVEX
    through tps_run_schedule_local; per-variant memory measured by the allocator (PyTorch's
    caching allocator via the dev_alloc hook) and the library's per-stage accounting.  Then the
    "staleness sweep 0..3": one stage (2 x 4096^2 + head) keeping K = 1..4 mini-batches in
    flight (tps_config.max_inflight), steady δ = K - 1, I-EQ1 and I-CONVEX."""
    dims, bounds, m, b = [WIDTH] * 9 + [CLASSES], [0, 2, 4, 6, 9], 8, 64
    B = m * b
    cur = torch.cuda.current_stream()
    x = torch.empty(pool, B, WIDTH, dtype=torch.bfloat16, device="cuda")
    y = torch.empty(pool, B, dtype=torch.int32, device="cuda")
    for j in range(pool):
        tps.fill_synthetic(0, 1, 0x10000 + j, B, WIDTH, 0, x[j], cur.cuda_stream)
        tps.fill_synthetic(2, 1, 0x20000 + j, B, 1, CLASSES, y[j], cur.cuda_stream)
    torch.cuda.synchronize()
    fl_c2 = sum(2.0 * dims[l] * dims[l + 1] * (3 if l > 0 else 2) for l in range(len(dims) - 1))

    def timed(stages, n_windows, xp=None):
        xp = x if xp is None else xp
        mb = 0
        tps.run_schedule_local(stages, mb, epoch, xp, y, pool)         # warm-up epoch
        mb += epoch
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(n_windows + 1)]
        ev[0].record()
        for i in range(n_windows):
            tps.run_schedule_local(stages, mb, epoch, xp, y, pool)
            mb += epoch
            for st in stages:
                st.join(cur.cuda_stream)                                  # stream-ordered end of the window
            ev[i + 1].record()
        torch.cuda.synchronize()
        v = sorted(epoch * B / (ev[i].elapsed_time(ev[i + 1]) / 1e3) for i in range(n_windows))
        return {"median": statistics.median(v), "min": v[0], "max": v[-1], "windows": n_windows,
                "unit": "samples/s"}

    out = {"workload": "C2 (BASELINE.json configs[1]): 8 x Linear(4096,4096)+ReLU + head, S = 4 stages as LOCAL "
                       "handles on ONE GPU, m = 8 x b = 64, staleness 3/2/1/0 by stage, SGD momentum 0.9, "
                       f"lambda {LAM}; {epoch}-mini-batch windows",
           "flops_per_sample": fl_c2, "variants": {}}
    for name, var, blend in (("V", tps.TPS_V, tps.TPS_BLEND_EQ1), ("I-EQ1", tps.TPS_I, tps.TPS_BLEND_EQ1),
                             ("I-CONVEX", tps.TPS_I, tps.TPS_BLEND_CONVEX)):
        torch.cuda.synchronize()
        torch.cuda.reset_peak_memory_stats()
        base = torch.cuda.memory_allocated()
        stages = [tps.Pipeline(tps.StageSpec(dims=dims, stage_bounds=bounds, stage_id=s, micro_batches=m,
                                             micro_batch_size=b, variant=var, blend=blend, lam=LAM, lr=LR, momentum=MU,
                                             transport=tps.TPS_TRANSPORT_LOCAL, seed=1, torch_alloc=True))
                  for s in range(4)]
        for st in stages:
            st.init_weights_synthetic()
        tps.local_link(stages)
        held = torch.cuda.memory_allocated() - base
        t = timed(stages, windows)
        deltas = sorted({(e.stage, e.delta) for st in stages for e in st.trace() if e.kind == 1})
        out["variants"][name] = {
            "samples_per_s": t, "tflops_median": fl_c2 * t["median"] / 1e12,
            "memory_measured_bytes_all_stages": int(torch.cuda.max_memory_allocated() - base),
            "memory_held_after_init_bytes": int(held),
            "per_stage_library_bytes": [st.memory_stats() for st in stages],
            "per_stage_stash_peak_bytes": [st.stash_info()[2] for st in stages],
            "max_delta_per_stage": [max(d for s_, d in deltas if s_ == s) for s in range(4)],
        }
        for st in stages:
            st.close()
    # the same C2 pipeline in tf32 storage (tps_config.dtype = TPS_TF32, reading Z28): I-EQ1,
    # fp32-container inputs (the synthetic inputs are exact in both precisions)
    xf = x.float()
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats()
    base = torch.cuda.memory_allocated()
    stages = [tps.Pipeline(tps.StageSpec(dims=dims, stage_bounds=bounds, stage_id=s, micro_batches=m, micro_batch_size=b,
                                         variant=tps.TPS_I, blend=tps.TPS_BLEND_EQ1, lam=LAM, lr=LR, momentum=MU,
                                         transport=tps.TPS_TRANSPORT_LOCAL, seed=1, torch_alloc=True,
                                         dtype=tps.TPS_TF32))
              for s in range(4)]
    for st in stages:
        st.init_weights_synthetic()
    tps.local_link(stages)
    t = timed(stages, windows, xf)
    out["tf32"] = {"variant": "I-EQ1", "samples_per_s": t, "tflops_median": fl_c2 * t["median"] / 1e12,
                   "memory_measured_bytes_all_stages": int(torch.cuda.max_memory_allocated() - base),
                   "per_stage_stash_peak_bytes": [st.stash_info()[2] for st in stages],
                   "note": "kind::tf32 stage GEMMs, activations / versions / gradients as tf32 in fp32 containers"}
    for st in stages:
        st.close()
    del xf
    # staleness sweep on one stage
    dims1 = [WIDTH, WIDTH, WIDTH, CLASSES]
    fl1 = sum(2.0 * dims1[l] * dims1[l + 1] * (3 if l > 0 else 2) for l in range(3))
    sweep = {}
    for name, blend in (("I-EQ1", tps.TPS_BLEND_EQ1), ("I-CONVEX", tps.TPS_BLEND_CONVEX)):
        for K in (1, 2, 3, 4):
            st = tps.Pipeline(tps.StageSpec(dims=dims1, stage_bounds=[0, 3], stage_id=0, micro_batches=m,
                                            micro_batch_size=b, variant=tps.TPS_I, blend=blend, lam=LAM, lr=LR,
                                            momentum=MU, seed=1, max_inflight=K))
            st.init_weights_synthetic()
            t = timed([st], windows)
            sweep[f"{name} delta={K - 1}"] = {"samples_per_s": t["median"], "tflops": fl1 * t["median"] / 1e12,
                                              "stash_bytes": st.stash_info()[2]}
            st.close()
    out["staleness_sweep"] = {"workload": "one C2 stage (2 x Linear(4096,4096) + head), S = 1 with K = delta+1 "
                                          "mini-batches in flight, m = 8 x b = 64", "results": sweep}
    return out


# ------------------------------------------------------------------ GPU leg
def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        args.gpus = world if world > 1 else args.gpus
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import torch
    import torch.distributed as dist

    from paper_2509_23241_b200 import tps

    if args.same_device:
        local = 0
    torch.cuda.set_device(local)
    S = world
    if world > 1:
        if args.same_device:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    red_dev = "cpu" if args.same_device else "cuda"
    dims, bounds = model(S)
    # a real (non-default) stream: the library enqueues its compute work on it and joins its
    # weight-gradient / optimizer streams into it at the end of every run, so CUDA events on it
    # bracket ALL of a step's device work.  (On the legacy default stream, handle 0, the library
    # would create its own non-blocking stream and events on stream 0 would time the host's
    # enqueue instead of the device.)  --prio-stream: high priority for the compute stream.
    torch.cuda.set_stream(torch.cuda.Stream(priority=-1 if args.prio_stream else 0))
    stream = torch.cuda.current_stream().cuda_stream
    assert stream != 0

    use_ipc = S > 1 and args.transport == "ipc"

    def fresh_ids():
        # an ncclUniqueId bootstraps exactly one communicator: new ids for every pipeline
        if S == 1 or use_ipc:
            return None
        obj = [b"".join(tps.nccl_unique_id() for _ in range(2 * (S - 1)))] if rank == 0 else [None]
        dist.broadcast_object_list(obj, src=0)
        return obj[0]

    def make(variant):
        ids = fresh_ids()
        spec = tps.StageSpec(dims=dims, stage_bounds=bounds, stage_id=rank, micro_batches=MICRO_M,
                             micro_batch_size=MICRO_B, fwd_group=args.fwd_group, variant=variant,
                             blend=tps.TPS_BLEND_EQ1, lam=LAM, lr=LR, momentum=MU,
                             transport=(tps.TPS_TRANSPORT_IPC if use_ipc else tps.TPS_TRANSPORT_NCCL) if S > 1
                             else tps.TPS_TRANSPORT_NONE,
                             nccl_ids=ids, device=local, seed=0, compute_stream=stream,
                             fuse_update=args.fuse_update, torch_alloc=not args.no_torch_alloc)
        p = tps.Pipeline(spec)
        p.init_weights_synthetic()
        if use_ipc:   # exchange descriptors with the neighbouring stages, map their buffers
            blobs = [None] * world
            dist.all_gather_object(blobs, p.ipc_export())
            p.ipc_connect(blobs[rank - 1] if rank > 0 else None, blobs[rank + 1] if rank < world - 1 else None)
            dist.barrier()
        return p

    B = MICRO_B * MICRO_M
    x_pool = y_pool = None
    if rank == 0:
        x_pool = torch.empty(POOL, B, WIDTH, dtype=torch.bfloat16, device="cuda")
        for j in range(POOL):
            tps.fill_synthetic(0, 0, 0x10000 + j, B, WIDTH, 0, x_pool[j], stream)
    if rank == S - 1:
        y_pool = torch.empty(POOL, B, dtype=torch.int32, device="cuda")
        for j in range(POOL):
            tps.fill_synthetic(2, 0, 0x20000 + j, B, 1, CLASSES, y_pool[j], stream)
    torch.cuda.synchronize()

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    def sum_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return t.item()

    def timed_epochs(p, steps, warmup, xp, yp, profile=False, clocks=None):
        """K timed steps (epochs) after W warm-up ones; CUDA events on the compute stream around
        every step (one window each), barrier + synchronize on both sides.  Returns the total
        device ms (max over ranks), the per-window ms (max over ranks), launches, clocks."""
        mb = p.next_mb if hasattr(p, "next_mb") else 0
        graph = None
        if args.graph and world == 1 and not profile:
            # the first warm-up epoch is captured (and run); every later epoch replays the graph
            graph = tps.Graph([p], mb, args.epoch_mb, xp, yp, POOL, stream)
            mb += args.epoch_mb
            warmup = max(0, warmup - 1)

        def step(mb_):
            if graph is not None:
                graph.replay()
            else:
                p.run_schedule(mb_, args.epoch_mb, xp, yp, POOL)

        for _ in range(warmup):
            step(mb)
            mb += args.epoch_mb
        barrier()
        if profile:
            p.set_profiling(True)
        n0 = p.launch_count()
        if clocks:
            clocks.start()
        barrier()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
        ev[0].record()
        for i in range(steps):
            step(mb)
            mb += args.epoch_mb
            ev[i + 1].record()
        barrier()
        ck = clocks.stop() if clocks else None
        p.next_mb = mb
        ms = max_over_ranks(ev[0].elapsed_time(ev[-1]))
        win = [max_over_ranks(ev[i].elapsed_time(ev[i + 1])) for i in range(steps)]
        launches = sum_over_ranks(p.launch_count() - n0)
        if graph is not None:
            graph.close()
        return ms, win, launches, ck

    def spread(win_ms, samples):
        v = sorted(samples / (w / 1e3) for w in win_ms)
        return {"windows": len(v), "median": statistics.median(v), "min": v[0], "max": v[-1],
                "rel_spread": (v[-1] - v[0]) / statistics.median(v), "unit": "samples/s"}

    samples_per_step = args.epoch_mb * B
    # ---- I-TiMePReSt (headline)
    torch.cuda.reset_peak_memory_stats()
    pI = make(tps.TPS_I)
    clocks = ClockSampler(local)
    ms, winI, launches, ck = timed_epochs(pI, args.steps, args.warmup, x_pool, y_pool, clocks=clocks)
    value = samples_per_step * args.steps / (ms / 1e3)
    spreadI = spread(winI, samples_per_step)
    # second timed region with CUDA events around every GEMM / update launch on the compute
    # stream (the events add small gaps, so the headline value above is taken without them)
    ms_prof, _, _, _ = timed_epochs(pI, max(1, args.steps // 2), 0, x_pool, y_pool, profile=True)
    # per-kernel stats (GEMMs on the compute stream, CUDA events around every launch)
    n_g, ms_g, fl_g = pI.kernel_stats(3)
    per_kind = {}
    for kind, nm in ((0, "fwd"), (1, "dgrad"), (2, "wgrad" + ("+update" if args.fuse_update else ""))):
        n_k, ms_k, fl_k = pI.kernel_stats(kind)
        if n_k:
            per_kind[nm] = {"launches": n_k, "ms": round(ms_k, 3), "tflops": round(fl_k / (ms_k * 1e-3) / 1e12, 1)}
    n_u, ms_u, by_u = pI.kernel_stats(4)
    peaks_early, _ = load_peaks()
    # dominant kernel: the fused wgrad + update (17 weight-gradient launches per mini-batch: 16 x
    # 4096^2 fused, and the 16-row head, whose tiles cannot fill the GPU, as a split-K weight
    # gradient with its update in a separate kernel -- its update bytes are < 0.5 % of the sum);
    # algorithmic bytes per launch = G and X read once + 18 B/param (w, v read + write, bf16
    # version), averaged over the 17 launches like the measured duration
    n_w, ms_w, fl_w = pI.kernel_stats(2)
    Bm = MICRO_B * MICRO_M
    dmod = [WIDTH] * (HIDDEN + 1) + [CLASSES]
    lay = [(((dmod[l + 1] + 15) // 16) * 16, ((dmod[l] + 15) // 16) * 16) for l in range(len(dmod) - 1)]
    dom_bytes = sum(2.0 * Bm * (npad + kpad) + 18.0 * npad * kpad for npad, kpad in lay) / len(lay)
    dom_flops = sum(2.0 * Bm * npad * kpad for npad, kpad in lay) / len(lay)
    dom_us = ms_w / n_w * 1e3 if n_w else None
    dom = {"bytes": dom_bytes, "flops": dom_flops, "us": dom_us,
           "gbs": dom_bytes / (dom_us * 1e-6) / 1e9 if dom_us else None,
           "roof_us": max(dom_flops / (peaks_early.get("bf16_tflops_sustained", 1400.0) * 1e12),
                          dom_bytes / (peaks_early.get("hbm_gbs", 6500.0) * 1e9)) * 1e6}
    memI = pI.memory_stats()
    memI["torch_max_allocated"] = int(torch.cuda.max_memory_allocated())   # device-observed (allocator hook)
    lossesI = pI.losses()
    peaks, src = load_peaks()
    achieved = (fl_g / n_g) / (ms_g / n_g * 1e-3) / 1e12 if n_g else None
    peak = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops"))
    # whole-step tensor fraction and per-rank GEMM time share
    gemm_share = max_over_ranks(ms_g / max(ms_prof, 1e-9)) if n_g else None
    traffic = None
    tr_path = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tr_path):
        try:
            traffic = json.load(open(tr_path)).get("gemm_bytes_per_launch")
        except Exception:
            traffic = None

    # per-kind tensor-pipe / DRAM utilisation from the committed ncu --set full capture (one
    # launch of each stage-GEMM kind at these shapes; read, not measured, by this run)
    ncu_kinds = None
    ncu_path = os.path.join(ROOT, "profiles", "r02_ncu_full_summary.json")
    if os.path.exists(ncu_path):
        try:
            # gemm_kernel<BN, A_MN, B_MN, BLEND, SGD, CG, CONV, MH, TF>
            names = {"<256, 1, 1, 0, 1, 2, 0, 1, 0>": "wgrad+update", "<256, 0, 0, 0, 0, 2, 0, 1, 0>": "fwd",
                     "<256, 0, 1, 0, 0, 2, 0, 1, 0>": "dgrad", "<256, 0, 1, 1, 0, 2, 0, 2, 0>": "dgrad_blend"}
            ncu_kinds = {"source": "profiles/r02_ncu_full_summary.json (ncu --set full --clock-control none)"}
            for r in json.load(open(ncu_path)):
                for key, kind in names.items():
                    if key in r["kernel"]:
                        ncu_kinds[kind] = {"time_us": r["time_us"], "tensor_pipe_pct": r["tensor_pipe_pct"],
                                           "dram_pct": r["dram_pct"],
                                           "dram_bytes": round((r["dram_read_MB"] + r["dram_write_MB"]) * 1e6)}
        except Exception:
            ncu_kinds = None

    pI.set_profiling(False)   # per-launch events off again (they also cannot be captured)

    # ---- e2e: host pools (pinned), H2D inside the timed region, D2H of losses
    e2e = None
    if not args.no_e2e:
        hx = x_pool.cpu().pin_memory() if x_pool is not None else None
        hy = y_pool.cpu().pin_memory() if y_pool is not None else None
        lossbuf = torch.empty(args.steps * args.epoch_mb, dtype=torch.float32).pin_memory()
        use_graph = bool(args.graph) and world == 1
        g_e2e = None
        if use_graph:   # the warm-up epoch is captured with the host pools (H2D copies are graph nodes)
            g_e2e = tps.Graph([pI], pI.next_mb, args.epoch_mb, hx, hy, POOL, stream)
        else:
            pI.run_schedule(pI.next_mb, args.epoch_mb, hx, hy, POOL)   # warm the host path
        pI.next_mb += args.epoch_mb
        barrier()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        n_loss0 = len(pI.losses()) if rank == S - 1 else 0
        t0.record()
        for i in range(args.steps):
            if g_e2e is not None:
                g_e2e.replay()
            else:
                pI.run_schedule(pI.next_mb, args.epoch_mb, hx, hy, POOL)
            pI.next_mb += args.epoch_mb
            if rank == S - 1:   # device -> host read of the step's result (its losses), stream-ordered
                pI.read_losses_async(n_loss0 + i * args.epoch_mb, args.epoch_mb,
                                     lossbuf[i * args.epoch_mb:], stream)
        t1.record()
        barrier()
        if g_e2e is not None:
            g_e2e.close()
        if rank == S - 1:
            assert torch.isfinite(lossbuf).all(), "non-finite loss in the e2e run"
        ms_e = max_over_ranks(t0.elapsed_time(t1))
        h2d = (args.epoch_mb * B * WIDTH * 2 if rank == 0 else 0) + (args.epoch_mb * B * 4 if rank == S - 1 else 0)
        e2e = {"value": samples_per_step * args.steps / (ms_e / 1e3), "unit": "samples/s",
               "h2d_bytes_per_step": int(sum_over_ranks(h2d)), "d2h_bytes_per_step": 4 * args.epoch_mb,
               "api": ("tps_graph_replay of an epoch captured with pinned host x/y pools" if use_graph else
                       "tps_run_schedule with pinned host x/y pools") +
                      "; per step the H2D copies of its inputs and an async D2H read of its losses"}
    pI.close()

    # ---- V-TiMePReSt (memory + throughput)
    v_out = None
    if not args.no_v:
        torch.cuda.synchronize()
        torch.cuda.reset_peak_memory_stats()
        pV = make(tps.TPS_V)
        msV, winV, _, _ = timed_epochs(pV, args.steps, 1, x_pool, y_pool)
        memV = pV.memory_stats()
        memV["torch_max_allocated"] = int(torch.cuda.max_memory_allocated())
        v_out = {"value": samples_per_step * args.steps / (msV / 1e3), "unit": "samples/s",
                 "spread": spread(winV, samples_per_step), "mem_bytes": memV}
        pV.close()

    mem_all = [{"I": memI, "V": v_out["mem_bytes"] if v_out else None}]
    if world > 1:
        mem_all = [None] * world
        dist.all_gather_object(mem_all, {"I": memI, "V": v_out["mem_bytes"] if v_out else None})
    method = None
    if world == 1 and not args.no_method:
        method = method_leg(torch, tps)
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            v, dt, cores, desc = oracle_sample(rows_m=4)
            cpu = {"value": v, "unit": "samples/s", "cores": cores, "kind": "oracle", "sample": desc,
                   "seconds": dt}
        fps = flops_per_sample()
        line = {
            "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic (splitmix64 inputs, random labels, "
            "synthetic-init weights)", "config": config_dict(args),
            # the stage GEMMs are ~all of the step and, with the split backward, the weight-gradient
            # GEMMs overlap the input-gradient GEMMs on a second stream: per-launch event durations
            # then include SM sharing, so the roofline uses the algorithmic GEMM FLOPs of the whole
            # timed step over its device time (per-launch event numbers kept under per_kind)
            # the dominant kernel: wgrad + fused SGD/momentum update (HBM-bound: its roofline time
            # max(FLOPs / tensor peak, algorithmic bytes / HBM peak) is the HBM term); achieved =
            # algorithmic bytes per launch / average launch duration (CUDA events on its stream)
            "roofline": {"bound": "hbm", "kernel": "wgrad + fused SGD/momentum update, gemm_kernel<256,1,1,0,1,2,0,1,0> "
                         "(CTA pairs, 256x256 tiles with a split tail, TMA-fed update epilogue)",
                         "achieved": dom["gbs"], "peak": peaks.get("hbm_gbs"), "unit": "GB/s",
                         "frac": dom["gbs"] / peaks.get("hbm_gbs") if dom["gbs"] else None, "traffic": traffic,
                         "algorithmic_bytes_per_launch": dom["bytes"], "flops_per_launch": dom["flops"],
                         "avg_launch_us": dom["us"], "roofline_time_us": dom["roof_us"],
                         "frac_of_roofline_time": dom["roof_us"] / dom["us"] if dom["us"] else None,
                         "isolated": "tools/gemm_bench.py --modes 4 (same kernel alone): 84.1 us at 1965 MHz = 0.57 "
                                     "of its HBM roofline time, 96.0 us sustained under the power cap "
                                     "(profiles/r02_gemm_microbench.txt, r02_fused_kernel_variants.txt)",
                         "launch_note": "in the pipeline each launch runs concurrently with the next layer's input "
                                        "gradient on the compute stream (split backward), so its event duration "
                                        "includes SM sharing",
                         "step_tensor_achieved_tflops": fps * value / world / 1e12,
                         "per_launch_event_tflops": achieved,
                         "per_launch_note": "per_kind / per_launch_event_tflops: CUDA-event durations of each "
                         "launch on its own stream; they overlap across the two backward streams",
                         "frac_of_burst_peak": fps * value / world / 1e12 / peaks["bf16_tflops"],
                         "peak_source": f"{src} bf16_tflops_sustained (MEASURED_PEAKS.json)",
                         "gemm_launches": n_g, "gemm_ms": ms_g, "gemm_share_of_step": gemm_share,
                         "per_kind": per_kind, "ncu_per_kind": ncu_kinds,
                         "step_tensor_frac": fps * value / world / 1e12 / peak,
                         "update_kernel": {"bound": "hbm", "achieved_gbs": (by_u / (ms_u * 1e-3) / 1e9) if n_u else None,
                                           "peak_gbs": peaks.get("hbm_gbs"), "launches": n_u, "ms": ms_u}},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
            "clocks": ck, "memory_per_gpu": mem_all, "v_variant": {k: v for k, v in (v_out or {}).items()
                                                                   if k != "mem_bytes"},
            "losses_first_last": [float(lossesI[0]), float(lossesI[-1])] if len(lossesI) else None,
            "spread": spreadI,
            "peaks": {"bf16_tflops_burst": peaks.get("bf16_tflops"), "bf16_tflops_sustained": peak,
                      "hbm_gbs": peaks.get("hbm_gbs"), "source": src,
                      "measured_at_sm_mhz": (peaks.get("clocks_under_load") or {}).get("sm_mhz_median"),
                      "bench_sm_mhz": (ck or {}).get("sm_mhz")},
            "method": method,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

"""Thin ctypes binding of include/tps.h — argument marshalling only.

Every step of the training path runs inside libtps.so (the sm_100a kernels and the C++
runtime).  Nothing here computes: if the library is missing the import of `lib()`
raises, and the library itself refuses to run without an sm_100 device (TPS_E_ARCH) —
there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TPS_LIB") or os.path.join(HERE, "lib", "libtps.so")

TPS_V, TPS_I = 0, 1
TPS_BLEND_EQ1, TPS_BLEND_CONVEX = 0, 1
TPS_BF16, TPS_TF32 = 0, 1            # tps_dtype (storage precision, reading Z28)
TPS_GEMM_TF32 = 16                   # tps_gemm mode flag: tf32 operands in fp32 containers
TPS_TRANSPORT_NONE, TPS_TRANSPORT_LOCAL, TPS_TRANSPORT_NCCL, TPS_TRANSPORT_IPC = 0, 1, 2, 3
TPS_IPC_BLOB_BYTES = 2048
TPS_EV_F, TPS_EV_B, TPS_EV_U = 0, 1, 2
GEMM_FWD, GEMM_DGRAD, GEMM_WGRAD, GEMM_DGRAD_BLEND = 0, 1, 2, 3
STATUS = {0: "TPS_OK", 1: "TPS_E_INVALID_ARG", 2: "TPS_E_CONFIG", 3: "TPS_E_ORDER", 4: "TPS_E_STALENESS",
          5: "TPS_E_CUDA", 6: "TPS_E_NCCL", 7: "TPS_E_OOM", 8: "TPS_E_ARCH", 9: "TPS_E_STATE",
          10: "TPS_E_UNSUPPORTED"}

# every symbol include/tps.h declares (tests check the .so exports all of them)
EXPORTS = [
    "tps_abi_version", "tps_last_error", "tps_nccl_unique_id", "tps_pipeline_init", "tps_pipeline_destroy",
    "tps_local_link", "tps_begin_run", "tps_stage_forward", "tps_stage_backward", "tps_stage_update",
    "tps_run_schedule", "tps_run_schedule_local", "tps_synchronize", "tps_blend_coeffs", "tps_stash_info",
    "tps_intermediate_weight", "tps_get_version", "tps_schedule_events", "tps_get_weights", "tps_set_weights",
    "tps_init_weights_synthetic", "tps_get_losses", "tps_get_trace", "tps_clear_trace", "tps_memory_stats",
    "tps_set_profiling", "tps_kernel_stats", "tps_launch_count", "tps_fill_synthetic", "tps_gemm",
    "tps_conv_gemm", "tps_partition", "tps_im2col", "tps_col2im", "tps_bn_forward", "tps_bn_backward",
    "tps_pool_op", "tps_conv2d_gemm", "tps_debug_progress", "tps_memory_observed", "tps_join", "tps_ipc_export", "tps_ipc_connect",
    "tps_dp_export", "tps_dp_connect", "tps_gemm_wgrad_sgd", "tps_graph_capture", "tps_graph_replay",
    "tps_graph_destroy", "tps_read_losses_async", "tps_set_timeline", "tps_get_timeline",
    "tps_gemm_bwd_dual",
]
TPS_LAYER_LINEAR, TPS_LAYER_CONV3X3, TPS_LAYER_MAXPOOL2 = 0, 1, 2
TPS_LAYER_CONV, TPS_LAYER_BN, TPS_LAYER_MAXPOOL3, TPS_LAYER_AVGPOOL = 3, 4, 5, 6


class TpsError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class Event(C.Structure):
    _fields_ = [("stage", C.c_int32), ("kind", C.c_int32), ("micro", C.c_int32), ("micro_count", C.c_int32),
                ("mb", C.c_int64), ("v_used", C.c_int64), ("v_latest", C.c_int64), ("delta", C.c_int32),
                ("alpha", C.c_float), ("beta", C.c_float)]


class TimelineRec(C.Structure):
    _fields_ = [("ev", Event), ("t0_ms", C.c_double), ("t1_ms", C.c_double)]


class Layer(C.Structure):
    _fields_ = [("kind", C.c_int32), ("in_c", C.c_int32), ("out_c", C.c_int32), ("in_h", C.c_int32),
                ("in_w", C.c_int32), ("k", C.c_int32), ("stride", C.c_int32), ("pad", C.c_int32),
                ("src_back", C.c_int32), ("res_back", C.c_int32), ("relu", C.c_int32), ("reserved", C.c_int32 * 5)]


class Config(C.Structure):
    _fields_ = [("num_layers", C.c_int32), ("dims", C.POINTER(C.c_int32)), ("num_stages", C.c_int32),
                ("stage_bounds", C.POINTER(C.c_int32)), ("stage_id", C.c_int32), ("micro_batches", C.c_int32),
                ("micro_batch_size", C.c_int32), ("fwd_group", C.c_int32), ("variant", C.c_int32),
                ("blend", C.c_int32), ("lambda_", C.c_double), ("lr", C.c_float), ("momentum", C.c_float),
                ("weight_decay", C.c_float), ("transport", C.c_int32), ("nccl_ids", C.c_void_p),
                ("device", C.c_int32), ("seed", C.c_uint64), ("compute_stream", C.c_uint64),
                ("extra_recv_slot", C.c_int32), ("fuse_update", C.c_int32),
                ("num_layer_specs", C.c_int32), ("layer_specs", C.POINTER(Layer)),
                ("max_inflight", C.c_int32), ("staleness_mode", C.c_int32),
                ("dev_alloc", C.c_void_p), ("dev_free", C.c_void_p), ("alloc_ctx", C.c_void_p),
                ("dp_size", C.c_int32), ("dp_rank", C.c_int32), ("dtype", C.c_int32), ("reserved", C.c_int32)]


# tps_config.dev_alloc / dev_free signatures
ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p)
FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p)


class TorchAllocator:
    """dev_alloc / dev_free hooks backed by PyTorch's caching allocator, so the handle's
    buffers show up in torch.cuda.memory_allocated / max_memory_allocated (per-GPU peak
    memory, BASELINE metric).  Marshalling only: the callbacks forward to torch."""

    def __init__(self, device: int):
        import torch
        self.device = device

        def _alloc(nbytes, _ctx):
            try:
                return torch.cuda.caching_allocator_alloc(int(nbytes), self.device)
            except Exception:
                return None

        def _free(p, _ctx):
            torch.cuda.caching_allocator_delete(p)

        self.alloc = ALLOC_FN(_alloc)   # keep the ctypes thunks alive with the handle
        self.free = FREE_FN(_free)


_LIB = None


def lib() -> C.CDLL:
    """Load libtps.so (built by __graft_entry__.build()); raises if it is missing."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        P, I32, I64, U64, F, D = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_float, C.c_double
        sig = {
            "tps_abi_version": (I32, []),
            "tps_last_error": (C.c_char_p, []),
            "tps_nccl_unique_id": (I32, [P]),
            "tps_pipeline_init": (I32, [C.POINTER(Config), C.POINTER(P)]),
            "tps_pipeline_destroy": (I32, [P]),
            "tps_local_link": (I32, [C.POINTER(P), I32]),
            "tps_begin_run": (I32, [P, I64, I64]),
            "tps_stage_forward": (I32, [P, I64, I32, I32, P, P]),
            "tps_stage_backward": (I32, [P, I64, I32]),
            "tps_stage_update": (I32, [P, I64]),
            "tps_run_schedule": (I32, [P, I64, I64, P, P, I32]),
            "tps_run_schedule_local": (I32, [C.POINTER(P), I32, I64, I64, P, P, I32]),
            "tps_synchronize": (I32, [P]),
            "tps_blend_coeffs": (I32, [I32, I32, I32, D, C.POINTER(F), C.POINTER(F)]),
            "tps_stash_info": (I32, [P, C.POINTER(I32), C.POINTER(I64), C.POINTER(I64)]),
            "tps_intermediate_weight": (I32, [P, I32, I32, P]),
            "tps_get_version": (I32, [P, I32, I32, P]),
            "tps_schedule_events": (I32, [I32, I32, I32, I32, I64, C.POINTER(Event), I64, C.POINTER(I64)]),
            "tps_get_weights": (I32, [P, I32, P, P, P, P]),
            "tps_set_weights": (I32, [P, I32, P, P]),
            "tps_init_weights_synthetic": (I32, [P]),
            "tps_get_losses": (I32, [P, P, I64, C.POINTER(I64)]),
            "tps_get_trace": (I32, [P, C.POINTER(Event), I64, C.POINTER(I64)]),
            "tps_clear_trace": (I32, [P]),
            "tps_memory_stats": (I32, [P] + [C.POINTER(I64)] * 6),
            "tps_set_profiling": (I32, [P, I32]),
            "tps_set_timeline": (I32, [P, I32, U64]),
            "tps_get_timeline": (I32, [P, C.POINTER(TimelineRec), I64, C.POINTER(I64)]),
            "tps_kernel_stats": (I32, [P, I32, C.POINTER(I64), C.POINTER(D), C.POINTER(D)]),
            "tps_launch_count": (I32, [P, C.POINTER(I64)]),
            "tps_fill_synthetic": (I32, [I32, U64, U64, I64, I64, I32, P, U64]),
            "tps_gemm": (I32, [I32, I32, I32, I32, P, I32, P, I32, P, P, I32, I32, P, I32, F, F, P, I32, U64]),
            "tps_conv_gemm": (I32, [I32, I32, I32, I32, I32, I32, P, P, P, P, I32, P, I32, F, F, P, U64]),
            "tps_partition": (I32, [I32, P, P, P, I32, I32, I32, I32, P, P]),
            "tps_im2col": (I32, [P, P, I32, I32, I32, I32, I32, I32, I32, I32, U64]),
            "tps_col2im": (I32, [P, P, P, I32, I32, I32, I32, I32, I32, I32, I32, U64]),
            "tps_bn_forward": (I32, [P, P, P, P, P, P, P, I32, I32, I32, I32, U64]),
            "tps_bn_backward": (I32, [P, P, P, P, P, P, P, F, F, I32, I32, I32, I32, P, P, P, P, U64]),
            "tps_pool_op": (I32, [I32, P, P, P, I32, I32, I32, I32, U64]),
            "tps_debug_progress": (I32, [P, P, P, P]),
            "tps_conv2d_gemm": (I32, [I32, I32, I32, I32, I32, I32, I32, I32, I32, P, P, P, P, I32, F, F, U64]),
            "tps_memory_observed": (I32, [P, C.POINTER(I64)]),
            "tps_join": (I32, [P, U64]),
            "tps_ipc_export": (I32, [P, P, I64, C.POINTER(I64)]),
            "tps_ipc_connect": (I32, [P, P, P]),
            "tps_gemm_wgrad_sgd": (I32, [I32, I32, I32, P, I32, P, I32, P, P, P, I32, F, F, F, U64]),
            "tps_gemm_bwd_dual": (I32, [I32, I32, I32, P, I32, P, I32, P, P, P, I32, F, F, F,
                                        I32, I32, I32, P, I32, P, I32, P, I32, F, P, I32, U64]),
            "tps_graph_capture": (I32, [C.POINTER(P), I32, I64, I64, P, P, I32, U64, C.POINTER(P)]),
            "tps_graph_replay": (I32, [P]),
            "tps_graph_destroy": (I32, [P]),
            "tps_read_losses_async": (I32, [P, I64, I64, P, U64]),
            "tps_dp_export": (I32, [P, P, I64, C.POINTER(I64)]),
            "tps_dp_connect": (I32, [P, C.POINTER(P), I32]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = L
    return _LIB


def check(status: int) -> None:
    if status != 0:
        raise TpsError(status, lib().tps_last_error().decode())


def ptr(t) -> int | None:
    """Address of a torch tensor / numpy array / None."""
    if t is None:
        return None
    if hasattr(t, "data_ptr"):
        return t.data_ptr()
    return t.ctypes.data


# ------------------------------------------------------------------ free functions
def blend_coeffs(variant: int, blend: int, staleness: int, lam: float) -> tuple[float, float]:
    a, b = C.c_float(), C.c_float()
    check(lib().tps_blend_coeffs(variant, blend, staleness, lam, C.byref(a), C.byref(b)))
    return a.value, b.value


def schedule_events(S: int, s: int, m: int, fwd_group: int, M: int) -> list[Event]:
    n = C.c_int64()
    check(lib().tps_schedule_events(S, s, m, fwd_group, M, None, 0, C.byref(n)))
    buf = (Event * n.value)()
    check(lib().tps_schedule_events(S, s, m, fwd_group, M, buf, n.value, C.byref(n)))
    return list(buf)


def nccl_unique_id() -> bytes:
    b = C.create_string_buffer(128)
    check(lib().tps_nccl_unique_id(b))
    return b.raw


def fill_synthetic(kind: int, seed: int, tid: int, rows: int, cols: int, classes: int, dst, stream: int = 0) -> None:
    check(lib().tps_fill_synthetic(kind, seed, tid, rows, cols, classes, ptr(dst), stream))


def gemm(mode, M, N, K, A, lda, B, ldb, out, ldo, out_f32=0, bias=None, relu=0, alpha=1.0, beta=0.0,
         mask=None, ldm=0, B2=None, stream: int = 0) -> None:
    check(lib().tps_gemm(mode, M, N, K, ptr(A), lda, ptr(B), ldb, ptr(B2), ptr(out), ldo, out_f32, ptr(bias), relu,
                         alpha, beta, ptr(mask), ldm, stream))


def gemm_wgrad_sgd(M, N, K, A, lda, B, ldb, w, v, ver, ldw, lr, mu, wd=0.0, stream: int = 0) -> None:
    check(lib().tps_gemm_wgrad_sgd(M, N, K, ptr(A), lda, ptr(B), ldb, ptr(w), ptr(v), ptr(ver), ldw, lr, mu, wd,
                                   stream))


def gemm_bwd_dual(M, N, K, A, lda, B, ldb, w, v, ver, ldw, lr, mu, wd, Md, Nd, Kd, Ad, ldad, Bd, ldbd, outd, ldod,
                  alpha=1.0, mask=None, ldm=0, stream: int = 0) -> None:
    """One launch: gemm_wgrad_sgd(M, N, K, ...) and the masked input gradient outd = α·Ad·Bd (mode 1)."""
    check(lib().tps_gemm_bwd_dual(M, N, K, ptr(A), lda, ptr(B), ldb, ptr(w), ptr(v), ptr(ver), ldw, lr, mu, wd,
                                  Md, Nd, Kd, ptr(Ad), ldad, ptr(Bd), ldbd, ptr(outd), ldod, alpha, ptr(mask), ldm,
                                  stream))


def conv_gemm(mode, N, H, W, Ci, Co, A, Wt, out, out_f32=0, bias=None, relu=0, alpha=1.0, beta=0.0, mask=None,
              W2=None, stream: int = 0) -> None:
    check(lib().tps_conv_gemm(mode, N, H, W, Ci, Co, ptr(A), ptr(Wt), ptr(W2), ptr(out), out_f32, ptr(bias), relu,
                              alpha, beta, ptr(mask), stream))


def conv2d_gemm(mode, N, H, W, Ci, Co, k, stride, pad, A, Wt, out, out_f32=0, alpha=1.0, beta=0.0, W2=None,
                stream: int = 0) -> None:
    check(lib().tps_conv2d_gemm(mode, N, H, W, Ci, Co, k, stride, pad, ptr(A), ptr(Wt), ptr(W2), ptr(out), out_f32,
                                alpha, beta, stream))


def im2col(X, P, N, H, W, C, k, stride, pad, ldp, stream: int = 0) -> None:
    check(lib().tps_im2col(ptr(X), ptr(P), N, H, W, C, k, stride, pad, ldp, stream))


def col2im(dP, dX, add, N, H, W, C, k, stride, pad, ldp, stream: int = 0) -> None:
    check(lib().tps_col2im(ptr(dP), ptr(dX), ptr(add), N, H, W, C, k, stride, pad, ldp, stream))


def bn_forward(x, res, y, gamma, beta, mean, invstd, segs, seg_rows, C, relu, stream: int = 0) -> None:
    check(lib().tps_bn_forward(ptr(x), ptr(res), ptr(y), ptr(gamma), ptr(beta), ptr(mean), ptr(invstd), segs, seg_rows,
                               C, relu, stream))


def bn_backward(dy, y, x, mean, invstd, g_stash, g_latest, a, b, segs, seg_rows, C, relu, dx, dres, dgamma, dbeta,
                stream: int = 0) -> None:
    check(lib().tps_bn_backward(ptr(dy), ptr(y), ptr(x), ptr(mean), ptr(invstd), ptr(g_stash), ptr(g_latest), a, b,
                                segs, seg_rows, C, relu, ptr(dx), ptr(dres), ptr(dgamma), ptr(dbeta), stream))


def pool_op(op, a, b, out, N, H, W, C, stream: int = 0) -> None:
    check(lib().tps_pool_op(op, ptr(a), ptr(b), ptr(out), N, H, W, C, stream))


def partition(param_bytes, act_bytes, flops, S: int, variant: int = TPS_I, momentum: bool = True,
              objective: int = 0):
    """Balanced consecutive stage partition (C++ DP in libtps); returns (bounds, stage costs)."""
    import numpy as np
    L = len(param_bytes if param_bytes is not None else flops)
    arrs = [None if a is None else np.ascontiguousarray(a, dtype=np.float64) for a in (param_bytes, act_bytes, flops)]
    bounds = np.zeros(S + 1, np.int32)
    cost = np.zeros(S, np.float64)
    check(lib().tps_partition(L, *[None if a is None else a.ctypes.data for a in arrs], S, variant,
                              1 if momentum else 0, objective, bounds.ctypes.data, cost.ctypes.data))
    return bounds.tolist(), cost.tolist()


def layer_specs(specs: list[dict]):
    """oracle-style layer dicts -> ctypes tps_layer array."""
    arr = (Layer * len(specs))()
    for i, sp in enumerate(specs):
        back = i - sp.get("src", i - 1)          # graph layers name their input by global index
        k = sp["kind"]
        if k == "linear":
            arr[i] = Layer(TPS_LAYER_LINEAR, sp["in"], sp["out"], 1, 1, src_back=back)
        elif k == "conv3":
            arr[i] = Layer(TPS_LAYER_CONV3X3, sp["cin"], sp["cout"], sp["h"], sp["w"])
        elif k == "pool2":
            arr[i] = Layer(TPS_LAYER_MAXPOOL2, sp["c"], sp["c"], sp["h"], sp["w"])
        elif k == "conv":
            arr[i] = Layer(TPS_LAYER_CONV, sp["cin"], sp["cout"], sp["h"], sp["w"], sp["k"], sp["s"], sp["p"],
                           src_back=back)
        elif k == "bn":
            res = sp.get("res")
            arr[i] = Layer(TPS_LAYER_BN, sp["c"], sp["c"], sp["h"], sp["w"], src_back=back,
                           res_back=(i - res) if res is not None else 0, relu=1 if sp.get("relu") else 0)
        elif k == "maxpool3":
            arr[i] = Layer(TPS_LAYER_MAXPOOL3, sp["c"], sp["c"], sp["h"], sp["w"], src_back=back)
        elif k == "avgpool":
            arr[i] = Layer(TPS_LAYER_AVGPOOL, sp["c"], sp["c"], sp["h"], sp["w"], src_back=back)
        else:
            raise ValueError(f"layer {i}: unknown kind {k!r}")
    return arr


def layer_param_shape(sp: dict):
    """Logical [out, in] of a layer's weight as tps_get_weights returns it (None: no parameters)."""
    k = sp["kind"]
    if k == "conv3":
        return (sp["cout"], 9 * sp["cin"])
    if k == "conv":
        return (sp["cout"], sp["k"] * sp["k"] * sp["cin"])
    if k == "bn":
        return (sp["c"], 1)
    if k == "linear":
        return (sp["out"], sp["in"])
    return None


# ------------------------------------------------------------------ handle wrapper
@dataclass
class StageSpec:
    dims: list[int]
    stage_bounds: list[int]
    stage_id: int
    micro_batches: int
    micro_batch_size: int
    fwd_group: int = 0
    variant: int = TPS_I
    blend: int = TPS_BLEND_EQ1
    lam: float = 0.05
    lr: float = 0.01
    momentum: float = 0.0
    weight_decay: float = 0.0
    transport: int = TPS_TRANSPORT_NONE
    nccl_ids: bytes | None = None
    device: int = 0
    seed: int = 0
    compute_stream: int = 0
    extra_recv_slot: int = 1
    fuse_update: int = 1
    layers: list | None = None       # oracle-style layer dicts (image nets); None => MLP from dims
    max_inflight: int = 0            # 0 => S - s; S = 1 only otherwise (staleness sweep on one GPU)
    staleness_mode: int = 0          # 1 => explicit δ may be any live version (microbenchmark)
    torch_alloc: bool = False        # allocate through PyTorch's caching allocator
    dp_size: int = 1                 # data-parallel replicas of the pipeline (NEXT-2)
    dp_rank: int = 0
    dtype: int = TPS_BF16            # TPS_TF32: activations / versions / gradients as tf32 (fp32 containers)
    _keep: list = field(default_factory=list)


class Pipeline:
    """One pipeline stage (tps_pipeline*)."""

    def __init__(self, spec: StageSpec):
        self.spec = spec
        if spec.layers:
            L = len(spec.layers)
            s0 = spec.layers[0]
            feat = s0["h"] * s0["w"] * s0["cin"] if s0["kind"] in ("conv3", "conv") else s0["in"]
            dvals = [feat] + [0] * (L - 1) + [spec.layers[-1]["out"]]
        else:
            L = len(spec.dims) - 1
            dvals = list(spec.dims)
        dims = (C.c_int32 * (L + 1))(*dvals)
        bounds = (C.c_int32 * len(spec.stage_bounds))(*spec.stage_bounds)
        ids = C.create_string_buffer(spec.nccl_ids, len(spec.nccl_ids)) if spec.nccl_ids else None
        specs = layer_specs(spec.layers) if spec.layers else None
        self._alloc = TorchAllocator(spec.device) if spec.torch_alloc else None
        cfg = Config(num_layers=L, dims=dims, num_stages=len(spec.stage_bounds) - 1, stage_bounds=bounds,
                     stage_id=spec.stage_id, micro_batches=spec.micro_batches,
                     micro_batch_size=spec.micro_batch_size, fwd_group=spec.fwd_group, variant=spec.variant,
                     blend=spec.blend, lambda_=spec.lam, lr=spec.lr, momentum=spec.momentum,
                     weight_decay=spec.weight_decay, transport=spec.transport,
                     nccl_ids=C.cast(ids, C.c_void_p) if ids is not None else None, device=spec.device,
                     seed=spec.seed, compute_stream=spec.compute_stream, extra_recv_slot=spec.extra_recv_slot,
                     fuse_update=spec.fuse_update, num_layer_specs=len(spec.layers) if spec.layers else 0,
                     layer_specs=specs, max_inflight=spec.max_inflight, staleness_mode=spec.staleness_mode,
                     dev_alloc=C.cast(self._alloc.alloc, C.c_void_p) if self._alloc else None,
                     dev_free=C.cast(self._alloc.free, C.c_void_p) if self._alloc else None,
                     dp_size=spec.dp_size, dp_rank=spec.dp_rank, dtype=spec.dtype)
        h = C.c_void_p()
        check(lib().tps_pipeline_init(C.byref(cfg), C.byref(h)))
        self.h = h
        self.S = len(spec.stage_bounds) - 1
        self.layers = list(range(spec.stage_bounds[spec.stage_id], spec.stage_bounds[spec.stage_id + 1]))
        self.shapes = []   # logical [out, in] of each stage-local layer (None for pools)
        for g in self.layers:
            if spec.layers:
                self.shapes.append(layer_param_shape(spec.layers[g]))
            else:
                self.shapes.append((spec.dims[g + 1], spec.dims[g]))

    def close(self):
        if self.h:
            check(lib().tps_pipeline_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # the step
    def begin_run(self, first_mb: int, n_mb: int):
        check(lib().tps_begin_run(self.h, first_mb, n_mb))

    def stage_forward(self, mb: int, micro: int, count: int, x=None, labels=None):
        check(lib().tps_stage_forward(self.h, mb, micro, count, ptr(x), ptr(labels)))

    def stage_backward(self, mb: int, staleness: int = -1):
        check(lib().tps_stage_backward(self.h, mb, staleness))

    def stage_update(self, mb: int):
        check(lib().tps_stage_update(self.h, mb))

    def run_schedule(self, first_mb: int, n_mb: int, x_pool=None, y_pool=None, pool: int = 1):
        check(lib().tps_run_schedule(self.h, first_mb, n_mb, ptr(x_pool), ptr(y_pool), pool))

    def synchronize(self):
        check(lib().tps_synchronize(self.h))

    def ipc_export(self) -> bytes:
        """This stage's IPC exchange descriptor (send it to the neighbouring stages)."""
        buf = C.create_string_buffer(TPS_IPC_BLOB_BYTES)
        n = C.c_int64()
        check(lib().tps_ipc_export(self.h, buf, TPS_IPC_BLOB_BYTES, C.byref(n)))
        return buf.raw[: n.value]

    def ipc_connect(self, prev: bytes | None, nxt: bytes | None):
        pb = C.create_string_buffer(prev, len(prev)) if prev else None
        nb = C.create_string_buffer(nxt, len(nxt)) if nxt else None
        check(lib().tps_ipc_connect(self.h, pb, nb))

    def dp_export(self) -> bytes:
        n = C.c_int64()
        check(lib().tps_dp_export(self.h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value)
        check(lib().tps_dp_export(self.h, buf, n.value, C.byref(n)))
        return buf.raw[: n.value]

    def dp_connect(self, blobs: list[bytes]):
        bufs = [C.create_string_buffer(b, len(b)) for b in blobs]
        arr = (C.c_void_p * len(bufs))(*[C.cast(b, C.c_void_p) for b in bufs])
        check(lib().tps_dp_connect(self.h, arr, len(bufs)))

    def join(self, stream: int):
        """`stream` waits (stream-ordered) for all work the handle has enqueued."""
        check(lib().tps_join(self.h, stream))

    # state
    def init_weights_synthetic(self):
        check(lib().tps_init_weights_synthetic(self.h))

    def set_weights(self, layer: int, w, b):
        import numpy as np
        w = np.ascontiguousarray(w, dtype=np.float32)
        b = np.ascontiguousarray(b, dtype=np.float32)
        check(lib().tps_set_weights(self.h, layer, w.ctypes.data, b.ctypes.data))

    def get_weights(self, layer: int):
        import numpy as np
        out_f, in_f = self.shapes[layer]
        w = np.zeros((out_f, in_f), np.float32)
        b = np.zeros(out_f, np.float32)
        mw = np.zeros_like(w)
        mb = np.zeros_like(b)
        check(lib().tps_get_weights(self.h, layer, w.ctypes.data, b.ctypes.data, mw.ctypes.data, mb.ctypes.data))
        return w, b, mw, mb

    def losses(self):
        import numpy as np
        n = C.c_int64()
        check(lib().tps_get_losses(self.h, None, 0, C.byref(n)))
        out = np.zeros(n.value, np.float32)
        if n.value:
            check(lib().tps_get_losses(self.h, out.ctypes.data, n.value, C.byref(n)))
        return out

    def read_losses_async(self, first: int, n: int, host_dst, stream: int):
        """Enqueue a device -> host copy of losses [first, first + n) into (pinned) host_dst."""
        check(lib().tps_read_losses_async(self.h, first, n, ptr(host_dst), stream))

    def trace(self) -> list[Event]:
        n = C.c_int64()
        check(lib().tps_get_trace(self.h, None, 0, C.byref(n)))
        buf = (Event * max(1, n.value))()
        check(lib().tps_get_trace(self.h, buf, n.value, C.byref(n)))
        return list(buf)[: n.value]

    def clear_trace(self):
        check(lib().tps_clear_trace(self.h))

    def stash_info(self):
        lv, st, pk = C.c_int32(), C.c_int64(), C.c_int64()
        check(lib().tps_stash_info(self.h, C.byref(lv), C.byref(st), C.byref(pk)))
        return lv.value, st.value, pk.value

    def intermediate_weight(self, layer: int, staleness: int, out):
        check(lib().tps_intermediate_weight(self.h, layer, staleness, ptr(out)))

    def get_version(self, layer: int, staleness: int, out):
        check(lib().tps_get_version(self.h, layer, staleness, ptr(out)))

    def memory_stats(self) -> dict:
        v = [C.c_int64() for _ in range(6)]
        check(lib().tps_memory_stats(self.h, *[C.byref(x) for x in v]))
        return dict(zip(["weights", "stash", "acts", "optim", "comm", "peak"], [x.value for x in v]))

    def memory_observed(self) -> int:
        n = C.c_int64()
        check(lib().tps_memory_observed(self.h, C.byref(n)))
        return n.value

    def set_profiling(self, on: bool):
        check(lib().tps_set_profiling(self.h, 1 if on else 0))

    def set_timeline(self, on: bool, origin_event: int = 0):
        """Per-event device brackets; origin_event = a recorded torch.cuda.Event's .cuda_event (0: own)."""
        check(lib().tps_set_timeline(self.h, 1 if on else 0, origin_event))

    def timeline(self) -> list[TimelineRec]:
        n = C.c_int64()
        check(lib().tps_get_timeline(self.h, None, 0, C.byref(n)))
        buf = (TimelineRec * max(1, n.value))()
        check(lib().tps_get_timeline(self.h, buf, n.value, C.byref(n)))
        return list(buf)[: n.value]

    def kernel_stats(self, which: int):
        n, ms, work = C.c_int64(), C.c_double(), C.c_double()
        check(lib().tps_kernel_stats(self.h, which, C.byref(n), C.byref(ms), C.byref(work)))
        return n.value, ms.value, work.value

    def launch_count(self) -> int:
        n = C.c_int64()
        check(lib().tps_launch_count(self.h, C.byref(n)))
        return n.value


def local_link(stages: list[Pipeline]):
    arr = (C.c_void_p * len(stages))(*[s.h.value for s in stages])
    check(lib().tps_local_link(arr, len(stages)))


class Graph:
    """A captured run of linked handles (tps_graph_capture); replay() runs the next n_mb mini-batches."""

    def __init__(self, stages: list[Pipeline], first_mb: int, n_mb: int, x_pool, y_pool, pool: int, stream: int):
        arr = (C.c_void_p * len(stages))(*[s.h.value for s in stages])
        g = C.c_void_p()
        check(lib().tps_graph_capture(arr, len(stages), first_mb, n_mb, ptr(x_pool), ptr(y_pool), pool, stream,
                                      C.byref(g)))
        self.g = g
        self.stages = stages           # keep the handles alive with the graph
        self.n_mb = n_mb
        self.next_mb = first_mb + n_mb

    def replay(self):
        check(lib().tps_graph_replay(self.g))
        self.next_mb += self.n_mb

    def close(self):
        if self.g:
            check(lib().tps_graph_destroy(self.g))
            self.g = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def run_schedule_local(stages: list[Pipeline], first_mb: int, n_mb: int, x_pool=None, y_pool=None, pool: int = 1):
    arr = (C.c_void_p * len(stages))(*[s.h.value for s in stages])
    check(lib().tps_run_schedule_local(arr, len(stages), first_mb, n_mb, ptr(x_pool), ptr(y_pool), pool))

/*
 * tps.h — C ABI of the B200-native TiMePReSt pipeline-parallel training step
 *          (V-TiMePReSt and I-TiMePReSt, arXiv 2509.23241).
 *
 * One handle = one pipeline stage = one consecutive set of layers on one GPU
 * ("the layers of a DNN are divided into sets of consecutive
 * layers without overlapping, and these sets are distributed over the
 * accelerators").  Each mini-batch is split into m micro-batches whose forwards
 * run first, followed by ONE collective backward for the whole mini-batch
 * and a weight update.  V-TiMePReSt runs every pass on the
 * stage's latest weights; I-TiMePReSt runs the backward on the
 * intermediate weight W_i(x,y) = (2 - 1/f(δ))·W_i(x|y), f(δ) = e^{-λδ}
 * (Eq. 1, Eq. 2), generalised here to
 * W_res = α·W_stash + β·W_latest (reading Z1).
 *
 * Conventions (every entry point):
 *   - returns tps_status; TPS_OK = 0.  On error, tps_last_error() returns a
 *     thread-local message; no C++ exception crosses this boundary.
 *   - "device" pointers are CUDA device addresses on the handle's device;
 *     "host" pointers are CPU memory (pinned memory is faster but optional).
 *   - all tensors are row-major.  Feature dimensions are stored padded to a
 *     multiple of 16 elements ("ld" = pad16(d)); padding columns are zero.
 *   - enqueue calls are asynchronous w.r.t. the host (stream-ordered on the
 *     handle's compute stream).  Caller-owned inputs must stay valid until the
 *     next tps_synchronize().  Device-side failures are latched and reported by
 *     tps_synchronize() (TPS_E_CUDA / TPS_E_NCCL).
 *   - one host thread drives a handle; handles are not re-entrant.
 *   - the handle owns every device allocation it makes (cudaMalloc, or the
 *     caller's dev_alloc hook) and frees them in tps_pipeline_destroy().
 *   - there is no CPU fallback: without an sm_100 device every compute call
 *     returns TPS_E_ARCH.
 */
#ifndef TPS_H
#define TPS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TPS_ABI_VERSION 4

typedef enum {
  TPS_OK = 0,
  TPS_E_INVALID_ARG = 1,  /* null pointer, negative size, out-of-range index       */
  TPS_E_CONFIG = 2,       /* S<1, m<1, b<1, λ<=0 for I, bad partition, bad dims      */
  TPS_E_ORDER = 3,        /* call is not the next event of the stage's static order */
  TPS_E_STALENESS = 4,    /* explicit δ has no live stashed version                 */
  TPS_E_CUDA = 5,         /* CUDA runtime/driver error (message has the CUDA text)  */
  TPS_E_NCCL = 6,         /* NCCL error                                             */
  TPS_E_OOM = 7,          /* device allocation failed                               */
  TPS_E_ARCH = 8,         /* no sm_100 device                                       */
  TPS_E_STATE = 9,        /* handle poisoned by an earlier device error             */
  TPS_E_UNSUPPORTED = 10  /* valid request this build does not implement            */
} tps_status;

typedef enum { TPS_V = 0, TPS_I = 1 } tps_variant;

/* Z1: EQ1 = the paper's closed form α = 2 - e^{λδ}, β = 0 (Eq. 1, Eq. 12);
 *     CONVEX = the prose reading α = e^{-λδ}, β = 1 - α.               */
typedef enum { TPS_BLEND_EQ1 = 0, TPS_BLEND_CONVEX = 1 } tps_blend;

/* Storage precision of activations, weight versions and activation-gradients (reading Z13 /
 * Z28; north_star "bf16/tf32 inputs with fp32 accumulation"): bf16 (RNE) or tf32 values in
 * 4-byte fp32 containers (RNA).  See tps_config.dtype.                                    */
typedef enum { TPS_BF16 = 0, TPS_TF32 = 1 } tps_dtype;

/* How a stage exchanges activations / activation-gradients with its neighbours
 * (one-to-one transfers).  NONE: S = 1.  LOCAL: all stages are handles
 * in one process on one GPU (device copies; used by tests and replicas).
 * NCCL: one process per stage, ncclSend/ncclRecv over NVLink.
 * IPC: one process per stage; each stage maps its neighbours' receive buffers and flag words
 * (cudaIpcOpenMemHandle: NVLink peer memory across GPUs, the same HBM for processes sharing a
 * GPU).  The producing kernel stores straight into the consumer's buffer: the last forward
 * GEMM's epilogue writes the next stage's input slot and the first layer's input-gradient
 * GEMM writes the previous stage's gradient buffer (chain networks; graph networks copy from
 * their stash), and stream memory operations (write / wait on 64-bit flag words) order
 * producer and consumer with no host round trip and no collective.  Runs of an IPC handle
 * number their mini-batches contiguously from 0.                                          */
typedef enum { TPS_TRANSPORT_NONE = 0, TPS_TRANSPORT_LOCAL = 1, TPS_TRANSPORT_NCCL = 2,
               TPS_TRANSPORT_IPC = 3 } tps_transport;

typedef enum { TPS_EV_F = 0, TPS_EV_B = 1, TPS_EV_U = 2 } tps_event_kind;

/* One schedule / trace record.  F: micro-batches [micro, micro+micro_count) of
 * mini-batch mb, forward on version v_used (= the stage's latest).
 * B: backward of mb; v_used = version whose weights are read (I: the stash the
 * forward used; V: the latest), v_latest = latest version, delta = v_latest -
 * v_forward for I (reading Z5) and 0 for V; alpha/beta =
 * the fp32 blend coefficients applied.  U: update producing version v_latest.   */
typedef struct {
  int32_t stage, kind, micro, micro_count;
  int64_t mb, v_used, v_latest;
  int32_t delta;
  float alpha, beta;
} tps_event;

/* Layer description for image networks.  Activations are NHWC bf16; a sample's
 * row is its H·W·C values.  Two families, not mixed in one network:
 *
 * Chain networks (BASELINE.json configs[2]: VGG-16 on 32x32 inputs), layer l reads
 * layer l-1:
 *   LINEAR:   out_c = dims out, in_c = dims in (a conv/pool output is flattened in
 *             (h, w, c) order); followed by ReLU unless it is the last layer.
 *   CONV3X3:  stride 1, zero padding 1, in_h x in_w x in_c -> in_h x in_w x out_c,
 *             weight [out_c, 3, 3, in_c] (= [out_c, 9·in_c] rows), + bias, ReLU.
 *             in_c % 64 == 0, out_c % 64 == 0, except the network's first layer, which
 *             may have any in_c (it runs as a GEMM on explicit patches).
 *   MAXPOOL2: 2x2 / stride 2, in_c channels (no parameters).
 *
 * Graph networks (configs[3]: ResNet-50 v1.5; math in oracle/resnet.py): layer l reads
 * the output of layer l - max(1, src_back) (layer -1 = the network input; a stage may
 * read only its own layers and the previous stage's last output), shapes are the
 * layer's INPUT:
 *   CONV:     k x k, stride, zero pad; no bias, no activation; weight [out_c, k, k, in_c].
 *             out_c % 16 == 0; 1x1/stride-1 convs need in_c % 16 == 0 (plain GEMM);
 *             3x3/stride-1/pad-1 convs with in_c, out_c % 64 == 0 gather their input
 *             with 4-D TMA; every other conv runs on explicit patches.
 *   BN:       batch norm over in_c channels with the statistics of each micro-batch
 *             (reading Z22), biased variance, eps 1e-5; γ (versioned fp32, blended in
 *             the I-TiMePReSt backward like a weight, reading Z12) and β (latest, like
 *             a bias); then + the output of layer l - res_back if res_back > 0; then
 *             ReLU if relu != 0.
 *   MAXPOOL3: 3x3 / stride 2 / pad 1 max pool (gradient to the first maximum, Z15).
 *   AVGPOOL:  global average pool in_h x in_w x in_c -> in_c.
 *   LINEAR:   the head (last layer only): in_c % 16 == 0, + bias, no ReLU.       */
typedef enum {
  TPS_LAYER_LINEAR = 0, TPS_LAYER_CONV3X3 = 1, TPS_LAYER_MAXPOOL2 = 2,
  TPS_LAYER_CONV = 3, TPS_LAYER_BN = 4, TPS_LAYER_MAXPOOL3 = 5, TPS_LAYER_AVGPOOL = 6
} tps_layer_kind;
typedef struct {
  int32_t kind;
  int32_t in_c, out_c;
  int32_t in_h, in_w;
  int32_t k, stride, pad;       /* CONV                                               */
  int32_t src_back;             /* graph kinds: main input = layer l - max(1, src_back) */
  int32_t res_back;             /* BN: residual = layer l - res_back; 0 = none        */
  int32_t relu;                 /* BN: ReLU after the affine (+ residual)             */
  int32_t reserved[5];
} tps_layer;

/* Pipeline configuration (read once by tps_pipeline_init; arrays are copied).
 * Network: num_layers Linear layers; layer l maps dims[l] -> dims[l+1]; every
 * layer but the last is followed by ReLU; the last produces dims[L] logits for a
 * softmax cross-entropy loss (mean over the B = m·b rows of a mini-batch, Z11).
 * stage_bounds has num_stages+1 entries; stage s owns layers
 * [stage_bounds[s], stage_bounds[s+1]) (consecutive, non-empty).        */
typedef struct {
  int32_t num_layers;
  const int32_t* dims;          /* host, num_layers+1 entries, each >= 1            */
  int32_t num_stages;           /* S >= 1                                            */
  const int32_t* stage_bounds;  /* host, S+1 entries                                 */
  int32_t stage_id;             /* 0 <= s < S                                        */
  int32_t micro_batches;        /* m >= 1                                    */
  int32_t micro_batch_size;     /* b >= 1                                            */
  int32_t fwd_group;            /* micro-batches per forward launch/transfer; divides m;
                                   0 => m (all micro-batch forwards "in parallel") */
  int32_t variant;              /* tps_variant                                       */
  int32_t blend;                /* tps_blend (I only)                                */
  double lambda;                /* λ > 0, I only                             */
  float lr, momentum, weight_decay;  /* SGD, PyTorch momentum convention (Z10)       */
  int32_t transport;            /* tps_transport                                     */
  const void* nccl_ids;         /* NCCL only: 2(S-1) ncclUniqueId (128 B each); id[2e] =
                                   forward comm of edge e (stage e -> e+1), id[2e+1] =
                                   backward comm of edge e (e+1 -> e)                 */
  int32_t device;               /* CUDA device ordinal                               */
  uint64_t seed;                /* synthetic-init seed (tps_init_weights_synthetic)  */
  uint64_t compute_stream;      /* cudaStream_t to enqueue on; 0 => handle-owned.  A run
                                   (tps_begin_run / tps_run_schedule*) reads its inputs after
                                   all work already submitted to this stream (0: to the legacy
                                   default stream) when the run begins                      */
  int32_t extra_recv_slot;      /* 1 => one extra input slot so the next forward's
                                   receive overlaps the backward (costs B·d_in·2 B)   */
  int32_t fuse_update;          /* 1 => the SGD/momentum update of each layer runs in the
                                   epilogue of its wgrad GEMM during tps_stage_backward (the
                                   dgrad of that layer is issued first, so it still reads the
                                   pre-update weights); tps_stage_update then only commits the
                                   new version.  Legal because U(j) always directly follows
                                   B(j) in the static order (reading Z7).  0 => separate kernel. */
  int32_t num_layer_specs;      /* 0 => MLP from dims; else == num_layers entries below  */
  const tps_layer* layer_specs; /* host; image networks (dims[0] = H·W·C of the input,
                                   dims[num_layers] = classes; other dims ignored)    */
  int32_t max_inflight;         /* mini-batches in flight K; 0 => K_s = S - s (reading Z6).
                                   Another value is accepted for S = 1 only: a one-stage
                                   pipeline with K in flight sees the steady staleness
                                   δ = K - 1 of a stage at depth K (the staleness sweep of
                                   BASELINE.json configs[1] on one GPU); TPS_E_CONFIG else */
  int32_t staleness_mode;       /* 0 => an explicit staleness passed to tps_stage_backward
                                   must equal the logged δ (scheduled run).  1 => standalone
                                   microbenchmark: any δ >= 0 whose version is still in the
                                   ring (v_latest - δ >= max(0, v_latest - R + 1)) is used
                                   as given (SURVEY §8(b) "staleness override")          */
  /* Optional device allocator (e.g. PyTorch's caching allocator, so the framework's
   * memory accounting sees the handle's buffers).  NULL => cudaMalloc / cudaFree.
   * dev_alloc returns a device pointer (256-byte aligned) or NULL on failure
   * (=> TPS_E_OOM); dev_free is called for every such pointer by
   * tps_pipeline_destroy after a device synchronize.                               */
  void* (*dev_alloc)(size_t bytes, void* ctx);
  void (*dev_free)(void* ptr, void* ctx);
  void* alloc_ctx;
  /* Pipeline x data parallelism ("pipelining and data parallelism together";
   * SURVEY §8(f) NEXT-2): dp_size replicas of the whole pipeline, each on its own mini-batches;
   * stage s of every replica averages the R weight/bias gradients (replica order, fp32) inside
   * one fused reduce + SGD kernel that reads the peers' gradient buffers directly (NVLink peer
   * memory / same-process pointers), so the replicas stay bitwise identical.  dp_size = 1: off.
   * With dp_size > 1 the update runs as a separate kernel (fuse_update is ignored), chain
   * networks only (TPS_E_UNSUPPORTED for graph networks), mini-batches numbered contiguously.
   * Replica r of mini-batch j reads rows [r·B, (r+1)·B) of pool entry j % pool.               */
  int32_t dp_size;              /* R >= 1 (<= 8)                                        */
  int32_t dp_rank;              /* 0 <= dp_rank < R                                     */
  /* Storage precision (tps_dtype; reading Z28, north_star "bf16/tf32 inputs"): TPS_BF16 (0)
   * stores activations, weight versions / stash and activation-gradients as bf16 (RNE);
   * TPS_TF32 (1) stores them as tf32 values in fp32 containers (RNA, cvt.rna.tf32.f32) and
   * runs the stage GEMMs as kind::tf32: every activation / version buffer, input pool and
   * exchanged message then holds 4-byte elements.  fp32 master weights, momentum, weight
   * gradients and losses are the same in both.  TF32: chain MLP networks only (no
   * layer_specs, dp_size 1), else TPS_E_UNSUPPORTED; another value: TPS_E_CONFIG.            */
  int32_t dtype;
  int32_t reserved;
} tps_config;

typedef struct tps_pipeline tps_pipeline;  /* opaque; one per stage */

/* ---- lifecycle ------------------------------------------------------------ */
int32_t tps_abi_version(void);
const char* tps_last_error(void);
/* 128-byte ncclUniqueId into out128 (host).  TPS_E_NCCL on failure. */
tps_status tps_nccl_unique_id(void* out128);
/* Validates cfg (TPS_E_CONFIG), checks the device is sm_100 (TPS_E_ARCH),
 * allocates weights (fp32 master + momentum), the bf16 version ring (K_s = S - s
 * slots for I, 1 for V), activation stash and exchange buffers,
 * and (NCCL) joins the edge communicators.  Weights start at zero: call
 * tps_init_weights_synthetic or tps_set_weights before training.            */
tps_status tps_pipeline_init(const tps_config* cfg, tps_pipeline** out);
tps_status tps_pipeline_destroy(tps_pipeline* p);
/* LOCAL transport: connect the S handles of one process (stage order). */
tps_status tps_local_link(tps_pipeline* const* stages, int32_t num_stages);
/* IPC transport, after tps_pipeline_init on every stage:
 *   tps_ipc_export writes this stage's exchange descriptor (IPC handles of its input slots,
 *   gradient receive buffers and flag words; at most TPS_IPC_BLOB_BYTES) into host `out`;
 *   the caller hands every stage its neighbours' descriptors (e.g. an all-gather over the
 *   process group); tps_ipc_connect maps them (prev = stage s-1's descriptor, NULL on stage 0;
 *   next = stage s+1's, NULL on the last stage).  TPS_E_CONFIG for a descriptor of the wrong
 *   stage or shape, TPS_E_CUDA if a handle cannot be opened.                                  */
#define TPS_IPC_BLOB_BYTES 2048
tps_status tps_ipc_export(tps_pipeline* p, void* out, int64_t cap, int64_t* n);
tps_status tps_ipc_connect(tps_pipeline* p, const void* prev_blob, const void* next_blob);
/* Data parallelism (dp_size > 1): connect the R replicas of ONE stage, one process per
 * replica (each process its own CUDA context: replicas synchronise through flag words that
 * another process writes, which must never sit behind a blocked wait in a shared hardware
 * queue, so replicas are never handles of one process).  tps_dp_export writes this replica's
 * descriptor (IPC handles of its per-layer gradient buffers and flag words; out = NULL returns
 * the size in *n); tps_dp_connect takes all R descriptors in replica order (its own included).
 * TPS_E_CONFIG for mismatched shapes / stages / ranks.                                      */
tps_status tps_dp_export(tps_pipeline* p, void* out, int64_t cap, int64_t* n);
tps_status tps_dp_connect(tps_pipeline* p, const void* const* blobs, int32_t dp_size);

/* ---- the training step (one mini-batch = B(j) U(j) + m forwards) ----------- */
/* Declare a run of mini-batches [first_mb, first_mb+n_mb): builds the stage's
 * static order (fill, steady state, drain; reading Z7) against which the
 * following stage_forward/backward/update calls are checked.  A run must end
 * (all its events issued) before the next begins; versions carry over.        */
tps_status tps_begin_run(tps_pipeline* p, int64_t first_mb, int64_t n_mb);
/* Forward of micro-batches [micro, micro+count) of mini-batch mb on the latest
 * weights.  x: stage 0 only — [count·b, dims[0]] bf16, dense rows
 * (ld = dims[0]); device or host pointer.  labels: last stage only —
 * [count·b] int32, device or host.  Must be the stage's next static event
 * (TPS_E_ORDER otherwise).                                                     */
tps_status tps_stage_forward(tps_pipeline* p, int64_t mb, int32_t micro, int32_t count,
                             const void* x, const int32_t* labels);
/* Collective backward of mini-batch mb on the resolved weight:
 * V: latest; I: α·W_stash(v_fwd) + β·W_latest with δ = v_latest - v_fwd.
 * staleness = -1 => δ from the version log; >= 0 => must equal the logged δ in
 * a scheduled run (staleness_mode 0), or (staleness_mode 1, microbenchmark) any δ
 * whose version is still live in the ring.  TPS_E_STALENESS when δ != the logged
 * value (mode 0), when V is given δ > 0 (V has no stash), or when version
 * v_latest - δ is no longer (or not yet) held; nothing is enqueued then and the
 * call may be retried.  TPS_E_ORDER if B(mb) is not the stage's next event.     */
tps_status tps_stage_backward(tps_pipeline* p, int64_t mb, int32_t staleness);
/* SGD/momentum update of every layer of the stage from the gradients of mb;
 * writes the new bf16 version into a free ring slot (I) or in place (V); the
 * stash of a version is released once its last consumer's backward ran. */
tps_status tps_stage_update(tps_pipeline* p, int64_t mb);
/* Walk the stage's static order for mini-batches [first_mb, first_mb+n_mb)
 * (fill, steady state, drain).  x_pool: stage 0, [pool, B, dims[0]] bf16;
 * y_pool: last stage, [pool, B] int32; mini-batch j uses slot j % pool.
 * Pools may be device or host memory (host: copied per mini-batch inside).   */
tps_status tps_run_schedule(tps_pipeline* p, int64_t first_mb, int64_t n_mb,
                            const void* x_pool, const int32_t* y_pool, int32_t pool);
/* LOCAL transport: drive all linked handles of this process through the same range,
 * interleaving them in a dependency-respecting host order.  num_stages = S handles of one
 * pipeline in stage order, or R·S handles of R data-parallel replicas (replica-major).      */
tps_status tps_run_schedule_local(tps_pipeline* const* stages, int32_t num_stages,
                                  int64_t first_mb, int64_t n_mb,
                                  const void* x_pool, const int32_t* y_pool, int32_t pool);
tps_status tps_synchronize(tps_pipeline* p);

/* ---- CUDA-graph replay of whole runs (capture the periodic steady
 * state; P:136's nF1B order is static, so a run's work is identical from run to run) --------
 * tps_graph_capture walks the run [first_mb, first_mb + n_mb) of the linked handles exactly like
 * tps_run_schedule_local (same events, trace, host state), records the device work into one
 * CUDA graph instead of issuing it, and launches the graph once on `stream` (a real stream, not
 * 0).  tps_graph_replay launches it again for the NEXT n_mb mini-batches and advances the host
 * state as a walk would; valid because n_mb must be a multiple of the schedule period (lcm of 2,
 * pool and every handle's input slots, stash slots and version-ring size): every buffer slot,
 * ring slot and pool slot then repeats from run to run, and the loss slot is a device counter.
 * Requirements: LOCAL or single-stage handles (TPS_E_UNSUPPORTED otherwise), no per-launch
 * profiling, the caller leaves the handles and the pools (same contents per slot) alone between
 * replays (TPS_E_STATE if a handle's version moved).  Errors from the walk are returned as is. */
typedef struct tps_graph tps_graph;
tps_status tps_graph_capture(tps_pipeline* const* stages, int32_t num_handles, int64_t first_mb, int64_t n_mb,
                             const void* x_pool, const int32_t* y_pool, int32_t pool, uint64_t stream,
                             tps_graph** out);
tps_status tps_graph_replay(tps_graph* g);
tps_status tps_graph_destroy(tps_graph* g);
/* Stream-ordered join: `stream` (a cudaStream_t, 0 = legacy default) waits for everything the
 * handle has enqueued so far on all of its streams (compute, weight-gradient, optimizer,
 * transfers).  Non-blocking; lets a caller time or consume a run on its own stream.        */
tps_status tps_join(tps_pipeline* p, uint64_t stream);

/* ---- stash / intermediate-weight management -------------------------------- */
tps_status tps_blend_coeffs(int32_t variant, int32_t blend, int32_t staleness, double lambda,
                            float* alpha, float* beta);
/* live_versions: bf16 weight versions currently held; stash_bytes: bytes of live
 * versions other than the latest; peak_stash_bytes: max over the run.          */
tps_status tps_stash_info(tps_pipeline* p, int32_t* live_versions, int64_t* stash_bytes,
                          int64_t* peak_stash_bytes);
/* Debug materialiser (K8): out_bf16 (device, [out, ld_in]) =
 * bf16_rne(fp32(α·W_stash) + fp32(β·W_latest)) for stage-local layer index
 * `layer`, with W_stash = latest - staleness.  Never used by the training path.
 * (dtype TPS_TF32: out is fp32 [out, ld_in] = tf32_rna of the same fp32 sum.)    */
tps_status tps_intermediate_weight(tps_pipeline* p, int32_t layer, int32_t staleness,
                                   void* out_bf16);

/* Debug read of a live bf16 weight version (device out, [pad16(out), pad16(in)]):
 * version latest - staleness of stage-local layer `layer`.  (TPS_TF32: fp32 elements.) */
tps_status tps_get_version(tps_pipeline* p, int32_t layer, int32_t staleness, void* out_bf16);

/* ---- static schedule (host only) ------------------------------------------- */
/* Stage s's static order for M mini-batches (reading Z6/Z7): F of mini-batches
 * 0..K-1 (K = min(S-s, M)), then per j: B(j), U(j), F(j+K).  One F record per
 * forward group.  Writes up to cap records; *n = total.                       */
tps_status tps_schedule_events(int32_t S, int32_t s, int32_t m, int32_t fwd_group, int64_t M,
                               tps_event* out, int64_t cap, int64_t* n);

/* ---- state access ------------------------------------------------------------ */
/* Stage-local layer `layer`: host fp32 buffers of logical size [out, in] / [out]
 * (any may be NULL).  Synchronizes the handle.                                */
tps_status tps_get_weights(tps_pipeline* p, int32_t layer, float* w, float* b,
                           float* mom_w, float* mom_b);
/* Sets the fp32 master (and the latest bf16 version) of a layer; zeroes momentum. */
tps_status tps_set_weights(tps_pipeline* p, int32_t layer, const float* w, const float* b);
/* Device-side synthetic init, bit-identical to synthgen.weights(seed, global layer). */
tps_status tps_init_weights_synthetic(tps_pipeline* p);
/* Per-mini-batch mean losses of the last stage, in mini-batch order since init. */
tps_status tps_get_losses(tps_pipeline* p, float* out, int64_t cap, int64_t* n);
/* Stream-ordered read of losses [first, first + n) into host memory (pinned for asynchrony):
 * enqueued on `stream` after the loss kernels; the caller synchronises before reading dst.  */
tps_status tps_read_losses_async(tps_pipeline* p, int64_t first, int64_t n, float* host_dst, uint64_t stream);
tps_status tps_get_trace(tps_pipeline* p, tps_event* out, int64_t cap, int64_t* n);
tps_status tps_clear_trace(tps_pipeline* p);
/* Bytes held by category; peak = max over the handle's life of their sum (the library's
 * own allocation arithmetic; every buffer is allocated by tps_pipeline_init).       */
tps_status tps_memory_stats(tps_pipeline* p, int64_t* weights, int64_t* stash, int64_t* acts,
                            int64_t* optim, int64_t* comm, int64_t* peak);
/* Device-observed bytes: the drop of cudaMemGetInfo's free memory across the allocations
 * of tps_pipeline_init (allocation granularity included; 0 when a dev_alloc hook served
 * them from a cache).  Meaningful when nothing else allocates concurrently.          */
tps_status tps_memory_observed(tps_pipeline* p, int64_t* device_bytes);
/* Kernel timing: when enabled, CUDA events bracket every GEMM launch on the
 * compute stream; tps_kernel_stats returns launch count, summed device ms and
 * summed algorithmic FLOPs of GEMM kind `which` (0 fwd, 1 dgrad, 2 wgrad,
 * 3 all GEMMs, 4 update kernel [bytes instead of FLOPs]).  Synchronizes.       */
tps_status tps_set_profiling(tps_pipeline* p, int32_t enable);
tps_status tps_kernel_stats(tps_pipeline* p, int32_t which, int64_t* launches, double* ms,
                            double* work);
/* Per-event device timeline (Chrome trace export, tools/chrome_trace.py): when enabled, every
 * schedule event this handle executes (walker or step-wise) is bracketed by two CUDA events on
 * its compute stream; tps_get_timeline returns, per event, its trace record and the device times
 * of the brackets in ms since `origin_event` (a caller-owned cudaEvent_t recorded BEFORE the
 * events, on any stream of this device, so several handles share one time axis; 0: the handle
 * records its own origin on its compute stream now).  F spans the forward's launches, B the
 * backward's (with the fused update, if on), U is a zero-width commit marker.  Enabling or
 * disabling synchronises and clears the records; graph capture is refused while enabled.
 * tps_get_timeline synchronises on the last bracket.  With TPS_NVTX=1 in the environment at
 * tps_pipeline_init, every event is also an NVTX range "s<stage> <F|B|U> mb<j>" (host side). */
typedef struct {
  tps_event ev;
  double t0_ms, t1_ms;
} tps_timeline_rec;
tps_status tps_set_timeline(tps_pipeline* p, int32_t enable, uint64_t origin_event);
tps_status tps_get_timeline(tps_pipeline* p, tps_timeline_rec* out, int64_t cap, int64_t* n);
/* Number of kernels this handle has launched since init (product kernels only). */
tps_status tps_launch_count(tps_pipeline* p, int64_t* n);

/* ---- synthetic inputs (device counter-based generator = synthgen) ------------ */
/* kind 0: x = ((h & 0xFF) - 128)/128; kind 1: x = (h & 0xFF)/256 (bf16 out, rows×cols
 * dense); kind 2: labels (h >> 8) % classes (int32 out, `rows` entries).  tid as in
 * synthgen (TID_X + mb, TID_Y + mb).  dst is a device pointer.                  */
tps_status tps_fill_synthetic(int32_t kind, uint64_t seed, uint64_t tid, int64_t rows,
                              int64_t cols, int32_t classes, void* dst, uint64_t stream);

/* ---- debugging: progress of a handle's static order (safe to call from another host thread
 * while a run is in progress).  pos = index of the next event, n_events = events in the run,
 * busy = bitmask of streams with pending work (compute, fwd-in, fwd-out, bwd-in, bwd-out,
 * optimizer).                                                                              */
tps_status tps_debug_progress(tps_pipeline* p, int64_t* pos, int64_t* n_events, int32_t* busy);

/* ---- raw stage GEMM (kernel unit tests / microbenchmarks) -------------------- */
/* D[M,N] = alpha · A·Bᵀ (fp32 accumulate on tcgen05), A and B bf16, device.
 * mode 0 (forward):  A [M,K] ld=lda (K-major), B [N,K] ld=ldb (K-major);
 *        epilogue: + bias[N] (fp32, may be NULL), ReLU if relu, out bf16 or fp32.
 * mode 1 (dgrad):    A [M,K] (K-major), B stored [K,N] ld=ldb (MN-major);
 *        epilogue: ·alpha, then zero where mask[M,N] (bf16, ld=ldm) is <= 0 (mask may be NULL).
 * mode 2 (wgrad):    A stored [K,M] ld=lda (MN-major), B stored [K,N] (MN-major); fp32 out.
 * mode 3 (dgrad, blended operand, CONVEX/I): B = alpha·B + beta·B2 formed in shared memory
 *        before the MMA (B2 same layout/ld as B); mask as mode 1; no extra alpha scale.
 * out_f32: 1 => fp32 output, else bf16.  Requires N % 8 == 0 and 16-byte aligned rows.
 * mode | TPS_GEMM_TF32: tf32 storage (reading Z28): A, B, B2, mask and a non-fp32 out are fp32
 *        arrays holding tf32 values (ld in elements), the MMAs run kind::tf32 and a non-fp32
 *        out is rounded RNA to tf32.                                                       */
#define TPS_GEMM_TF32 16
tps_status tps_gemm(int32_t mode, int32_t M, int32_t N, int32_t K,
                    const void* A, int32_t lda, const void* B, int32_t ldb, const void* B2,
                    void* out, int32_t ldo, int32_t out_f32, const float* bias, int32_t relu,
                    float alpha, float beta, const void* mask, int32_t ldm, uint64_t stream);

/* Weight gradient with the fused SGD/momentum update epilogue (the kernel the pipeline runs
 * with fuse_update = 1; row a10): for g = Aᵀ·B (A stored [K,M] ld=lda, B stored [K,N] ld=ldb,
 * bf16, fp32 accumulation), per element of the fp32 master w [M,N] (ld=ldw) and momentum v:
 *   g' = g + wd·w ; v = mu·v + g' ; w = w - lr·v  (fp32, one rounding per op; mu = 0: v unused)
 * and ver [M,N] (bf16, ld=ldw) = bf16_rne(w).  The gradient is never written to memory.      */
tps_status tps_gemm_wgrad_sgd(int32_t M, int32_t N, int32_t K, const void* A, int32_t lda, const void* B,
                              int32_t ldb, float* w, float* v, void* ver, int32_t ldw, float lr, float mu,
                              float wd, uint64_t stream);

/* The dual backward launch the pipeline runs with fuse_update = 1 (rows a8 + a10): ONE
 * persistent kernel computing tps_gemm_wgrad_sgd(M, N, K, A, lda, B, ldb, w, v, ver, ldw, lr,
 * mu, wd) (layer k's weight gradient + update) AND the input gradient of layer k-1,
 *   outd [Md, Nd] (bf16, ld=ldod) = bf16_rne(alpha · (Ad · Bd)) zeroed where mask <= 0,
 * Ad [Md, Kd] K-major (ld=ldad), Bd stored [Kd, Nd] (ld=ldbd), mask bf16 [Md, Nd] (ld=ldm, may
 * be NULL) — i.e. tps_gemm mode 1.  Each cluster pair interleaves tiles of both, so the input
 * gradient's MMAs run while the update epilogue streams w / v.  Both outputs are bit-identical
 * to the two separate calls.  The two problems must not overlap in memory.  TPS_E_UNSUPPORTED
 * when either has fewer than 256 rows or N <= 128, or the balanced tile split does not exist. */
tps_status tps_gemm_bwd_dual(int32_t M, int32_t N, int32_t K, const void* A, int32_t lda, const void* B,
                             int32_t ldb, float* w, float* v, void* ver, int32_t ldw, float lr, float mu,
                             float wd, int32_t Md, int32_t Nd, int32_t Kd, const void* Ad, int32_t ldad,
                             const void* Bd, int32_t ldbd, void* outd, int32_t ldod, float alpha,
                             const void* mask, int32_t ldm, uint64_t stream);

/* ---- stage partitioner ("distribute the DNNs ... in such a way
 * that a balance is maintained between the memory consumptions in each node") ----------
 * Splits L layers into S consecutive non-empty stages minimising the largest per-stage
 * cost (exact dynamic programme).  Per layer (host arrays): param_bytes = bytes of one copy
 * of its parameters' fp32 master, act_bytes = bytes of its stashed input for one mini-batch,
 * flops = its training FLOPs per mini-batch.  objective 0 = memory, 1 = time (flops).
 * Memory of stage s (0-based) holding layers P:
 *   Σ_P param_bytes·(1 + momentum + 0.5·R_s) + K_s·Σ_P act_bytes,  K_s = S - s,
 *   R_s = K_s for I-TiMePReSt (the bf16 version ring) and 1 for V,
 *   momentum = 1 if mu != 0 (fp32 momentum) else 0.
 * bounds_out: S+1 entries; stage_cost_out: S entries (may be NULL).                       */
tps_status tps_partition(int32_t num_layers, const double* param_bytes, const double* act_bytes,
                         const double* flops, int32_t num_stages, int32_t variant, int32_t momentum,
                         int32_t objective, int32_t* bounds_out, double* stage_cost_out);

/* ---- raw 3x3 convolution GEMMs (implicit im2col via 4-D TMA; unit tests) ----
 * NHWC bf16 device tensors, stride 1, padding 1, Ci % 64 == 0, Co % 64 == 0.
 * mode 0 (forward): out[N·H·W, Co] = conv(X[N,H,W,Ci]; W[Co,3,3,Ci]) + bias, ReLU if relu.
 * mode 1 (dgrad):   out[N·H·W, Ci] = alpha · conv_transpose(dY[N,H,W,Co]; W), zero where
 *                   mask[N·H·W, Ci] <= 0 (mask may be NULL).
 * mode 2 (wgrad):   out[Co, 9·Ci] (fp32) = dY[N·H·W, Co]ᵀ · im2col(X[N,H,W,Ci]).
 * mode 3 (dgrad, blended operand): as mode 1 with W = alpha·W + beta·W2 formed on load.   */
tps_status tps_conv_gemm(int32_t mode, int32_t N, int32_t H, int32_t W, int32_t Ci, int32_t Co,
                         const void* A, const void* Wt, const void* W2, void* out, int32_t out_f32,
                         const float* bias, int32_t relu, float alpha, float beta, const void* mask,
                         uint64_t stream);

/* ---- general convolution GEMMs (TMA im2col-mode loads; unit tests) ------------
 * NHWC bf16 device tensors; k x k filter, stride, zero padding pad; Ho = (H+2pad-k)/stride+1.
 * Ci % 64 == 0, Co % 64 == 0.  No bias / activation.
 * mode 0 (forward): out[N·Ho·Wo, Co] = conv(X[N,H,W,Ci]; W[Co,k,k,Ci]) (bf16, or fp32 if out_f32).
 * mode 1 (dgrad, k = 3, stride 1, pad 1): out[N·H·W, Ci] = alpha · conv_transpose(dY; W) (bf16).
 * mode 2 (wgrad):   out[Co, k·k·Ci] (fp32) = dY[N·Ho·Wo, Co]ᵀ · im2col(X).
 * mode 3 (dgrad, blended operand): as mode 1 with W = alpha·W + beta·W2 formed on load.       */
tps_status tps_conv2d_gemm(int32_t mode, int32_t N, int32_t H, int32_t W, int32_t Ci, int32_t Co, int32_t k,
                           int32_t stride, int32_t pad, const void* A, const void* Wt, const void* W2, void* out,
                           int32_t out_f32, float alpha, float beta, uint64_t stream);

/* ---- ResNet op kernels (unit tests; the pipeline calls the same kernels) --------
 * All tensors NHWC bf16 on the device unless stated; `stream` = cudaStream_t (0 = legacy).
 * Definitions: oracle/resnet.py (textbook conv / batch norm / pooling, reading Z22).
 *
 * tps_im2col: P[(n,ho,wo), (kh,kw,c)] = X[n, s·ho+kh-p, s·wo+kw-p, c] (0 outside), columns
 *   k·k·C .. ldp-1 zero; Ho = (H+2p-k)/s+1.  Bit-exact gather.
 * tps_col2im: dX[n,h,w,c] = bf16(Σ_{kh,kw} dP[...] (+ add[n,h,w,c])), dP fp32 [N·Ho·Wo, ldp],
 *   add bf16 may be NULL or alias dX; fp32 sum in (kh, kw) order.
 * tps_bn_forward: per segment of seg_rows rows (one micro-batch) and channel:
 *   mean, invstd = 1/sqrt(biased var + 1e-5) (fp64 sums, fp32 out, [segs, C]);
 *   y = bf16(act(γ·(x-mean)·invstd + β (+ res))), act = ReLU if relu; res may be NULL.
 * tps_bn_backward: dy' = dy ⊙ [y > 0] if relu; per segment/channel Σdy', Σdy'·x̂ (fp64);
 *   dγ = Σ_seg Σdy'·x̂, dβ = Σ_seg Σdy' (fp32 [C]);
 *   dx = bf16(γ_r·invstd·(dy' - Σdy'/m - x̂·Σdy'x̂/m)), γ_r = a·γ_stash + b·γ_latest (fp32);
 *   dres = bf16(dy') when non-NULL.
 * tps_pool_op: op 0 maxpool3 forward  out = max over the 3x3/2/1 window of a (= X);
 *              op 1 maxpool3 backward out = dX from a = X and b = dY (first maximum, Z15);
 *              op 2 avgpool forward   out[N, C] = mean over H·W of a;
 *              op 3 avgpool backward  out[N,H,W,C] = b[N, C] / (H·W);
 *              op 4 maxpool3 forward recording taps: out = Y, b = uint8 tap (0..8, row-major
 *                   in the window) of the first maximum per output (written), C % 8 == 0;
 *              op 5 maxpool3 backward from recorded taps: a = taps, b = dY, out = dX.
 * Errors: TPS_E_INVALID_ARG for null/ill-sized arguments, TPS_E_ARCH off sm_100,
 *         TPS_E_CUDA on launch failure.                                                  */
tps_status tps_im2col(const void* X, void* P, int32_t N, int32_t H, int32_t W, int32_t C, int32_t k,
                      int32_t stride, int32_t pad, int32_t ldp, uint64_t stream);
tps_status tps_col2im(const float* dP, void* dX, const void* add, int32_t N, int32_t H, int32_t W, int32_t C,
                      int32_t k, int32_t stride, int32_t pad, int32_t ldp, uint64_t stream);
tps_status tps_bn_forward(const void* x, const void* res, void* y, const float* gamma, const float* beta,
                          float* mean, float* invstd, int32_t segs, int32_t seg_rows, int32_t C, int32_t relu,
                          uint64_t stream);
tps_status tps_bn_backward(const void* dy, const void* y, const void* x, const float* mean, const float* invstd,
                           const float* gamma_stash, const float* gamma_latest, float a, float b, int32_t segs,
                           int32_t seg_rows, int32_t C, int32_t relu, void* dx, void* dres, float* dgamma,
                           float* dbeta, uint64_t stream);
tps_status tps_pool_op(int32_t op, const void* a, const void* b, void* out, int32_t N, int32_t H, int32_t W,
                       int32_t C, uint64_t stream);

#ifdef __cplusplus
}
#endif
#endif /* TPS_H */

// runtime.cpp — host runtime behind include/tps.h: one handle per pipeline stage.
//
// What it does per mini-batch j at stage s:
//   F(j, group)  forward of a group of micro-batches on the stage's LATEST bf16 weights
//                (V: P:182/P:188; I: P:213, reading Z8), activations kept for the backward
//   B(j)         one collective backward over the B = m·b rows: wgrad + bias grad and
//                dgrad on the resolved weight (V: latest; I: α·W_stash + β·W_latest,
//                Eq. 1 P:220 / reading Z1) with δ = latest - version the forward used
//   U(j)         fused SGD/momentum update; the new bf16 version goes into ring slot
//                (version mod R): R = S - s for I (stash kept until its last consumer,
//                P:408), R = 1 for V (old version overwritten at once)
// in the static per-stage order of reading Z7 (K_s = S - s mini-batches in flight).
// The host only enqueues: kernels on the compute stream, transfers on four comm
// streams ordered by CUDA events; nothing blocks until tps_synchronize.
#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "../../include/tps.h"
#include "gemm.h"
#include "kernels.h"

namespace {

thread_local std::string g_err;

tps_status fail(tps_status st, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

#define CUDA_OK(expr)                                                                                   \
  do {                                                                                                  \
    cudaError_t _e = (expr);                                                                            \
    if (_e != cudaSuccess) return fail(TPS_E_CUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(_e), __FILE__, __LINE__); \
  } while (0)

#define NCCL_OK(expr)                                                                                   \
  do {                                                                                                  \
    ncclResult_t _r = (expr);                                                                           \
    if (_r != ncclSuccess) return fail(TPS_E_NCCL, "%s: %s", #expr, ncclGetErrorString(_r));           \
  } while (0)

#define TPS_TRY(expr)                  \
  do {                                 \
    tps_status _s = (expr);            \
    if (_s != TPS_OK) return _s;       \
  } while (0)

inline int pad16(int d) { return (d + 15) / 16 * 16; }

// TPS_RELU_MASK=0: BN backward reads y for the ReLU mask (A/B of the bit-mask path)
bool no_relu_mask() {
  const char* e = std::getenv("TPS_RELU_MASK");
  return e && e[0] == '0';
}

bool is_host_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeUnregistered;
}

tps_status check_arch(int device) {
  static thread_local int ok_device = -1;   // cache a positive answer (cudaGetDeviceProperties is slow)
  if (device == ok_device) return TPS_OK;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n <= device) {
    cudaGetLastError();
    return fail(TPS_E_ARCH, "no CUDA device %d (this build has no CPU fallback)", device);
  }
  cudaDeviceProp pr;
  CUDA_OK(cudaGetDeviceProperties(&pr, device));
  if (pr.major != 10) return fail(TPS_E_ARCH, "device %d is sm_%d%d; this library targets sm_100a", device, pr.major, pr.minor);
  ok_device = device;
  return TPS_OK;
}

struct Layer {
  int gidx = 0;
  int kind = TPS_LAYER_LINEAR;
  bool im2col = false;      // conv run as a GEMM on explicit patches (network layer 0, few channels)
  // parameters (none for pools): logical [out, in], stored [Np, Kp]
  int in = 0, out = 0, Kp = 0, Np = 0;
  // activation geometry: a sample's input is hw_in pixels x ld_in channels (linear: 1 x Kp)
  int H = 1, Wd = 1, Ci = 0, Co = 0;
  int hw_in = 1, ld_in = 0, hw_out = 1, ld_out = 0;
  float *W = nullptr, *b = nullptr, *mW = nullptr, *mb = nullptr, *dW = nullptr, *db = nullptr;
  std::vector<uint16_t*> ver;  // R bf16 [Np, Kp] slots
  // graph networks (ResNet): input = output of local layer `src` (-1 = stage input),
  // BN residual = output of local layer `res` (-2 = none; -1 = stage input)
  int k = 1, st = 1, pad = 0, src = -1, res = -2;
  bool relu = false;
  int Ho = 1, Wo = 1;
  int conv_mode = 0;                  // CONV: 0 plain GEMM (1x1/s1), 1 implicit 3x3, 2 explicit patches
  std::vector<float*> verf;           // BN: R fp32 γ versions [C]
  std::vector<float*> mean, invstd;   // BN: per stash slot, [m, C] per-micro-batch statistics
  std::vector<uint8_t*> argmax;       // MAXPOOL3 (C % 8 == 0): per stash slot, first-max tap per output
  // BN with ReLU (C % 8 == 0): per stash slot, [rows, C/8] bytes, bit e = [y > 0]; the backward
  // reads it instead of y (0.125 instead of 2 B per element, in both backward passes)
  std::vector<uint8_t*> relu_mask;
  // this backward's bias gradient source: 32-row column sums of G written by the input-gradient
  // GEMM of the layer above (GemmArgs.colsum), or null (full pass over G)
  const float* bias_part = nullptr;
  int bias_groups = 0;
  // graph networks: this conv's epilogue also writes the column sums (Σx, Σx²) that the batch norm
  // right after it needs, so the BN skips its statistics pass over the conv output
  bool stats_to_next = false;
  // fuse_update run: this layer's SGD step rides in its weight-gradient epilogue.  False for the
  // layers whose weight-gradient output tiles cannot fill the GPU (small M x N, long K: the
  // convolutions of VGG's early blocks, the patch layer): those take the split-K weight gradient
  // and the separate update kernel on the same stream (one fused CTA per 64-column tile ran
  // ~0.7 ms at 32 x 32 x 64 channels, B = 128)
  bool fuse = false;
  bool has_w() const {
    return kind == TPS_LAYER_LINEAR || kind == TPS_LAYER_CONV3X3 || kind == TPS_LAYER_CONV || kind == TPS_LAYER_BN;
  }
  bool has_b() const { return kind == TPS_LAYER_LINEAR || kind == TPS_LAYER_CONV3X3 || kind == TPS_LAYER_BN; }
  int64_t in_elems() const { return static_cast<int64_t>(hw_in) * ld_in; }    // per sample (stash)
  int64_t out_elems() const { return static_cast<int64_t>(hw_out) * ld_out; }
};

struct Msg {  // LOCAL transport mailbox entry
  const void* src;
  size_t bytes;
  cudaEvent_t ready;
  cudaEvent_t consumed;  // owned by the sender; recorded by the receiver after its copy
};

struct TimedLaunch {
  int kind;
  double work;
  cudaEvent_t a, b;
};

}  // namespace

struct tps_pipeline {
  // ---- configuration
  int S = 1, s = 0, m = 1, bsz = 1, B = 1, g = 1, ng = 1, Kmax = 1, R = 1, A0 = 1;
  int variant = TPS_V, blend = TPS_BLEND_EQ1, transport = TPS_TRANSPORT_NONE, device = 0;
  double lambda = 0.05;
  float lr = 0.01f, mu = 0.f, wd = 0.f;
  uint64_t seed = 0;
  bool first = true, last = true, eq1_on_load = false, fuse_update = false;
  bool graph = false;                        // ResNet-style layer graph (CONV/BN/MAXPOOL3/AVGPOOL)
  // storage precision (reading Z28): bf16 (ew = 1 uint16 unit per element, 2 bytes) or tf32 values
  // in fp32 containers (ew = 2, 4 bytes).  Buffers stay typed uint16_t*; offsets scale by ew.
  bool tf = false;
  int ew = 1, esz = 2;
  int staleness_mode = 0;                    // 1: explicit δ may be any live version (microbenchmark)
  void* (*alloc_fn)(size_t, void*) = nullptr;   // caller's device allocator (tps_config.dev_alloc)
  void (*free_fn)(void*, void*) = nullptr;
  void* alloc_ctx = nullptr;
  int64_t observed_bytes = 0;                // device free-memory drop across the allocations of init
  int upd_blocks_per_sm = 2;
  std::vector<int> dims;  // global
  std::vector<Layer> layers;
  int classes = 0;

  // ---- device buffers
  std::vector<std::vector<uint16_t*>> act;  // act[slot][k]  bf16 [B, in_elems_k]  (slot count A0 for k=0, Kmax else)
  std::vector<uint16_t*> x_stage;           // im2col first layer: raw input [B, H·W·C] per input slot
  int64_t in0_elems = 0;                    // per-sample elements of the stage input as received
  uint16_t* send_fwd[2] = {nullptr, nullptr};
  uint16_t* gin[2] = {nullptr, nullptr};
  uint16_t* gout[2] = {nullptr, nullptr};
  uint16_t* gwork[3] = {nullptr, nullptr, nullptr};
  float* bpart[3] = {nullptr, nullptr, nullptr};   // column partial sums of gwork[i] (bias gradients)
  float* logits = nullptr;
  uint16_t* gce = nullptr;                  // dlogits, one [B, ld] slot per in-flight mini-batch
  float* loss_rows = nullptr;
  float* losses = nullptr;
  int64_t* loss_ctr = nullptr;               // device: next loss slot (== loss_count once drained)
  int64_t loss_cap = 0, loss_count = 0;
  int32_t* labels_dev = nullptr;
  float* scratch = nullptr;        // bias-gradient reduction scratch of the compute stream
  float* scratch_side = nullptr;   // ... of the optimizer stream (bias steps moved under the GEMMs)
  // graph networks: one gradient buffer per local layer output, two accumulation temps,
  // explicit-patch / patch-gradient scratch, batch-norm reduction scratch
  std::vector<uint16_t*> gbuf;
  uint16_t* gtmp[2] = {nullptr, nullptr};
  uint16_t* patches = nullptr;
  float* dpatches = nullptr;
  double* bn_scr = nullptr;
  float* bn_colsum = nullptr;               // conv epilogue -> next BN: Σx, Σx² per 32-row group
  float* splitk_ws = nullptr;               // split-K partials of weight-gradient GEMMs
  // split-K partials of tile-starved forward / input-gradient GEMMs (compute stream; its own
  // buffer because the weight gradients run concurrently on the weight-gradient stream)
  float* splitk_ws_fd = nullptr;
  int64_t splitk_fd_floats = 0;
  int64_t splitk_floats = 0;
  std::vector<void*> allocs;

  // ---- memory accounting
  int64_t mem_weights = 0, mem_stash = 0, mem_acts = 0, mem_optim = 0, mem_comm = 0, mem_peak = 0;
  int64_t ver_bytes = 0, peak_stash_live = 0;

  // ---- versions and run state
  int64_t latest = 0;
  std::map<int64_t, int64_t> fwd_version;  // mb -> version its forward used (until its backward)
  std::map<int64_t, int> fwd_groups_done;
  std::vector<tps_event> order;
  size_t pos = 0;
  int64_t run_first = 0, run_n = 0;
  bool in_run = false;
  int64_t pending_update = -1;
  std::vector<tps_event> trace;

  // ---- streams, events, transport
  cudaStream_t cs = nullptr;
  bool own_cs = false;
  cudaStream_t s_fin = nullptr, s_fout = nullptr, s_bin = nullptr, s_bout = nullptr;
  cudaStream_t s_upd = nullptr;                        // optimizer stream (overlaps the next GEMMs)
  cudaStream_t caller = cudaStreamLegacy;              // whose prior work a run's inputs depend on
  cudaEvent_t ev_caller = nullptr;
  std::vector<cudaEvent_t> ev_grad_ready, ev_upd_done;  // per layer
  cudaEvent_t ev_bias_in = nullptr, ev_bias_done = nullptr;   // bias step on the optimizer stream
  // split backward (default; TPS_SPLIT_W=0 disables): weight gradients + fused update on their
  // own stream s_w, concurrent with the next layer's input gradient; three rotating gradient
  // buffers (each dgrad waits for the weight gradient / bias step two layers up)
  bool split_w = false;
  bool dual = false;    // split backward: layer k's wgrad + update and layer k-1's dgrad in one launch
  cudaStream_t s_w = nullptr;
  int nsm = 148, part_dgrad = 0;   // SMs of a concurrent (dgrad, wgrad+update) pair given to the dgrad
  std::vector<cudaEvent_t> ev_dg, ev_w_done, ev_bias_l;   // per layer
  std::vector<cudaEvent_t> ev_fwd_ready, ev_fwd_sent;  // [2 * ng]
  std::vector<cudaEvent_t> ev_act_free;                // [A0]
  cudaEvent_t ev_recv = nullptr, ev_gin_free[2] = {nullptr, nullptr}, ev_gout_ready = nullptr,
              ev_bwd_sent[2] = {nullptr, nullptr}, ev_gin_ready = nullptr;
  ncclComm_t c_fin = nullptr, c_fout = nullptr, c_bin = nullptr, c_bout = nullptr;
  tps_pipeline* prev_local = nullptr;
  tps_pipeline* next_local = nullptr;
  // IPC transport: own flag words (written by the neighbours, waited on locally)
  //   [0] fwd_ready     = last forward message (j·ng + grp + 1) stored into my input slots
  //   [1] bwd_ready     = j + 1 once the gradient of mb j is in my receive buffer
  //   [2] fwd_slot_free = j + 1 once the next stage freed its input slot of mb j
  //   [3] bwd_buf_free  = j + 1 once the previous stage finished reading its receive buffer of mb j
  uint64_t* flags = nullptr;
  uint64_t* prev_flags = nullptr;             // mapped flag words of stage s-1 / s+1
  uint64_t* next_flags = nullptr;
  std::vector<uint16_t*> next_in;             // stage s+1's input slots (its A0)
  uint16_t* prev_gin[2] = {nullptr, nullptr}; // stage s-1's gradient receive buffers
  std::vector<void*> ipc_opened;
  bool ipc_connected = false, ipc_direct = false;
  int64_t ipc_next_mb = 0;                    // runs number their mini-batches contiguously from 0
  // data parallelism (NEXT-2): R replicas of this stage
  int dp = 1, dp_rank = 0;
  uint64_t* dp_flags = nullptr;               // own [L][2R]: [k][q] = j+1 when replica q's gradients of
                                              // layer k for mb j are ready; [k][R+q] = j+1 when replica
                                              // q has consumed MY gradients of layer k for mb j
  std::vector<uint64_t*> dp_peer_flags;       // [R] flag arrays of the replicas (own at dp_rank)
  std::vector<std::vector<float*>> dp_dW, dp_db;   // [layer][R] gradient buffers of the replicas
  bool dp_connected = false;
  std::map<std::pair<int64_t, int>, Msg> mbox_fwd;  // keyed (mb, group), filled by prev stage
  std::map<int64_t, Msg> mbox_bwd;                  // keyed mb, filled by next stage

  // ---- profiling / counters
  bool profiling = false;
  std::vector<TimedLaunch> timed;
  std::vector<cudaEvent_t> ev_pool;
  double stat_ms[6] = {0, 0, 0, 0, 0, 0}, stat_work[6] = {0, 0, 0, 0, 0, 0};
  int64_t stat_n[6] = {0, 0, 0, 0, 0, 0};
  int64_t launches = 0;
  bool poisoned = false;
  // ---- per-event device timeline (tps_set_timeline; Chrome trace) and NVTX ranges (TPS_NVTX=1)
  bool timeline = false, own_origin = false, nvtx = false;
  cudaEvent_t tl_origin = nullptr;
  struct TlPending { tps_event e; cudaEvent_t a, b; };
  std::vector<TlPending> tl_pending;
  std::vector<tps_timeline_rec> tl_done;

  int nlayers() const { return static_cast<int>(layers.size()); }
};

namespace {

// ------------------------------------------------------------------ helpers
tps_status dev_alloc(tps_pipeline* p, void** out, size_t bytes, int64_t* category) {
  *out = nullptr;
  if (bytes == 0) return TPS_OK;
  if (p->alloc_fn) {
    *out = p->alloc_fn(bytes, p->alloc_ctx);
    if (!*out) return fail(TPS_E_OOM, "dev_alloc hook failed for %zu bytes", bytes);
  } else {
    cudaError_t e = cudaMalloc(out, bytes);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(TPS_E_OOM, "cudaMalloc(%zu) failed: %s", bytes, cudaGetErrorString(e));
    }
  }
  CUDA_OK(cudaMemset(*out, 0, bytes));
  p->allocs.push_back(*out);
  if (category) *category += static_cast<int64_t>(bytes);
  p->mem_peak = std::max(p->mem_peak, p->mem_weights + p->mem_stash + p->mem_acts + p->mem_optim + p->mem_comm);
  return TPS_OK;
}

template <class T>
tps_status alloc_t(tps_pipeline* p, T** out, size_t count, int64_t* category) {
  void* v = nullptr;
  TPS_TRY(dev_alloc(p, &v, count * sizeof(T), category));
  *out = static_cast<T*>(v);
  return TPS_OK;
}

cudaEvent_t new_event() {
  cudaEvent_t e = nullptr;
  cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  return e;
}

void compute_coeffs(int variant, int blend, int delta, double lambda, float* a, float* b) {
  if (variant == TPS_V) {
    *a = 1.0f;
    *b = 0.0f;
    return;
  }
  const double f = std::exp(-lambda * static_cast<double>(delta));  // Eq. 2
  if (blend == TPS_BLEND_EQ1) {
    *a = static_cast<float>(2.0 - 1.0 / f);                         // Eq. 1
    *b = 0.0f;
  } else {
    *a = static_cast<float>(f);                                     // reading Z1 (CONVEX)
    *b = static_cast<float>(1.0 - f);
  }
}

void build_order(int Kin, int s, int m, int g, int64_t first, int64_t n, std::vector<tps_event>* out) {
  out->clear();
  const int64_t K = std::min<int64_t>(Kin, n);   // K_s mini-batches in flight (Z6)
  auto push_f = [&](int64_t j) {
    for (int a = 0; a < m; a += g) {
      tps_event e{};
      e.stage = s; e.kind = TPS_EV_F; e.micro = a; e.micro_count = g; e.mb = j;
      e.v_used = e.v_latest = -1; e.alpha = 1.f;
      out->push_back(e);
    }
  };
  for (int64_t j = first; j < first + K; ++j) push_f(j);
  for (int64_t j = first; j < first + n; ++j) {
    tps_event e{};
    e.stage = s; e.kind = TPS_EV_B; e.mb = j; e.v_used = e.v_latest = -1; e.alpha = 1.f;
    out->push_back(e);
    e.kind = TPS_EV_U;
    out->push_back(e);
    if (j + K < first + n) push_f(j + K);
  }
}

double gemm_flops(int M, int N, int K) { return 2.0 * M * static_cast<double>(N) * K; }

tps_status run_gemm(tps_pipeline* p, int mode, const tps::GemmOperands& op, const tps::GemmArgs& args, int kind,
                    cudaStream_t stream = nullptr) {
  cudaStream_t gs = stream ? stream : p->cs;
  TimedLaunch tl{};
  if (p->profiling) {
    if (p->ev_pool.size() < 2) {
      for (int i = 0; i < 64; ++i) {
        cudaEvent_t e;
        CUDA_OK(cudaEventCreate(&e));
        p->ev_pool.push_back(e);
      }
    }
    tl.kind = kind;
    tl.work = gemm_flops(args.M, args.N, args.K);
    tl.a = p->ev_pool.back(); p->ev_pool.pop_back();
    tl.b = p->ev_pool.back(); p->ev_pool.pop_back();
    CUDA_OK(cudaEventRecord(tl.a, gs));
  }
  tps::GemmArgs a2 = args;
  const bool fd = mode == tps::GEMM_FWD || mode == tps::GEMM_DGRAD || mode == tps::GEMM_CONV_FWD ||
                  mode == tps::GEMM_CONV_DGRAD;
  a2.ws = fd ? p->splitk_ws_fd : p->splitk_ws;
  a2.ws_floats = fd ? p->splitk_fd_floats : p->splitk_floats;
  a2.tf32 = p->tf ? 1 : 0;
  CUDA_OK(tps::gemm_run(mode, op, a2, gs));
  p->launches += 1;
  if (p->profiling) {
    CUDA_OK(cudaEventRecord(tl.b, gs));
    p->timed.push_back(tl);
  }
  return TPS_OK;
}

// the dual backward launch (gemm_bwd_dual); *done = false when the shapes do not suit it
tps_status run_dual(tps_pipeline* p, const tps::GemmOperands& opw, const tps::GemmArgs& aw,
                    const tps::GemmOperands& opd, const tps::DualArgs& dg, bool* done) {
  TimedLaunch tl{};
  if (p->profiling) {
    if (p->ev_pool.size() < 2) {
      for (int i = 0; i < 64; ++i) {
        cudaEvent_t e;
        CUDA_OK(cudaEventCreate(&e));
        p->ev_pool.push_back(e);
      }
    }
    tl.kind = 5;
    tl.work = gemm_flops(aw.M, aw.N, aw.K) + gemm_flops(dg.M, dg.N, dg.K);
    tl.a = p->ev_pool.back(); p->ev_pool.pop_back();
    tl.b = p->ev_pool.back(); p->ev_pool.pop_back();
    CUDA_OK(cudaEventRecord(tl.a, p->cs));
  }
  const cudaError_t e = tps::gemm_bwd_dual(opw, aw, opd, dg, p->cs);
  *done = e == cudaSuccess;
  if (e == cudaErrorNotSupported) {
    if (p->profiling) { p->ev_pool.push_back(tl.a); p->ev_pool.push_back(tl.b); }
    return TPS_OK;
  }
  CUDA_OK(e);
  p->launches += 1;
  if (p->profiling) {
    CUDA_OK(cudaEventRecord(tl.b, p->cs));
    p->timed.push_back(tl);
  }
  return TPS_OK;
}

tps_status time_begin(tps_pipeline* p, TimedLaunch* tl, int kind, double work, cudaStream_t st = nullptr) {
  if (!p->profiling) return TPS_OK;
  if (p->ev_pool.size() < 2) {
    for (int i = 0; i < 64; ++i) {
      cudaEvent_t e;
      CUDA_OK(cudaEventCreate(&e));
      p->ev_pool.push_back(e);
    }
  }
  tl->kind = kind;
  tl->work = work;
  tl->a = p->ev_pool.back(); p->ev_pool.pop_back();
  tl->b = p->ev_pool.back(); p->ev_pool.pop_back();
  CUDA_OK(cudaEventRecord(tl->a, st ? st : p->cs));
  return TPS_OK;
}

tps_status time_end(tps_pipeline* p, TimedLaunch* tl, cudaStream_t st = nullptr) {
  if (!p->profiling) return TPS_OK;
  CUDA_OK(cudaEventRecord(tl->b, st ? st : p->cs));
  p->timed.push_back(*tl);
  return TPS_OK;
}

tps_status drain_timing(tps_pipeline* p) {
  for (auto& t : p->timed) {
    float ms = 0.f;
    CUDA_OK(cudaEventElapsedTime(&ms, t.a, t.b));
    const int k = t.kind;
    p->stat_ms[k] += ms; p->stat_work[k] += t.work; p->stat_n[k] += 1;
    if (k <= 2 || k == 5) { p->stat_ms[3] += ms; p->stat_work[3] += t.work; p->stat_n[3] += 1; }
    p->ev_pool.push_back(t.a);
    p->ev_pool.push_back(t.b);
  }
  p->timed.clear();
  return TPS_OK;
}

// make the compute stream wait for the optimizer stream (end of a run: the caller's
// stream-ordered view then includes every update of the run)
tps_status join_update_stream(tps_pipeline* p) {
  for (auto e : p->ev_upd_done) CUDA_OK(cudaStreamWaitEvent(p->cs, e, 0));
  return TPS_OK;
}

tps_status sync_streams(tps_pipeline* p) {
  CUDA_OK(cudaStreamSynchronize(p->cs));
  if (p->s_upd) CUDA_OK(cudaStreamSynchronize(p->s_upd));
  if (p->s_w) CUDA_OK(cudaStreamSynchronize(p->s_w));
  return TPS_OK;
}

tps_status check_usable(tps_pipeline* p) {
  if (!p) return fail(TPS_E_INVALID_ARG, "null handle");
  if (p->poisoned) return fail(TPS_E_STATE, "handle poisoned by an earlier device error");
  CUDA_OK(cudaSetDevice(p->device));
  return TPS_OK;
}

// ------------------------------------------------------------------ IPC flag words
typedef CUresult (*StreamValue64Fn)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);

StreamValue64Fn stream_op(const char* name) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
    return nullptr;
  return reinterpret_cast<StreamValue64Fn>(fn);
}

// stream-ordered: `st` stalls (in the GPU front end, no SM held) until *flag >= v
tps_status flag_wait(cudaStream_t st, const uint64_t* flag, uint64_t v) {
  static StreamValue64Fn wait = stream_op("cuStreamWaitValue64");
  if (!wait) return fail(TPS_E_CUDA, "cuStreamWaitValue64 unavailable");
  const CUresult r = wait(reinterpret_cast<CUstream>(st), reinterpret_cast<CUdeviceptr>(flag), v,
                          CU_STREAM_WAIT_VALUE_GEQ);
  if (r != CUDA_SUCCESS) return fail(TPS_E_CUDA, "cuStreamWaitValue64 failed (%d)", static_cast<int>(r));
  return TPS_OK;
}

// stream-ordered: *flag = v after all prior work of `st` (default flags: with a memory barrier,
// so the data the flag announces is visible first)
tps_status flag_write(cudaStream_t st, uint64_t* flag, uint64_t v) {
  static StreamValue64Fn write = stream_op("cuStreamWriteValue64");
  if (!write) return fail(TPS_E_CUDA, "cuStreamWriteValue64 unavailable");
  const CUresult r = write(reinterpret_cast<CUstream>(st), reinterpret_cast<CUdeviceptr>(flag), v,
                           CU_STREAM_WRITE_VALUE_DEFAULT);
  if (r != CUDA_SUCCESS) return fail(TPS_E_CUDA, "cuStreamWriteValue64 failed (%d)", static_cast<int>(r));
  return TPS_OK;
}

// ------------------------------------------------------------------ transport
tps_status send_fwd(tps_pipeline* p, int64_t j, int grp, const void* src, size_t bytes) {
  const int e = static_cast<int>(j & 1) * p->ng + grp;
  CUDA_OK(cudaEventRecord(p->ev_fwd_ready[e], p->cs));
  if (p->transport == TPS_TRANSPORT_NCCL) {
    CUDA_OK(cudaStreamWaitEvent(p->s_fout, p->ev_fwd_ready[e], 0));
    NCCL_OK(ncclSend(src, bytes / p->esz, p->tf ? ncclFloat32 : ncclBfloat16, 1, p->c_fout, p->s_fout));
    CUDA_OK(cudaEventRecord(p->ev_fwd_sent[e], p->s_fout));
  } else if (p->transport == TPS_TRANSPORT_IPC) {
    const uint64_t seq = static_cast<uint64_t>(j) * p->ng + grp + 1;
    if (!p->ipc_direct) {   // copy into the next stage's input slot once it is free
      const int nA0 = static_cast<int>(p->next_in.size());
      CUDA_OK(cudaStreamWaitEvent(p->s_fout, p->ev_fwd_ready[e], 0));
      TPS_TRY(flag_wait(p->s_fout, &p->flags[2], static_cast<uint64_t>(std::max<int64_t>(0, j - nA0 + 1))));
      uint16_t* dst = p->next_in[j % nA0] + static_cast<size_t>(grp) * p->g * p->bsz *
                                                 p->layers[p->nlayers() - 1].out_elems() * p->ew;
      CUDA_OK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, p->s_fout));
      TPS_TRY(flag_write(p->s_fout, &p->next_flags[0], seq));
      CUDA_OK(cudaEventRecord(p->ev_fwd_sent[e], p->s_fout));
    } else {                // the last forward GEMM already stored into the slot: announce it
      TPS_TRY(flag_write(p->cs, &p->next_flags[0], seq));
    }
  } else {
    tps_pipeline* q = p->next_local;
    if (!q) return fail(TPS_E_STATE, "LOCAL transport not linked");
    q->mbox_fwd[{j, grp}] = Msg{src, bytes, p->ev_fwd_ready[e], p->ev_fwd_sent[e]};
  }
  return TPS_OK;
}

tps_status recv_fwd(tps_pipeline* p, int64_t j, int grp, void* dst, size_t bytes) {
  const int slot = static_cast<int>(j % p->A0);
  CUDA_OK(cudaStreamWaitEvent(p->s_fin, p->ev_act_free[slot], 0));
  if (p->transport == TPS_TRANSPORT_NCCL) {
    NCCL_OK(ncclRecv(dst, bytes / p->esz, p->tf ? ncclFloat32 : ncclBfloat16, 0, p->c_fin, p->s_fin));
  } else if (p->transport == TPS_TRANSPORT_IPC) {
    // the previous stage stores straight into this slot; wait for its announcement
    TPS_TRY(flag_wait(p->s_fin, &p->flags[0], static_cast<uint64_t>(j) * p->ng + grp + 1));
  } else {
    auto it = p->mbox_fwd.find({j, grp});
    if (it == p->mbox_fwd.end()) return fail(TPS_E_ORDER, "stage %d: forward input of mb %lld group %d not sent yet", p->s, (long long)j, grp);
    Msg msg = it->second;
    p->mbox_fwd.erase(it);
    if (msg.bytes != bytes) return fail(TPS_E_STATE, "forward message size mismatch");
    CUDA_OK(cudaStreamWaitEvent(p->s_fin, msg.ready, 0));
    CUDA_OK(cudaMemcpyAsync(dst, msg.src, bytes, cudaMemcpyDeviceToDevice, p->s_fin));
    CUDA_OK(cudaEventRecord(msg.consumed, p->s_fin));
  }
  CUDA_OK(cudaEventRecord(p->ev_recv, p->s_fin));
  CUDA_OK(cudaStreamWaitEvent(p->cs, p->ev_recv, 0));
  return TPS_OK;
}

tps_status send_bwd(tps_pipeline* p, int64_t j, const void* src, size_t bytes) {
  const int e = static_cast<int>(j & 1);
  CUDA_OK(cudaEventRecord(p->ev_gout_ready, p->cs));
  if (p->transport == TPS_TRANSPORT_NCCL) {
    CUDA_OK(cudaStreamWaitEvent(p->s_bout, p->ev_gout_ready, 0));
    NCCL_OK(ncclSend(src, bytes / p->esz, p->tf ? ncclFloat32 : ncclBfloat16, 0, p->c_bout, p->s_bout));
    CUDA_OK(cudaEventRecord(p->ev_bwd_sent[e], p->s_bout));
  } else if (p->transport == TPS_TRANSPORT_IPC) {
    if (!p->ipc_direct) {
      CUDA_OK(cudaStreamWaitEvent(p->s_bout, p->ev_gout_ready, 0));
      TPS_TRY(flag_wait(p->s_bout, &p->flags[3], static_cast<uint64_t>(std::max<int64_t>(0, j - 1))));
      CUDA_OK(cudaMemcpyAsync(p->prev_gin[j & 1], src, bytes, cudaMemcpyDeviceToDevice, p->s_bout));
      TPS_TRY(flag_write(p->s_bout, &p->prev_flags[1], static_cast<uint64_t>(j) + 1));
      CUDA_OK(cudaEventRecord(p->ev_bwd_sent[e], p->s_bout));
    } else {                // the first layer's input-gradient GEMM stored into the buffer
      TPS_TRY(flag_write(p->cs, &p->prev_flags[1], static_cast<uint64_t>(j) + 1));
    }
  } else {
    tps_pipeline* q = p->prev_local;
    if (!q) return fail(TPS_E_STATE, "LOCAL transport not linked");
    // the ready event must stay distinct per message: use the sent-event slot's twin
    cudaEvent_t ready = new_event();
    CUDA_OK(cudaEventRecord(ready, p->cs));
    q->mbox_bwd[j] = Msg{src, bytes, ready, p->ev_bwd_sent[e]};
  }
  return TPS_OK;
}

tps_status recv_bwd(tps_pipeline* p, int64_t j, void* dst, size_t bytes) {
  const int e = static_cast<int>(j & 1);
  CUDA_OK(cudaStreamWaitEvent(p->s_bin, p->ev_gin_free[e], 0));
  if (p->transport == TPS_TRANSPORT_NCCL) {
    NCCL_OK(ncclRecv(dst, bytes / p->esz, p->tf ? ncclFloat32 : ncclBfloat16, 1, p->c_bin, p->s_bin));
  } else if (p->transport == TPS_TRANSPORT_IPC) {
    TPS_TRY(flag_wait(p->s_bin, &p->flags[1], static_cast<uint64_t>(j) + 1));
  } else {
    auto it = p->mbox_bwd.find(j);
    if (it == p->mbox_bwd.end()) return fail(TPS_E_ORDER, "stage %d: gradient of mb %lld not sent yet", p->s, (long long)j);
    Msg msg = it->second;
    p->mbox_bwd.erase(it);
    if (msg.bytes != bytes) return fail(TPS_E_STATE, "backward message size mismatch");
    CUDA_OK(cudaStreamWaitEvent(p->s_bin, msg.ready, 0));
    CUDA_OK(cudaMemcpyAsync(dst, msg.src, bytes, cudaMemcpyDeviceToDevice, p->s_bin));
    CUDA_OK(cudaEventRecord(msg.consumed, p->s_bin));
    cudaEventDestroy(msg.ready);  // destruction is deferred by the runtime until the event completes
  }
  CUDA_OK(cudaEventRecord(p->ev_gin_ready, p->s_bin));
  CUDA_OK(cudaStreamWaitEvent(p->cs, p->ev_gin_ready, 0));
  return TPS_OK;
}

// ------------------------------------------------------------------ order checking
tps_status expect(tps_pipeline* p, int kind, int64_t mb, int micro, int count) {
  if (!p->in_run) return fail(TPS_E_ORDER, "stage %d: no run declared (tps_begin_run)", p->s);
  if (p->pos >= p->order.size()) return fail(TPS_E_ORDER, "stage %d: run already complete", p->s);
  const tps_event& e = p->order[p->pos];
  static const char* kn[3] = {"F", "B", "U"};
  if (e.kind != kind || e.mb != mb || (kind == TPS_EV_F && (e.micro != micro || e.micro_count != count)))
    return fail(TPS_E_ORDER, "stage %d: got %s(mb=%lld, micro=%d, count=%d), next static event is %s(mb=%lld, micro=%d, count=%d)",
                p->s, kn[kind], (long long)mb, micro, count, kn[e.kind], (long long)e.mb, e.micro, e.micro_count);
  return TPS_OK;
}

void advance(tps_pipeline* p) {
  p->pos += 1;
  if (p->pos == p->order.size()) p->in_run = false;
}

void update_stash_peak(tps_pipeline* p) {
  // live versions = latest + distinct versions referenced by forwarded-but-not-backwarded mbs
  std::vector<int64_t> live{p->latest};
  for (auto& kv : p->fwd_version)
    if (std::find(live.begin(), live.end(), kv.second) == live.end()) live.push_back(kv.second);
  // V keeps one version (R = 1): versions of in-flight forwards are already overwritten
  const int64_t n_live = std::min<int64_t>(static_cast<int64_t>(live.size()), p->R);
  const int64_t stash = (n_live - 1) * p->ver_bytes;
  p->peak_stash_live = std::max(p->peak_stash_live, stash);
}

// ------------------------------------------------------------------ data parallelism
// Layer k's gradients of mb j are complete on the compute stream: on the optimizer stream,
// announce them to every replica, wait for theirs, run the fused replica-average + SGD step
// (weights and bias), then tell every replica its gradients were consumed.
tps_status dp_update(tps_pipeline* p, Layer& L, int k, int64_t j, int64_t vn) {
  cudaStream_t us = p->s_upd;
  const int R = p->dp;
  CUDA_OK(cudaEventRecord(p->ev_grad_ready[k], p->cs));
  CUDA_OK(cudaStreamWaitEvent(us, p->ev_grad_ready[k], 0));
  const size_t base = static_cast<size_t>(k) * 2 * R;
  const uint64_t v = static_cast<uint64_t>(j) + 1;
  for (int q = 0; q < R; ++q)
    if (q != p->dp_rank) TPS_TRY(flag_write(us, &p->dp_peer_flags[q][base + p->dp_rank], v));
  for (int q = 0; q < R; ++q)
    if (q != p->dp_rank) TPS_TRY(flag_wait(us, &p->dp_flags[base + q], v));
  tps::GradList gw{}, gb{};
  gw.n = gb.n = R;
  for (int q = 0; q < R; ++q) {
    gw.p[q] = p->dp_dW[k][q];
    gb.p[q] = p->dp_db[k][q];
  }
  const int64_t n = static_cast<int64_t>(L.Np) * L.Kp;
  TimedLaunch tl{};
  TPS_TRY(time_begin(p, &tl, 4, (p->mu != 0.f ? 18.0 + 4.0 * R : 10.0 + 4.0 * R) * n, us));
  CUDA_OK(tps::launch_sgd_update_dp(L.W, L.mW, gw, L.ver[vn % p->R], n, p->lr, p->mu, p->wd, us));
  TPS_TRY(time_end(p, &tl, us));
  CUDA_OK(tps::launch_sgd_update_dp(L.b, L.mb, gb, nullptr, L.Np, p->lr, p->mu, p->wd, us));
  p->launches += 2;
  for (int q = 0; q < R; ++q)
    if (q != p->dp_rank) TPS_TRY(flag_write(us, &p->dp_peer_flags[q][base + R + p->dp_rank], v));
  return TPS_OK;
}

// ------------------------------------------------------------------ the three events
// one layer's forward on rows [r0, r0+nr) of the group: input Xin (this layer's stash rows),
// output `out` (next layer's stash rows, the send buffer, or fp32 logits)
tps_status layer_forward(tps_pipeline* p, Layer& Lk, int nr, const uint16_t* Xin, void* out, bool logits,
                         int64_t v) {
  const bool relu = !logits;
  if (Lk.kind == TPS_LAYER_MAXPOOL2) {
    CUDA_OK(tps::launch_maxpool2_fwd(Xin, static_cast<uint16_t*>(out), nr, Lk.H, Lk.Wd, Lk.Ci, p->cs));
    p->launches += 1;
    return TPS_OK;
  }
  tps::GemmArgs ga{};
  ga.alpha = 1.f; ga.bias = Lk.b; ga.xa = 1.f; ga.xb = 0.f; ga.relu = relu ? 1 : 0; ga.out_f32 = logits ? 1 : 0;
  ga.out = out; ga.ldo = Lk.Np;
  ga.M = nr * Lk.hw_out; ga.N = Lk.Np; ga.K = Lk.Kp;
  if (Lk.kind == TPS_LAYER_CONV3X3 && !Lk.im2col) {
    // implicit im2col: Y[n·H·W, Co] = conv3x3(X) via 4-D TMA boxes of the NHWC input
    tps::GemmOperands op{Xin, 0, Lk.ver[v % p->R], Lk.Kp, nullptr};
    op.cv = tps::ConvGeom{nr, Lk.H, Lk.Wd, Lk.Ci};
    return run_gemm(p, tps::GEMM_CONV_FWD, op, ga, 0);
  }
  // Linear, or the first conv on its explicit patches [n·H·W, Kp]
  tps::GemmOperands op{Xin, Lk.Kp, Lk.ver[v % p->R], Lk.Kp, nullptr};
  return run_gemm(p, tps::GEMM_FWD, op, ga, 0);
}

// ------------------------------------------------------------------ graph networks (ResNet)
// local tensor t: -1 = stage input (input slot), k = output of local layer k (stash slot)
// relu-mask bytes of rows [r0, ...) of stash slot `slot` (null: the backward reads y)
uint8_t* relu_mask_at(Layer& L, int slot, int r0) {
  if (L.relu_mask.empty()) return nullptr;
  return L.relu_mask[slot] + static_cast<size_t>(r0) * L.hw_in * (L.Ci / 8);
}

uint16_t* gtensor(tps_pipeline* p, int slot0, int slot, int t) {
  return t < 0 ? p->act[slot0][0] : p->act[slot][t + 1];
}
int64_t gelems(tps_pipeline* p, int t) { return t < 0 ? p->in0_elems : p->layers[t].out_elems(); }

tps_status graph_forward(tps_pipeline* p, int64_t j, int a0, int cnt, int64_t v) {
  const int slot0 = static_cast<int>(j % p->A0), slot = static_cast<int>(j % p->Kmax);
  const int r0 = a0 * p->bsz, nr = cnt * p->bsz;
  const int nl = p->nlayers();
  for (int k = 0; k < nl; ++k) {
    Layer& L = p->layers[k];
    if (L.has_w()) CUDA_OK(cudaStreamWaitEvent(p->cs, p->ev_upd_done[k], 0));   // latest version written
    const uint16_t* X = gtensor(p, slot0, slot, L.src) + static_cast<size_t>(r0) * gelems(p, L.src);
    const bool head = L.kind == TPS_LAYER_LINEAR;
    void* out = head ? static_cast<void*>(p->logits + static_cast<size_t>(r0) * L.Np)
                     : static_cast<void*>(gtensor(p, slot0, slot, k) + static_cast<size_t>(r0) * L.out_elems());
    switch (L.kind) {
      case TPS_LAYER_CONV: {
        tps::GemmArgs ga{};
        ga.alpha = 1.f; ga.xa = 1.f; ga.out = out; ga.ldo = L.Co;
        ga.M = nr * L.hw_out; ga.N = L.Co; ga.K = L.Kp;
        if (L.stats_to_next) {
          ga.colsum = p->bn_colsum;
          ga.colsum_sq = 1;
        }
        const uint16_t* Wv = L.ver[v % p->R];
        if (L.conv_mode == 1 || L.conv_mode == 3) {
          tps::GemmOperands op{X, 0, Wv, L.Kp, nullptr};
          op.cv = tps::ConvGeom{nr, L.H, L.Wd, L.Ci, 1, L.k, L.st, L.pad, L.Ho, L.Wo};
          TPS_TRY(run_gemm(p, tps::GEMM_CONV_FWD, op, ga, 0));
        } else {
          const uint16_t* A = X;
          if (L.conv_mode == 2) {
            CUDA_OK(tps::launch_im2col(X, p->patches, nr, L.H, L.Wd, L.Ci, L.k, L.st, L.pad, L.Kp, p->cs));
            p->launches += 1;
            A = p->patches;
          }
          tps::GemmOperands op{A, L.Kp, Wv, L.Kp, nullptr};
          TPS_TRY(run_gemm(p, tps::GEMM_FWD, op, ga, 0));
        }
        break;
      }
      case TPS_LAYER_BN: {
        const uint16_t* res = L.res >= -1 ? gtensor(p, slot0, slot, L.res) + static_cast<size_t>(r0) * gelems(p, L.res)
                                          : nullptr;
        if (k > 0 && L.src == k - 1 && p->layers[k - 1].stats_to_next) {
          CUDA_OK(tps::launch_bn_forward_colsum(p->bn_colsum, X, res, static_cast<uint16_t*>(out), L.verf[v % p->R], L.b,
                                                L.mean[slot] + static_cast<size_t>(a0) * L.Ci,
                                                L.invstd[slot] + static_cast<size_t>(a0) * L.Ci, cnt,
                                                p->bsz * L.hw_in, L.Ci, L.relu ? 1 : 0, p->bn_scr, p->cs,
                                                relu_mask_at(L, slot, r0)));
          p->launches += 3;
        } else {
          CUDA_OK(tps::launch_bn_forward(X, res, static_cast<uint16_t*>(out), L.verf[v % p->R], L.b,
                                         L.mean[slot] + static_cast<size_t>(a0) * L.Ci,
                                         L.invstd[slot] + static_cast<size_t>(a0) * L.Ci, cnt, p->bsz * L.hw_in, L.Ci,
                                         L.relu ? 1 : 0, p->bn_scr, p->cs, relu_mask_at(L, slot, r0)));
          p->launches += 3;
        }
        break;
      }
      case TPS_LAYER_MAXPOOL3:
        if (!L.argmax.empty())
          CUDA_OK(tps::launch_maxpool3_fwd_idx(X, static_cast<uint16_t*>(out),
                                               L.argmax[slot] + static_cast<size_t>(r0) * L.out_elems(), nr, L.H,
                                               L.Wd, L.Ci, p->cs));
        else
          CUDA_OK(tps::launch_maxpool3_fwd(X, static_cast<uint16_t*>(out), nr, L.H, L.Wd, L.Ci, p->cs));
        p->launches += 1;
        break;
      case TPS_LAYER_AVGPOOL:
        CUDA_OK(tps::launch_avgpool_fwd(X, static_cast<uint16_t*>(out), nr, L.hw_in, L.Ci, p->cs));
        p->launches += 1;
        break;
      default: {  // the head: fp32 logits
        tps::GemmArgs ga{};
        ga.alpha = 1.f; ga.xa = 1.f; ga.bias = L.b; ga.out_f32 = 1; ga.out = out; ga.ldo = L.Np;
        ga.M = nr; ga.N = L.Np; ga.K = L.Kp;
        tps::GemmOperands op{X, L.Kp, L.ver[v % p->R], L.Kp, nullptr};
        TPS_TRY(run_gemm(p, tps::GEMM_FWD, op, ga, 0));
      }
    }
  }
  return TPS_OK;
}

// gradient accumulation target of tensor t in the current backward: the first contribution
// writes the tensor's gradient buffer, later ones (a block input read by two layers) are
// added to it (bf16(stored + new), reverse layer order, like oracle/graph.py)
struct GradTarget {
  uint16_t* buf;     // gradient buffer of the tensor
  bool filled;       // already holds a contribution
};

tps_status graph_backward(tps_pipeline* p, int64_t j, int64_t v_used, int64_t vl, int64_t vn, float alpha, float beta,
                          bool blend_on_load, const uint16_t* G_last) {
  const int slot0 = static_cast<int>(j % p->A0), slot = static_cast<int>(j % p->Kmax);
  const int nl = p->nlayers();
  const int B = p->B;
  std::vector<char> filled(nl + 1, 0);
  bool gout_waited = false;
  auto target = [&](int t) -> GradTarget {
    if (t < 0) {
      if (!gout_waited) {  // gout of mb j-2 has left
        cudaStreamWaitEvent(p->cs, p->ev_bwd_sent[j & 1], 0);
        gout_waited = true;
      }
      return GradTarget{p->gout[j & 1], filled[0] != 0};
    }
    return GradTarget{p->gbuf[t], filled[t + 1] != 0};
  };
  auto mark = [&](int t) { filled[t + 1] = 1; };
  // contribution written to `tmp` when the target is already filled: add it in
  auto settle = [&](int t, const GradTarget& g, uint16_t* tmp) -> tps_status {
    if (g.filled) {
      CUDA_OK(tps::launch_add_bf16(g.buf, tmp, static_cast<int64_t>(B) * gelems(p, t), p->cs));
      p->launches += 1;
    }
    mark(t);
    return TPS_OK;
  };
  auto update = [&](Layer& L, int k, bool gemm_grad) -> tps_status {
    // U(j) directly follows B(j) (reading Z7): issue this layer's SGD step now on the
    // optimizer stream; the next forward of layer k waits for ev_upd_done[k]
    cudaStream_t us = p->s_upd;
    CUDA_OK(cudaEventRecord(p->ev_grad_ready[k], p->cs));
    CUDA_OK(cudaStreamWaitEvent(us, p->ev_grad_ready[k], 0));
    const int64_t n = static_cast<int64_t>(L.Np) * L.Kp;
    TimedLaunch tl{};
    if (gemm_grad) TPS_TRY(time_begin(p, &tl, 4, (p->mu != 0.f ? 22.0 : 14.0) * n, us));
    CUDA_OK(tps::launch_sgd_update(L.W, L.mW, L.dW, L.kind == TPS_LAYER_BN ? nullptr : L.ver[vn % p->R], n, p->lr,
                                   p->mu, p->wd, us, p->upd_blocks_per_sm));
    if (gemm_grad) TPS_TRY(time_end(p, &tl, us));
    p->launches += 1;
    if (L.kind == TPS_LAYER_BN)
      CUDA_OK(cudaMemcpyAsync(L.verf[vn % p->R], L.W, static_cast<size_t>(n) * 4, cudaMemcpyDeviceToDevice, us));
    if (L.b) {
      CUDA_OK(tps::launch_sgd_update(L.b, L.mb, L.db, nullptr, L.Np, p->lr, p->mu, p->wd, us));
      p->launches += 1;
    }
    CUDA_OK(cudaEventRecord(p->ev_upd_done[k], us));
    return TPS_OK;
  };
  for (int k = nl - 1; k >= 0; --k) {
    Layer& L = p->layers[k];
    // the previous update of this layer (optimizer stream) must be done: it reads dW / db,
    // which this backward rewrites, and (V) it writes the weights this backward reads
    if (L.has_w()) CUDA_OK(cudaStreamWaitEvent(p->cs, p->ev_upd_done[k], 0));
    const uint16_t* g;
    if (k == nl - 1) {
      g = G_last;
    } else {
      if (!filled[k + 1]) return fail(TPS_E_STATE, "layer %d output has no gradient", L.gidx);
      g = p->gbuf[k];
    }
    const uint16_t* X = gtensor(p, slot0, slot, L.src);
    const bool need_dx = !(p->first && L.src == -1);
    switch (L.kind) {
      case TPS_LAYER_CONV:
      case TPS_LAYER_LINEAR: {
        const bool head = L.kind == TPS_LAYER_LINEAR;
        if (need_dx) {
          // input gradient first: the update must not rewrite this layer's weights before
          const GradTarget dst = target(L.src);
          tps::GemmArgs ga{};
          ga.alpha = 1.f; ga.xa = 1.f; ga.xb = 0.f;
          const int ldg = head ? L.Np : L.Co;
          tps::GemmOperands op{g, ldg, L.ver[v_used % p->R], L.Kp, nullptr};
          const bool expl = !head && (L.conv_mode == 2 || L.conv_mode == 3);
          if (expl) {      // patch gradient (fp32), then col2im adds it into the target
            ga.out = p->dpatches; ga.out_f32 = 1; ga.ldo = L.Kp;
            ga.M = B * L.hw_out; ga.N = L.Kp; ga.K = L.Co;
          } else {
            ga.out = dst.buf; ga.ldo = head ? L.Kp : L.Ci; ga.addend = dst.filled ? dst.buf : nullptr;
            ga.M = B * L.hw_in; ga.N = head ? L.Kp : L.Ci; ga.K = head ? L.Np : L.Co;
          }
          int mode = tps::GEMM_DGRAD;
          if (!head && L.conv_mode == 1) {
            op.cv = tps::ConvGeom{B, L.H, L.Wd, L.Co, 1, 3, 1, 1, L.H, L.Wd};
            op.Cw = L.Ci;
            ga.K = 9 * L.Co;
            mode = tps::GEMM_CONV_DGRAD;
          }
          if (blend_on_load) {
            op.B2 = L.ver[vl % p->R];
            ga.xa = alpha; ga.xb = beta;
            mode = mode == tps::GEMM_CONV_DGRAD ? tps::GEMM_CONV_DGRAD_BLEND : tps::GEMM_DGRAD_BLEND;
          } else {
            ga.alpha = (p->variant == TPS_I) ? alpha : 1.f;   // EQ1: α·(G·W_stash) = G·(α·W_stash)
          }
          TPS_TRY(run_gemm(p, mode, op, ga, 1));
          if (expl) {
            CUDA_OK(tps::launch_col2im(p->dpatches, dst.buf, dst.filled ? dst.buf : nullptr, B, L.H, L.Wd, L.Ci, L.k,
                                       L.st, L.pad, L.Kp, p->cs));
            p->launches += 1;
          }
          mark(L.src);
        }
        // weight gradient dW[Np, Kp] = Gᵀ·(input or its patches)
        tps::GemmArgs ga{};
        ga.M = L.Np; ga.N = L.Kp; ga.out = L.dW; ga.ldo = L.Kp; ga.out_f32 = 1; ga.alpha = 1.f; ga.xa = 1.f;
        if (!head && (L.conv_mode == 1 || L.conv_mode == 3)) {
          ga.K = B * L.hw_out;
          tps::GemmOperands op{g, L.Np, X, 0, nullptr};
          op.cv = tps::ConvGeom{B, L.H, L.Wd, L.Ci, 1, L.k, L.st, L.pad, L.Ho, L.Wo};
          TPS_TRY(run_gemm(p, tps::GEMM_CONV_WGRAD, op, ga, 2));
        } else {
          const uint16_t* Xb = X;
          if (!head && L.conv_mode == 2) {
            CUDA_OK(tps::launch_im2col(X, p->patches, B, L.H, L.Wd, L.Ci, L.k, L.st, L.pad, L.Kp, p->cs));
            p->launches += 1;
            Xb = p->patches;
          }
          ga.K = head ? B : B * L.hw_out;
          tps::GemmOperands op{g, L.Np, Xb, L.Kp, nullptr};
          TPS_TRY(run_gemm(p, tps::GEMM_WGRAD, op, ga, 2));
        }
        if (head) {
          CUDA_OK(tps::launch_bias_grad(g, B, L.Np, L.Np, L.db, p->scratch, p->cs));
          p->launches += 1;
        }
        TPS_TRY(update(L, k, true));
        break;
      }
      case TPS_LAYER_BN: {
        const uint16_t* y = gtensor(p, slot0, slot, k);
        uint16_t* dres = nullptr;
        GradTarget rt{nullptr, false};
        if (L.res >= -1) {
          rt = target(L.res);
          dres = rt.filled ? p->gtmp[0] : rt.buf;
        }
        const GradTarget xt = target(L.src);
        uint16_t* dx = xt.filled ? p->gtmp[1] : xt.buf;
        // γ_res = α·γ_stash + β·γ_latest (V: α = 1, β = 0 on the latest; EQ1: β = 0)
        const float ga = p->variant == TPS_I ? alpha : 1.f, gb = p->variant == TPS_I ? beta : 0.f;
        CUDA_OK(tps::launch_bn_backward(g, y, X, L.mean[slot], L.invstd[slot], L.verf[v_used % p->R],
                                        L.verf[vl % p->R], ga, gb, p->m, p->bsz * L.hw_in, L.Ci, L.relu ? 1 : 0, dx,
                                        dres, L.dW, L.db, p->bn_scr, p->cs, relu_mask_at(L, slot, 0)));
        p->launches += 3;
        if (L.res >= -1) TPS_TRY(settle(L.res, rt, p->gtmp[0]));
        TPS_TRY(settle(L.src, xt, p->gtmp[1]));
        TPS_TRY(update(L, k, false));
        break;
      }
      case TPS_LAYER_MAXPOOL3:
      case TPS_LAYER_AVGPOOL: {
        if (!need_dx) break;
        const GradTarget xt = target(L.src);
        uint16_t* dx = xt.filled ? p->gtmp[1] : xt.buf;
        if (L.kind == TPS_LAYER_MAXPOOL3 && !L.argmax.empty())
          CUDA_OK(tps::launch_maxpool3_bwd_idx(L.argmax[slot], g, dx, B, L.H, L.Wd, L.Ci, p->cs));
        else if (L.kind == TPS_LAYER_MAXPOOL3)
          CUDA_OK(tps::launch_maxpool3_bwd(X, g, dx, B, L.H, L.Wd, L.Ci, p->cs));
        else CUDA_OK(tps::launch_avgpool_bwd(g, dx, B, L.hw_in, L.Ci, p->cs));
        p->launches += 1;
        TPS_TRY(settle(L.src, xt, p->gtmp[1]));
        break;
      }
      default:
        return fail(TPS_E_STATE, "layer kind %d in a graph network", L.kind);
    }
  }
  if (!p->first && !filled[0]) return fail(TPS_E_STATE, "stage input received no gradient");
  return TPS_OK;
}

tps_status do_forward(tps_pipeline* p, int64_t j, int a0, int cnt, const void* x, const int32_t* labels) {
  TPS_TRY(expect(p, TPS_EV_F, j, a0, cnt));
  if (p->first && !x) return fail(TPS_E_INVALID_ARG, "stage 0 forward needs x");
  if (p->last && !labels) return fail(TPS_E_INVALID_ARG, "last stage forward needs labels");
  const int grp = a0 / p->g;
  // a rejected call must leave the handle untouched: check the LOCAL mailbox up front
  if (!p->first && p->transport == TPS_TRANSPORT_LOCAL && !p->mbox_fwd.count({j, grp}))
    return fail(TPS_E_ORDER, "stage %d: forward input of mb %lld group %d not sent yet", p->s, (long long)j, grp);
  const int r0 = a0 * p->bsz, nr = cnt * p->bsz;
  const int64_t v = p->latest;
  if (a0 == 0) p->fwd_version[j] = v;
  const int slot0 = static_cast<int>(j % p->A0);
  const int slot = static_cast<int>(j % p->Kmax);
  Layer& L0 = p->layers[0];
  uint16_t* X = p->act[slot0][0] + static_cast<size_t>(r0) * (p->graph ? p->in0_elems : L0.in_elems()) * p->ew;
  if (p->first && p->graph) {
    CUDA_OK(cudaStreamWaitEvent(p->s_fin, p->ev_act_free[slot0], 0));
    CUDA_OK(cudaMemcpyAsync(X, x, static_cast<size_t>(nr) * p->in0_elems * 2, cudaMemcpyDefault, p->s_fin));
    CUDA_OK(cudaEventRecord(p->ev_recv, p->s_fin));
    CUDA_OK(cudaStreamWaitEvent(p->cs, p->ev_recv, 0));
  } else if (p->first) {
    // input copy (device pool or pinned host) on the input stream: with the extra input
    // slot it overlaps the backward/update still running on the compute stream
    CUDA_OK(cudaStreamWaitEvent(p->s_fin, p->ev_act_free[slot0], 0));
    if (L0.im2col) {
      uint16_t* xs = p->x_stage[slot0] + static_cast<size_t>(r0) * p->in0_elems;
      CUDA_OK(cudaMemcpyAsync(xs, x, static_cast<size_t>(nr) * p->in0_elems * 2, cudaMemcpyDefault, p->s_fin));
    } else if (L0.kind == TPS_LAYER_LINEAR && L0.in != L0.Kp) {
      const size_t w = static_cast<size_t>(L0.in) * p->esz;   // pad the rows to the 16-aligned ld
      CUDA_OK(cudaMemcpy2DAsync(X, static_cast<size_t>(L0.Kp) * p->esz, x, w, w, nr, cudaMemcpyDefault, p->s_fin));
    } else if (L0.kind == TPS_LAYER_LINEAR) {
      CUDA_OK(cudaMemcpyAsync(X, x, static_cast<size_t>(nr) * L0.Kp * p->esz, cudaMemcpyDefault, p->s_fin));
    } else {
      CUDA_OK(cudaMemcpyAsync(X, x, static_cast<size_t>(nr) * L0.in_elems() * 2, cudaMemcpyDefault, p->s_fin));
    }
    CUDA_OK(cudaEventRecord(p->ev_recv, p->s_fin));
    CUDA_OK(cudaStreamWaitEvent(p->cs, p->ev_recv, 0));
    if (L0.im2col) {
      CUDA_OK(tps::launch_im2col3x3(p->x_stage[slot0] + static_cast<size_t>(r0) * p->in0_elems, X, nr, L0.H, L0.Wd,
                                    L0.Ci, L0.Kp, p->cs));
      p->launches += 1;
    }
  } else {
    TPS_TRY(recv_fwd(p, j, grp, X, static_cast<size_t>(nr) * (p->graph ? p->in0_elems : L0.in_elems()) * p->esz));
  }
  if (!p->last) {  // the send buffer of mb j-2 must have left
    CUDA_OK(cudaStreamWaitEvent(p->cs, p->ev_fwd_sent[static_cast<int>(j & 1) * p->ng + grp], 0));
  }
  const int nl = p->nlayers();
  const uint16_t* Xin = X;
  if (p->graph) TPS_TRY(graph_forward(p, j, a0, cnt, v));
  for (int k = 0; k < (p->graph ? 0 : nl); ++k) {
    Layer& Lk = p->layers[k];
    if (Lk.has_w()) CUDA_OK(cudaStreamWaitEvent(p->cs, p->ev_upd_done[k], 0));   // latest version written
    void* out;
    const bool logits = (k == nl - 1) && p->last;
    if (k < nl - 1) {
      out = p->act[slot][k + 1] + static_cast<size_t>(r0) * Lk.out_elems() * p->ew;
    } else if (!p->last && p->ipc_direct) {
      // fused compute + send: the epilogue stores into the next stage's input slot (NVLink peer
      // memory across GPUs) once that stage has freed it (its backward of mb j - A0_next)
      const int nA0 = static_cast<int>(p->next_in.size());
      TPS_TRY(flag_wait(p->cs, &p->flags[2], static_cast<uint64_t>(std::max<int64_t>(0, j - nA0 + 1))));
      out = p->next_in[j % nA0] + static_cast<size_t>(r0) * Lk.out_elems() * p->ew;
    } else if (!p->last) {
      out = p->send_fwd[j & 1] + static_cast<size_t>(r0) * Lk.out_elems() * p->ew;
    } else {
      out = p->logits + static_cast<size_t>(r0) * Lk.Np;
    }
    TPS_TRY(layer_forward(p, Lk, nr, Xin, out, logits, v));
    Xin = static_cast<const uint16_t*>(out);
  }
  if (p->last) {
    Layer& Ll = p->layers[nl - 1];
    const int32_t* lab = labels;
    if (is_host_ptr(labels)) {
      CUDA_OK(cudaMemcpyAsync(p->labels_dev + r0, labels, static_cast<size_t>(nr) * 4, cudaMemcpyHostToDevice, p->cs));
      lab = p->labels_dev + r0;
    }
    CUDA_OK(tps::launch_softmax_xent(p->logits + static_cast<size_t>(r0) * Ll.Np, Ll.Np, lab, nr, p->classes, p->B,
                                     p->loss_rows + r0,
                                     p->gce + (static_cast<size_t>(slot) * p->B + r0) * Ll.Np * p->ew, Ll.Np, p->cs,
                                     p->tf ? 1 : 0));
    p->launches += 1;
    if (a0 + cnt == p->m) {
      if (p->loss_count >= p->loss_cap) return fail(TPS_E_STATE, "loss buffer full (%lld mini-batches)", (long long)p->loss_cap);
      CUDA_OK(tps::launch_loss_mean(p->loss_rows, p->B, p->losses, p->loss_ctr, p->cs));
      p->loss_count += 1;
      p->launches += 1;
    }
  } else {
    Layer& Ll = p->layers[nl - 1];
    uint16_t* sb = p->graph ? p->act[slot][nl] : p->send_fwd[j & 1];   // graph: send from the stash
    TPS_TRY(send_fwd(p, j, grp, sb + static_cast<size_t>(r0) * Ll.out_elems() * p->ew,
                     static_cast<size_t>(nr) * Ll.out_elems() * p->esz));
  }
  tps_event e{};
  e.stage = p->s; e.kind = TPS_EV_F; e.micro = a0; e.micro_count = cnt; e.mb = j;
  e.v_used = v; e.v_latest = v; e.delta = 0; e.alpha = 1.f; e.beta = 0.f;
  p->trace.push_back(e);
  p->fwd_groups_done[j] += 1;
  update_stash_peak(p);
  advance(p);
  return TPS_OK;
}

tps_status do_backward(tps_pipeline* p, int64_t j, int staleness) {
  TPS_TRY(expect(p, TPS_EV_B, j, -1, 0));
  auto fv = p->fwd_version.find(j);
  if (fv == p->fwd_version.end()) return fail(TPS_E_ORDER, "backward of mb %lld without its forward", (long long)j);
  const int64_t vf = fv->second, vl = p->latest;
  const int64_t dlog = vl - vf;
  int64_t delta, v_used;
  if (p->variant == TPS_V) {
    delta = 0;          // V reads the latest weights: zero staleness
    v_used = vl;
    if (staleness > 0) return fail(TPS_E_STALENESS, "V-TiMePReSt has no stash (requested staleness %d)", staleness);
  } else {
    delta = staleness >= 0 ? staleness : dlog;
    if (staleness >= 0 && staleness != dlog && p->staleness_mode == 0)
      return fail(TPS_E_STALENESS, "explicit staleness %d != logged %lld for mb %lld", staleness, (long long)dlog, (long long)j);
    v_used = vl - delta;
    if (v_used < 0 || v_used < vl - p->R + 1)
      return fail(TPS_E_STALENESS, "no live stash for staleness %lld (latest %lld, ring of %d)", (long long)delta,
                  (long long)vl, p->R);
  }
  float alpha, beta;
  compute_coeffs(p->variant, p->blend, static_cast<int>(delta), p->lambda, &alpha, &beta);
  const int nl = p->nlayers();
  Layer& Ll = p->layers[nl - 1];
  if (!p->last && p->transport == TPS_TRANSPORT_LOCAL && !p->mbox_bwd.count(j))
    return fail(TPS_E_ORDER, "stage %d: gradient of mb %lld not sent yet", p->s, (long long)j);
  const uint16_t* G;
  if (p->last) {
    G = p->gce + static_cast<size_t>(j % p->Kmax) * p->B * Ll.Np * p->ew;   // slot of mb j (K_s may exceed 1, S = 1)
  } else {
    TPS_TRY(recv_bwd(p, j, p->gin[j & 1], static_cast<size_t>(p->B) * Ll.out_elems() * p->esz));
    G = p->gin[j & 1];
  }
  const int slot0 = static_cast<int>(j % p->A0);
  const int slot = static_cast<int>(j % p->Kmax);
  const int B = p->B;
  int wbuf = 0;
  const int64_t vn = vl + 1;   // version the update of this mini-batch produces
  const bool blend_on_load = p->variant == TPS_I && delta > 0 && (p->blend == TPS_BLEND_CONVEX || p->eq1_on_load);
  for (Layer& L : p->layers) { L.bias_part = nullptr; L.bias_groups = 0; }
  if (p->graph) TPS_TRY(graph_backward(p, j, v_used, vl, vn, alpha, beta, blend_on_load, G));
  // dual launches (p->dual): layer k's fused wgrad + update is held back and issued together with
  // layer k-1's input gradient (independent: different layers' weights, distinct gradient buffers
  // of the three-way rotation), on the compute stream
  struct PendingW {
    int k = -1;
    tps::GemmOperands op{};
    tps::GemmArgs ga{};
    bool bias_side = false;
  } pend;
  // a plain Linear input gradient of layer kk that can share a launch
  auto dgrad_pairable = [&](int kk) {
    if (kk < 0 || !p->dual || blend_on_load || p->part_dgrad > 0 || p->bpart[0]) return false;
    const Layer& L = p->layers[kk];
    return L.gidx > 0 && L.kind == TPS_LAYER_LINEAR;
  };
  // events that follow layer kk's fused wgrad + update on the split backward (stream st)
  auto finish_w = [&](int kk, bool bside, cudaStream_t st) -> tps_status {
    CUDA_OK(cudaEventRecord(p->ev_w_done[kk], st));
    if (bside) {
      CUDA_OK(cudaStreamWaitEvent(p->s_upd, p->ev_w_done[kk], 0));
      CUDA_OK(cudaEventRecord(p->ev_upd_done[kk], p->s_upd));
    } else {
      CUDA_OK(cudaEventRecord(p->ev_bias_l[kk], p->cs));   // bias ran on the compute stream
      CUDA_OK(cudaEventRecord(p->ev_upd_done[kk], st));
    }
    return TPS_OK;
  };
  auto flush_pending = [&]() -> tps_status {   // issue a held-back wgrad + update on its own
    if (pend.k < 0) return TPS_OK;
    TPS_TRY(run_gemm(p, tps::GEMM_WGRAD, pend.op, pend.ga, 2, p->cs));
    TPS_TRY(finish_w(pend.k, pend.bias_side, p->cs));
    pend.k = -1;
    return TPS_OK;
  };
  for (int k = (p->graph ? -1 : nl - 1); k >= 0; --k) {
    Layer& Lk = p->layers[k];
    // the previous update of this layer must be done: it reads dW / db (rewritten below) and,
    // for V, writes the weights this backward reads
    if (Lk.has_w()) CUDA_OK(cudaStreamWaitEvent(p->cs, p->ev_upd_done[k], 0));
    const uint16_t* X = (k == 0) ? p->act[slot0][0] : p->act[slot][k];
    // fused update: the bias gradient + bias step only needs G, so it runs on the optimizer
    // stream underneath this layer's dgrad / wgrad GEMMs; the compute stream waits for it
    // (ev_bias_done) before the next layer's dgrad overwrites G's ping-pong buffer
    static const bool bias_side_on = [] {
      const char* e = std::getenv("TPS_BIAS_SIDE");
      return !(e && e[0] == '0');
    }();
    // only where the bias pass is worth hiding: for small layers the two extra cross-stream
    // events cost more latency than the pass itself (C1 lost 30 % with it)
    const bool bias_side = bias_side_on && p->fuse_update && Lk.has_w() &&
                           static_cast<int64_t>(B) * Lk.hw_out * Lk.Np >= (int64_t{1} << 20);
    if (bias_side) {
      CUDA_OK(cudaEventRecord(p->ev_bias_in, p->cs));
      CUDA_OK(cudaStreamWaitEvent(p->s_upd, p->ev_bias_in, 0));
      // own scratch: a compute-stream bias step of a narrower layer below may run concurrently
      if (Lk.bias_part)
        CUDA_OK(tps::launch_bias_from_colsum(Lk.bias_part, Lk.bias_groups, Lk.Np, Lk.db, Lk.b, Lk.mb, p->lr, p->mu,
                                             p->wd, p->s_upd));
      else
        CUDA_OK(tps::launch_bias_grad_sgd(G, B * Lk.hw_out, Lk.Np, Lk.Np, Lk.db, p->scratch_side, Lk.b, Lk.mb, p->lr,
                                          p->mu, p->wd, p->s_upd, p->tf ? 1 : 0));
      CUDA_OK(cudaEventRecord(p->split_w ? p->ev_bias_l[k] : p->ev_bias_done, p->s_upd));
      p->launches += 1;
    }
    // input gradient first: it must read this layer's weights before a fused update rewrites them
    uint16_t* dst = nullptr;
    int pidx = -1;      // which column-partial buffer goes with dst (bias gradient of layer k-1)
    if (Lk.gidx > 0) {  // the network's first layer has no input gradient
      if (k > 0 && p->split_w) {
        pidx = k % 3;
        // three rotating buffers: this dgrad overwrites the gradient that layer k+2's weight
        // gradient (stream s_w) and bias step (optimizer stream) read
        dst = p->gwork[k % 3];
        if (k + 2 < nl) {
          if (p->layers[k + 2].has_w()) CUDA_OK(cudaStreamWaitEvent(p->cs, p->ev_w_done[k + 2], 0));
          CUDA_OK(cudaStreamWaitEvent(p->cs, p->ev_bias_l[k + 2], 0));
        }
      } else if (k > 0) {
        pidx = wbuf;
        dst = p->gwork[wbuf];
        wbuf ^= 1;
      } else if (p->ipc_direct) {
        // fused compute + send: the input gradient goes straight into the previous stage's
        // receive buffer once that stage finished reading it (its backward of mb j - 2)
        TPS_TRY(flag_wait(p->cs, &p->flags[3], static_cast<uint64_t>(std::max<int64_t>(0, j - 1))));
        dst = p->prev_gin[j & 1];
      } else {
        CUDA_OK(cudaStreamWaitEvent(p->cs, p->ev_bwd_sent[j & 1], 0));  // gout of mb j-2 has left
        dst = p->gout[j & 1];
      }
      if (!dgrad_pairable(k)) TPS_TRY(flush_pending());
      if (Lk.kind == TPS_LAYER_MAXPOOL2) {
        // gradient to the first window maximum; the ReLU mask was applied by the layer above
        CUDA_OK(tps::launch_maxpool2_bwd(X, G, dst, B, Lk.H, Lk.Wd, Lk.Ci, p->cs));
        p->launches += 1;
      } else {
        const uint16_t* Ws = Lk.ver[v_used % p->R];
        const uint16_t* Wl = Lk.ver[vl % p->R];
        tps::GemmArgs ga{};
        ga.out = dst; ga.out_f32 = 0; ga.mask = X; ga.ldm = Lk.ld_in; ga.ldo = Lk.ld_in;
        ga.alpha = 1.f; ga.xa = 1.f; ga.xb = 0.f;
        const bool conv = Lk.kind == TPS_LAYER_CONV3X3;
        // concurrent with layer k+1's fused wgrad + update on s_w: take the dgrad's share of the SMs
        if (p->split_w && p->part_dgrad > 0 && k + 1 < nl && p->layers[k + 1].has_w()) ga.max_ctas = p->part_dgrad;
        ga.M = B * Lk.hw_in; ga.N = conv ? Lk.Ci : Lk.Kp; ga.K = Lk.Np;
        if (conv) ga.K = 9 * Lk.Co;
        tps::GemmOperands op{G, Lk.Np, Ws, Lk.Kp, nullptr};
        if (conv) {
          op.cv = tps::ConvGeom{B, Lk.H, Lk.Wd, Lk.Co};
          op.Cw = Lk.Ci;
        }
        // the layer below takes its bias gradient from this epilogue's column sums of G
        if (pidx >= 0 && p->bpart[pidx] && p->layers[k - 1].has_b() && p->layers[k - 1].Np == ga.N) {
          ga.colsum = p->bpart[pidx];
          p->layers[k - 1].bias_part = p->bpart[pidx];
          p->layers[k - 1].bias_groups = (ga.M + 31) / 32;
        }
        if (blend_on_load) {
          op.B2 = Wl;
          ga.xa = alpha; ga.xb = beta;
          TPS_TRY(run_gemm(p, conv ? tps::GEMM_CONV_DGRAD_BLEND : tps::GEMM_DGRAD_BLEND, op, ga, 1));
        } else {
          ga.alpha = (p->variant == TPS_I) ? alpha : 1.f;   // EQ1: α·(G·W_stash) = G·(α·W_stash)
          bool done = false;
          if (pend.k == k + 1 && dgrad_pairable(k) && !ga.colsum) {
            tps::DualArgs dg{ga.M, ga.N, ga.K, ga.alpha, ga.out, ga.ldo, ga.mask, ga.ldm};
            TPS_TRY(run_dual(p, pend.op, pend.ga, op, dg, &done));
            if (done) {
              TPS_TRY(finish_w(pend.k, pend.bias_side, p->cs));
              pend.k = -1;
            }
          }
          if (!done) {
            TPS_TRY(flush_pending());
            TPS_TRY(run_gemm(p, conv ? tps::GEMM_CONV_DGRAD : tps::GEMM_DGRAD, op, ga, 1));
          }
        }
      }
    }
    if (Lk.has_w()) {
      // weight gradient: dW[Np, Kp] = Gᵀ·X (Linear / patch layer) or conv wgrad (implicit im2col);
      // with fuse_update the epilogue applies the SGD/momentum step and writes version vn
      const int rows = B * Lk.hw_out;
      tps::GemmArgs ga{};
      ga.M = Lk.Np; ga.N = Lk.Kp; ga.K = rows; ga.out = Lk.dW; ga.ldo = Lk.Kp; ga.out_f32 = 1;
      ga.alpha = 1.f; ga.xa = 1.f;
      if (p->fuse_update && Lk.fuse) {
        ga.epi = tps::EPI_SGD;
        ga.w = Lk.W; ga.v = Lk.mW; ga.ver = Lk.ver[vn % p->R];
        ga.lr = p->lr; ga.mu = p->mu; ga.wd = p->wd;
      }
      cudaStream_t ws = p->cs;
      if (p->dp > 1) {   // the replicas must have read this layer's gradients of mb j-1 before they are rewritten
        for (int q = 0; q < p->dp; ++q)
          if (q != p->dp_rank)
            TPS_TRY(flag_wait(p->cs, &p->dp_flags[static_cast<size_t>(k) * 2 * p->dp + p->dp + q], static_cast<uint64_t>(j)));
      }
      // concurrent with layer k-1's dgrad on the compute stream: the other share of the SMs
      if (p->split_w && p->part_dgrad > 0 && k > 0 && p->layers[k - 1].gidx > 0 &&
          p->layers[k - 1].kind != TPS_LAYER_MAXPOOL2)
        ga.max_ctas = p->nsm - p->part_dgrad;
      TPS_TRY(flush_pending());   // (a held-back update of layer k+1 whose dgrad partner did not come)
      const bool defer = p->dual && p->dp == 1 && Lk.kind == TPS_LAYER_LINEAR && ga.max_ctas == 0 &&
                         Lk.fuse && dgrad_pairable(k - 1);
      if (p->split_w && !defer) {   // after this layer's dgrad (it reads the weights the fused update rewrites)
        CUDA_OK(cudaEventRecord(p->ev_dg[k], p->cs));
        CUDA_OK(cudaStreamWaitEvent(p->s_w, p->ev_dg[k], 0));
        ws = p->s_w;
      }
      if (defer) {
        pend.k = k;
        pend.op = tps::GemmOperands{G, Lk.Np, X, Lk.Kp, nullptr};
        pend.ga = ga;
        pend.bias_side = bias_side;
      } else if (Lk.kind == TPS_LAYER_CONV3X3 && !Lk.im2col) {
        tps::GemmOperands op{G, Lk.Np, X, 0, nullptr};
        op.cv = tps::ConvGeom{B, Lk.H, Lk.Wd, Lk.Ci};
        TPS_TRY(run_gemm(p, tps::GEMM_CONV_WGRAD, op, ga, 2, ws));
      } else {
        tps::GemmOperands op{G, Lk.Np, X, Lk.Kp, nullptr};
        TPS_TRY(run_gemm(p, tps::GEMM_WGRAD, op, ga, 2, ws));
      }
      if (p->fuse_update && !Lk.fuse) {   // split-K weight gradient above, its update right behind it
        const int64_t n = static_cast<int64_t>(Lk.Np) * Lk.Kp;
        CUDA_OK(tps::launch_sgd_update(Lk.W, Lk.mW, Lk.dW, Lk.ver[vn % p->R], n, p->lr, p->mu, p->wd, ws,
                                       p->upd_blocks_per_sm, p->tf ? 1 : 0));
        p->launches += 1;
      }
      if (p->split_w && !defer) CUDA_OK(cudaEventRecord(p->ev_w_done[k], p->s_w));
      if (!bias_side) {   // bias gradient and the bias's SGD/momentum step in one launch
        // (data parallel: the gradient only; the step runs on the replica average below)
        if (Lk.bias_part)
          CUDA_OK(tps::launch_bias_from_colsum(Lk.bias_part, Lk.bias_groups, Lk.Np, Lk.db, p->dp > 1 ? nullptr : Lk.b,
                                               Lk.mb, p->lr, p->mu, p->wd, p->cs));
        else
          CUDA_OK(tps::launch_bias_grad_sgd(G, rows, Lk.Np, Lk.Np, Lk.db, p->scratch, p->dp > 1 ? nullptr : Lk.b, Lk.mb,
                                            p->lr, p->mu, p->wd, p->cs, p->tf ? 1 : 0));
        p->launches += 1;
      }
      // U(j) always directly follows B(j) in the static order (reading Z7), so the update of
      // this layer is issued now: either it already ran in the wgrad epilogue (fuse_update), or
      // it runs on the optimizer stream, HBM-bound, underneath the remaining tensor-bound GEMMs
      // of this backward.  The next forward of layer k waits for ev_upd_done[k].
      cudaStream_t us = p->fuse_update ? p->cs : p->s_upd;
      if (!p->fuse_update && p->dp > 1) {
        TPS_TRY(dp_update(p, Lk, k, j, vn));
      } else if (!p->fuse_update) {
        CUDA_OK(cudaEventRecord(p->ev_grad_ready[k], p->cs));
        CUDA_OK(cudaStreamWaitEvent(us, p->ev_grad_ready[k], 0));
        const int64_t n = static_cast<int64_t>(Lk.Np) * Lk.Kp;
        TimedLaunch tl{};
        TPS_TRY(time_begin(p, &tl, 4, (p->mu != 0.f ? 22.0 : 14.0) * n, us));
        CUDA_OK(tps::launch_sgd_update(Lk.W, Lk.mW, Lk.dW, Lk.ver[vn % p->R], n, p->lr, p->mu, p->wd, us,
                                       p->upd_blocks_per_sm, p->tf ? 1 : 0));
        TPS_TRY(time_end(p, &tl, us));
        p->launches += 1;
      }
      if (defer) {
        // events follow the shared launch (finish_w) or flush_pending
      } else if (p->split_w) {
        // parameters final once the fused wgrad+update (s_w) and the bias step are done
        if (bias_side) {
          CUDA_OK(cudaStreamWaitEvent(p->s_upd, p->ev_w_done[k], 0));
          CUDA_OK(cudaEventRecord(p->ev_upd_done[k], p->s_upd));
        } else {
          CUDA_OK(cudaEventRecord(p->ev_bias_l[k], p->cs));   // bias ran on the compute stream
          CUDA_OK(cudaEventRecord(p->ev_upd_done[k], p->s_w));
        }
      } else if (bias_side) {
        // layer k's parameters are final once both the fused wgrad+update (compute stream) and
        // the bias step (optimizer stream) are done; G may be overwritten once the bias read it
        CUDA_OK(cudaEventRecord(p->ev_grad_ready[k], p->cs));
        CUDA_OK(cudaStreamWaitEvent(p->s_upd, p->ev_grad_ready[k], 0));
        CUDA_OK(cudaEventRecord(p->ev_upd_done[k], p->s_upd));
        CUDA_OK(cudaStreamWaitEvent(p->cs, p->ev_bias_done, 0));
      } else {
        CUDA_OK(cudaEventRecord(p->ev_upd_done[k], us));
      }
    }
    if (dst) G = dst;
  }
  TPS_TRY(flush_pending());
  if (p->split_w) {
    // the weight gradients read this mini-batch's stashed activations and the gradients: join
    for (int k = 0; k < nl; ++k) {
      if (p->layers[k].has_w()) {
        CUDA_OK(cudaStreamWaitEvent(p->cs, p->ev_w_done[k], 0));
        CUDA_OK(cudaStreamWaitEvent(p->cs, p->ev_upd_done[k], 0));
      }
    }
  }
  // the input slot and the received gradient buffer may now be refilled
  CUDA_OK(cudaEventRecord(p->ev_act_free[slot0], p->cs));
  if (!p->last) CUDA_OK(cudaEventRecord(p->ev_gin_free[j & 1], p->cs));
  if (p->transport == TPS_TRANSPORT_IPC) {   // tell the neighbours that write into them
    if (!p->first) TPS_TRY(flag_write(p->cs, &p->prev_flags[2], static_cast<uint64_t>(j) + 1));
    if (!p->last) TPS_TRY(flag_write(p->cs, &p->next_flags[3], static_cast<uint64_t>(j) + 1));
  }
  if (!p->first) {
    TPS_TRY(send_bwd(p, j, p->gout[j & 1], static_cast<size_t>(p->B) * p->in0_elems * p->esz));
  }
  tps_event e{};
  e.stage = p->s; e.kind = TPS_EV_B; e.micro = -1; e.mb = j;
  e.v_used = v_used; e.v_latest = vl; e.delta = static_cast<int32_t>(delta); e.alpha = alpha; e.beta = beta;
  p->trace.push_back(e);
  p->fwd_version.erase(j);
  p->fwd_groups_done.erase(j);
  p->pending_update = j;
  advance(p);
  return TPS_OK;
}

tps_status do_update(tps_pipeline* p, int64_t j) {
  TPS_TRY(expect(p, TPS_EV_U, j, -1, 0));
  if (p->pending_update != j) return fail(TPS_E_ORDER, "update of mb %lld without its backward", (long long)j);
  const int64_t vn = p->latest + 1;
  // the parameter update of mb j was issued by its backward (see do_backward); this event
  // commits the new version vn (ring slot vn mod R) as the stage's latest
  tps_event e{};
  e.stage = p->s; e.kind = TPS_EV_U; e.micro = -1; e.mb = j;
  e.v_used = p->latest; e.v_latest = vn; e.alpha = 1.f;
  p->trace.push_back(e);
  p->latest = vn;
  p->pending_update = -1;
  update_stash_peak(p);
  advance(p);
  return TPS_OK;
}

tps_status begin_run(tps_pipeline* p, int64_t first, int64_t n) {
  if (n <= 0 || first < 0) return fail(TPS_E_INVALID_ARG, "bad run [%lld, +%lld)", (long long)first, (long long)n);
  if (p->in_run) return fail(TPS_E_ORDER, "stage %d: previous run not finished", p->s);
  if (p->transport == TPS_TRANSPORT_IPC && !p->ipc_connected)
    return fail(TPS_E_STATE, "IPC transport: tps_ipc_connect first");
  if (p->dp > 1 && !p->dp_connected) return fail(TPS_E_STATE, "data parallelism: tps_dp_connect first");
  if (p->transport == TPS_TRANSPORT_IPC || p->dp > 1) {
    // flag words carry mini-batch numbers: runs continue the numbering from 0
    if (first != p->ipc_next_mb)
      return fail(TPS_E_ORDER, "IPC / data-parallel handle: runs number mini-batches contiguously (expected first %lld)",
                  (long long)p->ipc_next_mb);
    p->ipc_next_mb = first + n;
  }
  // inputs of the run (device pools, labels) may have been produced on the caller's stream:
  // the handle's streams start after everything already submitted there (the configured
  // compute stream, else the legacy default stream)
  CUDA_OK(cudaEventRecord(p->ev_caller, p->caller));
  for (cudaStream_t st : {p->cs, p->s_fin, p->s_upd}) CUDA_OK(cudaStreamWaitEvent(st, p->ev_caller, 0));
  if (p->s_w) CUDA_OK(cudaStreamWaitEvent(p->s_w, p->ev_caller, 0));
  build_order(p->Kmax, p->s, p->m, p->g, first, n, &p->order);
  p->pos = 0;
  p->run_first = first;
  p->run_n = n;
  p->in_run = true;
  return TPS_OK;
}

// Timeline / NVTX bracket of one schedule event on the compute stream (off: one branch).
tps_status tl_take(tps_pipeline* p, cudaEvent_t* e) {
  if (p->ev_pool.empty()) {
    for (int i = 0; i < 64; ++i) {
      cudaEvent_t ev;
      CUDA_OK(cudaEventCreate(&ev));
      p->ev_pool.push_back(ev);
    }
  }
  *e = p->ev_pool.back();
  p->ev_pool.pop_back();
  return TPS_OK;
}

template <class F>
tps_status bracket(tps_pipeline* p, int kind, int64_t mb, F&& body) {
  if (!p->timeline && !p->nvtx) return body();
  if (p->nvtx) {
    char name[64];
    std::snprintf(name, sizeof(name), "s%d %c mb%lld", p->s, "FBU"[kind], static_cast<long long>(mb));
    nvtxRangePushA(name);
  }
  cudaEvent_t a = nullptr, b = nullptr;
  if (p->timeline) {
    TPS_TRY(tl_take(p, &a));
    CUDA_OK(cudaEventRecord(a, p->cs));
  }
  const size_t n0 = p->trace.size();
  const tps_status st = body();
  if (p->nvtx) nvtxRangePop();
  if (p->timeline) {
    if (st != TPS_OK || p->trace.size() != n0 + 1) {
      p->ev_pool.push_back(a);
      return st;
    }
    TPS_TRY(tl_take(p, &b));
    CUDA_OK(cudaEventRecord(b, p->cs));
    p->tl_pending.push_back({p->trace.back(), a, b});
  }
  return st;
}

tps_status drain_timeline(tps_pipeline* p) {
  if (p->tl_pending.empty()) return TPS_OK;
  CUDA_OK(cudaEventSynchronize(p->tl_pending.back().b));
  for (auto& t : p->tl_pending) {
    tps_timeline_rec r{};
    r.ev = t.e;
    float a = 0.f, b = 0.f;
    CUDA_OK(cudaEventElapsedTime(&a, p->tl_origin, t.a));
    CUDA_OK(cudaEventElapsedTime(&b, p->tl_origin, t.b));
    r.t0_ms = a;
    r.t1_ms = b;
    p->tl_done.push_back(r);
    p->ev_pool.push_back(t.a);
    p->ev_pool.push_back(t.b);
  }
  p->tl_pending.clear();
  return TPS_OK;
}

tps_status fire(tps_pipeline* p, const tps_event& e, const void* x_pool, const int32_t* y_pool, int pool) {
  if (e.kind == TPS_EV_F) {
    const int64_t slot = e.mb % pool;
    const void* x = nullptr;
    const int32_t* y = nullptr;
    // replica r of mini-batch j reads rows [r·B, (r+1)·B) of pool entry j % pool
    const int64_t row = (slot * p->dp + p->dp_rank) * p->B + static_cast<int64_t>(e.micro) * p->bsz;
    if (p->first) x = static_cast<const uint16_t*>(x_pool) + row * p->dims[0] * p->ew;
    if (p->last) y = y_pool + row;
    return bracket(p, TPS_EV_F, e.mb, [&] { return do_forward(p, e.mb, e.micro, e.micro_count, x, y); });
  }
  if (e.kind == TPS_EV_B) return bracket(p, TPS_EV_B, e.mb, [&] { return do_backward(p, e.mb, -1); });
  return bracket(p, TPS_EV_U, e.mb, [&] { return do_update(p, e.mb); });
}

}  // namespace

// ======================================================================== C ABI
extern "C" {

int32_t tps_abi_version(void) { return TPS_ABI_VERSION; }
const char* tps_last_error(void) { return g_err.c_str(); }

tps_status tps_nccl_unique_id(void* out128) {
  if (!out128) return fail(TPS_E_INVALID_ARG, "null out");
  ncclUniqueId id;
  NCCL_OK(ncclGetUniqueId(&id));
  std::memcpy(out128, &id, sizeof(id));
  return TPS_OK;
}

tps_status tps_blend_coeffs(int32_t variant, int32_t blend, int32_t staleness, double lambda, float* alpha, float* beta) {
  if (!alpha || !beta) return fail(TPS_E_INVALID_ARG, "null out");
  if (staleness < 0) return fail(TPS_E_INVALID_ARG, "staleness must be >= 0 (P:211)");
  if (variant != TPS_V && variant != TPS_I) return fail(TPS_E_INVALID_ARG, "bad variant");
  if (variant == TPS_I && !(lambda > 0)) return fail(TPS_E_CONFIG, "lambda must be > 0 (P:227)");
  if (blend != TPS_BLEND_EQ1 && blend != TPS_BLEND_CONVEX) return fail(TPS_E_INVALID_ARG, "bad blend");
  compute_coeffs(variant, blend, staleness, lambda, alpha, beta);
  return TPS_OK;
}

tps_status tps_schedule_events(int32_t S, int32_t s, int32_t m, int32_t fwd_group, int64_t M, tps_event* out,
                               int64_t cap, int64_t* n) {
  if (S < 1 || s < 0 || s >= S || m < 1 || M < 0 || !n) return fail(TPS_E_INVALID_ARG, "bad schedule arguments");
  const int g = fwd_group <= 0 ? m : fwd_group;
  if (m % g) return fail(TPS_E_CONFIG, "fwd_group must divide m");
  std::vector<tps_event> ev;
  if (M > 0) build_order(S - s, s, m, g, 0, M, &ev);
  *n = static_cast<int64_t>(ev.size());
  if (out) std::memcpy(out, ev.data(), sizeof(tps_event) * static_cast<size_t>(std::min<int64_t>(cap, *n)));
  return TPS_OK;
}

// image-net layer list: kinds, shapes and chaining (include/tps.h, tps_layer)
tps_status validate_specs(const tps_config* c) {
  if (c->num_layer_specs != c->num_layers || !c->layer_specs) return fail(TPS_E_CONFIG, "need num_layers layer specs");
  int64_t prev_feat = -1;
  int ph = 0, pw = 0, pc = 0;   // spatial output of the previous conv/pool layer
  for (int l = 0; l < c->num_layers; ++l) {
    const tps_layer& sp = c->layer_specs[l];
    if (sp.kind == TPS_LAYER_LINEAR) {
      if (sp.in_c < 1 || sp.out_c < 1) return fail(TPS_E_CONFIG, "layer %d: bad linear dims", l);
      if (pc != 0 && sp.in_c % 16) return fail(TPS_E_CONFIG, "layer %d: flattened conv output must be a multiple of 16", l);
      if (prev_feat >= 0 && sp.in_c != prev_feat) return fail(TPS_E_CONFIG, "layer %d: in %d != %lld", l, sp.in_c, (long long)prev_feat);
      prev_feat = sp.out_c;
      ph = pw = pc = 0;
    } else if (sp.kind == TPS_LAYER_CONV3X3 || sp.kind == TPS_LAYER_MAXPOOL2) {
      if (sp.in_h < 1 || sp.in_w < 1 || sp.in_c < 1) return fail(TPS_E_CONFIG, "layer %d: bad shape", l);
      if (l > 0 && (pc == 0 || sp.in_h != ph || sp.in_w != pw || sp.in_c != pc))
        return fail(TPS_E_CONFIG, "layer %d: input %dx%dx%d does not match the previous output", l, sp.in_h, sp.in_w, sp.in_c);
      if (sp.kind == TPS_LAYER_CONV3X3) {
        if (sp.out_c % 64) return fail(TPS_E_CONFIG, "layer %d: conv out_c must be a multiple of 64", l);
        if (l > 0 && sp.in_c % 64) return fail(TPS_E_CONFIG, "layer %d: conv in_c must be a multiple of 64", l);
        ph = sp.in_h; pw = sp.in_w; pc = sp.out_c;
      } else {
        if (sp.in_h % 2 || sp.in_w % 2 || sp.in_c % 8) return fail(TPS_E_CONFIG, "layer %d: pool needs even H, W and C %% 8", l);
        ph = sp.in_h / 2; pw = sp.in_w / 2; pc = sp.in_c;
      }
      prev_feat = static_cast<int64_t>(ph) * pw * pc;
    } else {
      return fail(TPS_E_CONFIG, "layer %d: unknown kind %d", l, sp.kind);
    }
  }
  if (c->layer_specs[c->num_layers - 1].kind != TPS_LAYER_LINEAR) return fail(TPS_E_CONFIG, "the last layer must be Linear");
  return TPS_OK;
}

bool is_graph_kind(int k) {
  return k == TPS_LAYER_CONV || k == TPS_LAYER_BN || k == TPS_LAYER_MAXPOOL3 || k == TPS_LAYER_AVGPOOL;
}

struct GShape {
  int h = 0, w = 0, c = 0;   // flat tensors: h = w = 1
  int64_t elems() const { return static_cast<int64_t>(h) * w * c; }
  bool operator==(const GShape& o) const { return h == o.h && w == o.w && c == o.c; }
};

// output shape of every layer of a graph network (validated); shapes[l + 1] = output of layer l,
// shapes[0] = the network input
tps_status graph_shapes(const tps_config* c, std::vector<GShape>* shapes) {
  const int L = c->num_layers;
  shapes->assign(L + 1, GShape{});
  const tps_layer& s0 = c->layer_specs[0];
  (*shapes)[0] = GShape{s0.in_h, s0.in_w, s0.in_c};
  if ((*shapes)[0].elems() != c->dims[0]) return fail(TPS_E_CONFIG, "dims[0] must equal H·W·C of layer 0's input");
  for (int l = 0; l < L; ++l) {
    const tps_layer& sp = c->layer_specs[l];
    if (!is_graph_kind(sp.kind) && sp.kind != TPS_LAYER_LINEAR)
      return fail(TPS_E_CONFIG, "layer %d: kind %d cannot be mixed with graph layers", l, sp.kind);
    const int src = l - std::max(1, sp.src_back);
    if (src < -1) return fail(TPS_E_CONFIG, "layer %d: src_back %d reaches before the input", l, sp.src_back);
    const GShape in = (*shapes)[src + 1];
    GShape o;
    if (sp.kind == TPS_LAYER_LINEAR) {
      if (l != L - 1) return fail(TPS_E_CONFIG, "layer %d: in a graph network LINEAR is the last layer (the head)", l);
      if (in.h != 1 || in.w != 1 || in.c != sp.in_c) return fail(TPS_E_CONFIG, "layer %d: head input must be a flat %d-vector", l, sp.in_c);
      if (sp.in_c % 16 || sp.out_c < 1) return fail(TPS_E_CONFIG, "layer %d: head needs in_c %% 16 == 0", l);
      o = GShape{1, 1, sp.out_c};
    } else {
      if (!(in == GShape{sp.in_h, sp.in_w, sp.in_c}))
        return fail(TPS_E_CONFIG, "layer %d: input %dx%dx%d does not match its source (layer %d: %dx%dx%d)", l, sp.in_h,
                    sp.in_w, sp.in_c, src, in.h, in.w, in.c);
      if (sp.kind == TPS_LAYER_CONV) {
        if (sp.k < 1 || sp.stride < 1 || sp.pad < 0) return fail(TPS_E_CONFIG, "layer %d: bad conv k/stride/pad", l);
        const int ho = (sp.in_h + 2 * sp.pad - sp.k) / sp.stride + 1, wo = (sp.in_w + 2 * sp.pad - sp.k) / sp.stride + 1;
        if (ho < 1 || wo < 1) return fail(TPS_E_CONFIG, "layer %d: empty conv output", l);
        if (sp.out_c % 16) return fail(TPS_E_CONFIG, "layer %d: conv out_c must be a multiple of 16", l);
        o = GShape{ho, wo, sp.out_c};
      } else if (sp.kind == TPS_LAYER_BN) {
        o = in;
        if (sp.res_back > 0) {
          const int r = l - sp.res_back;
          if (r < -1) return fail(TPS_E_CONFIG, "layer %d: res_back %d reaches before the input", l, sp.res_back);
          if (!((*shapes)[r + 1] == o)) return fail(TPS_E_CONFIG, "layer %d: residual shape mismatch", l);
        }
      } else if (sp.kind == TPS_LAYER_MAXPOOL3) {
        o = GShape{(sp.in_h - 1) / 2 + 1, (sp.in_w - 1) / 2 + 1, sp.in_c};
      } else {
        o = GShape{1, 1, sp.in_c};
      }
    }
    (*shapes)[l + 1] = o;
  }
  if (c->layer_specs[L - 1].kind != TPS_LAYER_LINEAR) return fail(TPS_E_CONFIG, "the last layer must be the Linear head");
  // a stage reads only its own layers and the previous stage's last output
  for (int s = 0; s < c->num_stages; ++s)
    for (int l = c->stage_bounds[s]; l < c->stage_bounds[s + 1]; ++l) {
      const tps_layer& sp = c->layer_specs[l];
      const int src = l - std::max(1, sp.src_back);
      const int r = (sp.kind == TPS_LAYER_BN && sp.res_back > 0) ? l - sp.res_back : c->stage_bounds[s];
      if (src < c->stage_bounds[s] - 1 || r < c->stage_bounds[s] - 1)
        return fail(TPS_E_CONFIG, "layer %d (stage %d) reads a tensor of an earlier stage other than its input", l, s);
    }
  return TPS_OK;
}

tps_status init_graph(tps_pipeline* p, const tps_config* c, int lb, int le) {
  std::vector<GShape> sh;
  TPS_TRY(graph_shapes(c, &sh));
  p->fuse_update = false;   // graph networks update on the optimizer stream
  int64_t max_elems = sh[lb].elems();
  int64_t patch_elems = 0, dpatch_elems = 0, bn_doubles = 0, bias_scr = 0;
  for (int l = lb; l < le; ++l) {
    const tps_layer& sp = c->layer_specs[l];
    const GShape in = sh[l - std::max(1, sp.src_back) + 1], o = sh[l + 1];
    Layer L;
    L.gidx = l;
    L.kind = sp.kind;
    L.src = l - std::max(1, sp.src_back) - lb;
    L.res = (sp.kind == TPS_LAYER_BN && sp.res_back > 0) ? l - sp.res_back - lb : -2;
    L.relu = sp.kind == TPS_LAYER_BN && sp.relu != 0;
    L.H = in.h; L.Wd = in.w; L.Ci = in.c; L.Co = o.c; L.Ho = o.h; L.Wo = o.w;
    L.hw_in = in.h * in.w; L.ld_in = in.c; L.hw_out = o.h * o.w; L.ld_out = o.c;
    if (sp.kind == TPS_LAYER_CONV) {
      L.k = sp.k; L.st = sp.stride; L.pad = sp.pad;
      L.in = sp.k * sp.k * L.Ci; L.out = L.Co; L.Np = L.Co;
      if (L.k == 1 && L.st == 1 && L.pad == 0 && L.Ci % 16 == 0) {
        L.conv_mode = 0; L.Kp = L.Ci;
      } else if (L.k == 3 && L.st == 1 && L.pad == 1 && L.Ci % 64 == 0 && L.Co % 64 == 0) {
        L.conv_mode = 1; L.Kp = 9 * L.Ci;     // implicit GEMM: TMA im2col-mode loads, all three GEMMs
      } else if (L.Ci % 64 == 0 && L.Co % 64 == 0) {
        // strided conv: implicit forward / weight gradient; the input gradient of a strided conv
        // is a patch-gradient GEMM + col2im
        L.conv_mode = 3; L.Kp = L.k * L.k * L.Ci;
        if (!(p->first && L.src == -1))
          dpatch_elems = std::max(dpatch_elems, static_cast<int64_t>(p->B) * L.hw_out * L.Kp);
      } else {
        L.conv_mode = 2; L.Kp = pad16(L.in);
        const int64_t pe = static_cast<int64_t>(p->B) * L.hw_out * L.Kp;
        patch_elems = std::max(patch_elems, pe);
        if (!(p->first && L.src == -1)) dpatch_elems = std::max(dpatch_elems, pe);
      }
    } else if (sp.kind == TPS_LAYER_BN) {
      L.in = 1; L.out = L.Ci; L.Kp = 1; L.Np = L.Ci;
      bn_doubles = std::max(bn_doubles, tps::bn_scratch_doubles(p->m, p->bsz * L.hw_in, L.Ci));
    } else if (sp.kind == TPS_LAYER_LINEAR) {
      L.in = sp.in_c; L.out = sp.out_c; L.Kp = pad16(L.in); L.Np = pad16(L.out);
      L.ld_in = L.Kp; L.ld_out = L.Np;
      bias_scr = std::max(bias_scr, tps::bias_grad_scratch_floats(p->B, L.Np));
    } else if (sp.kind == TPS_LAYER_MAXPOOL3 && L.Ci % 8 == 0) {
      L.argmax.resize(p->Kmax);
      for (int r = 0; r < p->Kmax; ++r)
        TPS_TRY(alloc_t(p, &L.argmax[r], static_cast<size_t>(p->B) * L.out_elems(), &p->mem_acts));
    }
    max_elems = std::max({max_elems, L.in_elems(), L.out_elems()});
    if (L.has_w()) {
      const size_t n = static_cast<size_t>(L.Np) * L.Kp;
      TPS_TRY(alloc_t(p, &L.W, n, &p->mem_weights));
      if (L.has_b()) TPS_TRY(alloc_t(p, &L.b, L.Np, &p->mem_weights));
      if (p->mu != 0.f) {
        TPS_TRY(alloc_t(p, &L.mW, n, &p->mem_optim));
        if (L.has_b()) TPS_TRY(alloc_t(p, &L.mb, L.Np, &p->mem_optim));
      }
      TPS_TRY(alloc_t(p, &L.dW, n, &p->mem_optim));
      if (L.has_b()) TPS_TRY(alloc_t(p, &L.db, L.Np, &p->mem_optim));
      if (L.kind == TPS_LAYER_BN) {
        L.verf.resize(p->R);
        for (int r = 0; r < p->R; ++r) TPS_TRY(alloc_t(p, &L.verf[r], n, r == 0 ? &p->mem_weights : &p->mem_stash));
        p->ver_bytes += static_cast<int64_t>(n) * 4;
        L.mean.resize(p->Kmax);
        L.invstd.resize(p->Kmax);
        for (int r = 0; r < p->Kmax; ++r) {
          TPS_TRY(alloc_t(p, &L.mean[r], static_cast<size_t>(p->m) * L.Ci, &p->mem_acts));
          TPS_TRY(alloc_t(p, &L.invstd[r], static_cast<size_t>(p->m) * L.Ci, &p->mem_acts));
        }
        if (L.relu && L.Ci % 8 == 0 && !no_relu_mask()) {
          L.relu_mask.resize(p->Kmax);
          for (int r = 0; r < p->Kmax; ++r)
            TPS_TRY(alloc_t(p, &L.relu_mask[r], static_cast<size_t>(p->B) * L.hw_in * (L.Ci / 8), &p->mem_acts));
        }
      } else {
        L.ver.resize(p->R);
        for (int r = 0; r < p->R; ++r) TPS_TRY(alloc_t(p, &L.ver[r], n, r == 0 ? &p->mem_weights : &p->mem_stash));
        p->ver_bytes += static_cast<int64_t>(n) * 2;
      }
    }
    p->layers.push_back(L);
  }
  const int nl = p->nlayers();
  {
    // conv -> BN pairs where the conv's epilogue provides the BN statistics (the BN reads the
    // conv output directly and right after it; 32-row groups must not straddle micro-batches).
    // Off by default (TPS_COLSUM=1 enables): ResNet-50 7.25k vs 7.47k samples/s with it -- its
    // convolutions with small K are epilogue-bound, so the extra reduction is not free
    const char* e = std::getenv("TPS_COLSUM");
    const bool on = e && e[0] == '1';
    int64_t cf = 0;
    for (int k = 0; k + 1 < nl && on; ++k) {
      Layer& L = p->layers[k];
      const Layer& N = p->layers[k + 1];
      if (L.kind == TPS_LAYER_CONV && N.kind == TPS_LAYER_BN && N.src == k && (p->bsz * L.hw_out) % 32 == 0 &&
          L.Co % 8 == 0) {
        L.stats_to_next = true;
        const int64_t rows = static_cast<int64_t>(p->g) * p->bsz * L.hw_out;
        cf = std::max(cf, 2 * ((rows + 31) / 32) * L.Co);
      }
    }
    if (cf > 0) TPS_TRY(alloc_t(p, &p->bn_colsum, static_cast<size_t>(cf), &p->mem_acts));
  }
  p->in0_elems = sh[lb].elems();
  p->act.assign(std::max(p->A0, p->Kmax), std::vector<uint16_t*>(nl + 1, nullptr));
  for (int slot = 0; slot < static_cast<int>(p->act.size()); ++slot) {
    if (slot < p->A0) TPS_TRY(alloc_t(p, &p->act[slot][0], static_cast<size_t>(p->B) * p->in0_elems, &p->mem_acts));
    if (slot >= p->Kmax) continue;
    for (int k = 0; k < nl; ++k)
      if (k < nl - 1 || !p->last)
        TPS_TRY(alloc_t(p, &p->act[slot][k + 1], static_cast<size_t>(p->B) * p->layers[k].out_elems(), &p->mem_acts));
  }
  p->gbuf.assign(nl, nullptr);
  for (int k = 0; k + 1 < nl; ++k)
    TPS_TRY(alloc_t(p, &p->gbuf[k], static_cast<size_t>(p->B) * p->layers[k].out_elems(), &p->mem_acts));
  for (int i = 0; i < 2; ++i) TPS_TRY(alloc_t(p, &p->gtmp[i], static_cast<size_t>(p->B) * max_elems, &p->mem_acts));
  TPS_TRY(alloc_t(p, &p->patches, patch_elems, &p->mem_acts));
  TPS_TRY(alloc_t(p, &p->dpatches, dpatch_elems, &p->mem_acts));
  TPS_TRY(alloc_t(p, &p->bn_scr, bn_doubles, &p->mem_acts));
  const int64_t outL = p->layers[nl - 1].out_elems();
  for (int i = 0; i < 2; ++i) {
    if (!p->last) TPS_TRY(alloc_t(p, &p->gin[i], static_cast<size_t>(p->B) * outL, &p->mem_comm));
    if (!p->first) TPS_TRY(alloc_t(p, &p->gout[i], static_cast<size_t>(p->B) * p->in0_elems, &p->mem_comm));
  }
  if (p->last) {
    TPS_TRY(alloc_t(p, &p->logits, static_cast<size_t>(p->B) * outL, &p->mem_acts));
    TPS_TRY(alloc_t(p, &p->gce, static_cast<size_t>(p->Kmax) * p->B * outL, &p->mem_acts));
    TPS_TRY(alloc_t(p, &p->loss_rows, p->B, &p->mem_acts));
    TPS_TRY(alloc_t(p, &p->labels_dev, p->B, &p->mem_acts));
    p->loss_cap = 1 << 20;
    TPS_TRY(alloc_t(p, &p->losses, p->loss_cap, &p->mem_acts));
    TPS_TRY(alloc_t(p, &p->loss_ctr, 1, &p->mem_acts));
  }
  TPS_TRY(alloc_t(p, &p->scratch, bias_scr, &p->mem_optim));
  return TPS_OK;
}

tps_status tps_pipeline_init(const tps_config* c, tps_pipeline** out) {
  if (!c || !out) return fail(TPS_E_INVALID_ARG, "null argument");
  *out = nullptr;
  if (c->num_layers < 1 || !c->dims || !c->stage_bounds) return fail(TPS_E_CONFIG, "need >= 1 layer, dims and stage_bounds");
  if (c->num_stages < 1) return fail(TPS_E_CONFIG, "num_stages must be >= 1");
  if (c->stage_id < 0 || c->stage_id >= c->num_stages) return fail(TPS_E_CONFIG, "stage_id out of range");
  if (c->micro_batches < 1 || c->micro_batch_size < 1) return fail(TPS_E_CONFIG, "m and b must be >= 1");
  if (c->max_inflight < 0 || (c->max_inflight > 0 && c->max_inflight != c->num_stages - c->stage_id && c->num_stages != 1))
    return fail(TPS_E_CONFIG, "max_inflight other than S - s needs S = 1");
  if (c->staleness_mode != 0 && c->staleness_mode != 1) return fail(TPS_E_CONFIG, "bad staleness_mode");
  if ((c->dev_alloc == nullptr) != (c->dev_free == nullptr)) return fail(TPS_E_CONFIG, "dev_alloc and dev_free go together");
  if (c->dp_size < 0 || c->dp_size > 8 || (c->dp_size > 1 && (c->dp_rank < 0 || c->dp_rank >= c->dp_size)))
    return fail(TPS_E_CONFIG, "need 1 <= dp_size <= 8 and 0 <= dp_rank < dp_size");
  if (c->dp_size > 1 && c->num_stages > 1 && c->transport != TPS_TRANSPORT_IPC)
    return fail(TPS_E_CONFIG, "data parallelism runs one process per stage replica (IPC transport)");
  if (c->variant != TPS_V && c->variant != TPS_I) return fail(TPS_E_CONFIG, "bad variant");
  if (c->blend != TPS_BLEND_EQ1 && c->blend != TPS_BLEND_CONVEX) return fail(TPS_E_CONFIG, "bad blend");
  if (c->variant == TPS_I && !(c->lambda > 0)) return fail(TPS_E_CONFIG, "lambda must be > 0 (P:227)");
  bool graph = false;
  if (c->num_layer_specs > 0) {
    if (c->num_layer_specs != c->num_layers || !c->layer_specs) return fail(TPS_E_CONFIG, "need num_layers layer specs");
    for (int l = 0; l < c->num_layers; ++l) graph = graph || is_graph_kind(c->layer_specs[l].kind);
    if (!graph) TPS_TRY(validate_specs(c));
  } else {
    for (int l = 0; l <= c->num_layers; ++l)
      if (c->dims[l] < 1) return fail(TPS_E_CONFIG, "dims[%d] < 1", l);
  }
  if (c->stage_bounds[0] != 0 || c->stage_bounds[c->num_stages] != c->num_layers)
    return fail(TPS_E_CONFIG, "stage_bounds must start at 0 and end at num_layers");
  for (int s = 0; s < c->num_stages; ++s)
    if (c->stage_bounds[s + 1] <= c->stage_bounds[s]) return fail(TPS_E_CONFIG, "stage %d owns no layer", s);
  if (graph) {
    std::vector<GShape> sh;
    TPS_TRY(graph_shapes(c, &sh));
  }
  const int g = c->fwd_group <= 0 ? c->micro_batches : c->fwd_group;
  if (c->micro_batches % g) return fail(TPS_E_CONFIG, "fwd_group must divide micro_batches");
  if (c->transport < TPS_TRANSPORT_NONE || c->transport > TPS_TRANSPORT_IPC) return fail(TPS_E_CONFIG, "bad transport");
  if (c->num_stages > 1 && c->transport == TPS_TRANSPORT_NONE) return fail(TPS_E_CONFIG, "S > 1 needs a transport");
  if (c->transport == TPS_TRANSPORT_NCCL && c->num_stages > 1 && !c->nccl_ids) return fail(TPS_E_CONFIG, "NCCL transport needs ids");
  if (c->dtype != TPS_BF16 && c->dtype != TPS_TF32) return fail(TPS_E_CONFIG, "bad dtype %d", c->dtype);
  if (c->dtype == TPS_TF32 && (c->num_layer_specs > 0 || c->dp_size > 1))
    return fail(TPS_E_UNSUPPORTED, "tf32 storage is implemented for chain MLP networks (dims, no layer specs, dp_size 1)");
  TPS_TRY(check_arch(c->device));
  CUDA_OK(cudaSetDevice(c->device));

  tps_pipeline* p = new tps_pipeline();
  p->S = c->num_stages; p->s = c->stage_id; p->m = c->micro_batches; p->bsz = c->micro_batch_size;
  p->B = p->m * p->bsz; p->g = g; p->ng = p->m / g;
  p->variant = c->variant; p->blend = c->blend; p->lambda = c->lambda;
  p->lr = c->lr; p->mu = c->momentum; p->wd = c->weight_decay;
  p->transport = c->num_stages == 1 ? TPS_TRANSPORT_NONE : c->transport;
  p->device = c->device; p->seed = c->seed;
  p->first = p->s == 0; p->last = p->s == p->S - 1;
  p->dims.assign(c->dims, c->dims + c->num_layers + 1);
  p->classes = c->num_layer_specs > 0 ? c->layer_specs[c->num_layers - 1].out_c : c->dims[c->num_layers];
  p->Kmax = p->S - p->s;                         // in-flight mini-batches (reading Z6)
  if (c->max_inflight > 0) p->Kmax = c->max_inflight;
  p->staleness_mode = c->staleness_mode;
  p->alloc_fn = c->dev_alloc; p->free_fn = c->dev_free; p->alloc_ctx = c->alloc_ctx;
  if (p->transport == TPS_TRANSPORT_IPC || p->dp > 1) {
    // exported buffers must be whole cudaMalloc allocations (IPC handles name allocations)
    p->alloc_fn = nullptr; p->free_fn = nullptr;
  }
  // negative control of the parity tests (debug only): TPS_FAULT=skip_update makes every
  // parameter step a no-op (lr = 0), which the parity tests must detect
  if (const char* f = std::getenv("TPS_FAULT"); f && std::strcmp(f, "skip_update") == 0) p->lr = 0.f;
  p->R = (p->variant == TPS_I) ? p->Kmax : 1;    // weight version ring
  p->A0 = p->Kmax + (c->extra_recv_slot ? 1 : 0);
  const char* env = std::getenv("TPS_EQ1_ON_LOAD");
  p->eq1_on_load = env && env[0] == '1';
  p->fuse_update = c->fuse_update != 0;
  p->graph = graph;
  p->tf = c->dtype == TPS_TF32;
  p->ew = p->tf ? 2 : 1;
  p->esz = 2 * p->ew;
  p->dp = std::max(1, c->dp_size);
  p->dp_rank = p->dp > 1 ? c->dp_rank : 0;
  if (p->dp > 1) {
    if (graph) {
      delete p;
      return fail(TPS_E_UNSUPPORTED, "data parallelism is implemented for chain networks");
    }
    p->fuse_update = false;   // the update needs the replica average: separate fused reduce + SGD kernel
  }
  if (const char* e2 = std::getenv("TPS_UPD_BPS")) p->upd_blocks_per_sm = std::max(1, std::atoi(e2));

  auto cleanup = [&](tps_status st) {
    tps_pipeline_destroy(p);
    return st;
  };
  size_t free0 = 0, total0 = 0;
  cudaDeviceSynchronize();
  cudaMemGetInfo(&free0, &total0);
  const int lb = c->stage_bounds[p->s], le = c->stage_bounds[p->s + 1];
  if (p->graph) {
    const tps_status gs = init_graph(p, c, lb, le);
    if (gs != TPS_OK) return cleanup(gs);
  } else {
  int64_t max_elems = 0;
  for (int l = lb; l < le; ++l) {
    Layer L;
    L.gidx = l;
    if (c->num_layer_specs > 0) {
      const tps_layer& sp = c->layer_specs[l];
      L.kind = sp.kind;
      if (sp.kind == TPS_LAYER_LINEAR) {
        L.in = sp.in_c; L.out = sp.out_c; L.Kp = pad16(L.in); L.Np = pad16(L.out);
        L.ld_in = L.Kp; L.ld_out = L.Np;
      } else {
        L.H = sp.in_h; L.Wd = sp.in_w; L.Ci = sp.in_c;
        L.hw_in = L.H * L.Wd; L.ld_in = L.Ci;
        if (sp.kind == TPS_LAYER_CONV3X3) {
          L.Co = sp.out_c;
          L.in = 9 * L.Ci; L.out = L.Co; L.Np = L.Co;
          L.im2col = (L.Ci % 64) != 0;
          L.Kp = L.im2col ? pad16(L.in) : L.in;
          L.hw_out = L.hw_in; L.ld_out = L.Co;
          if (L.im2col) L.ld_in = L.Kp;            // the stash holds the patches
        } else {
          L.Co = L.Ci;
          L.hw_out = L.hw_in / 4; L.ld_out = L.Ci;
        }
      }
    } else {
      L.in = c->dims[l]; L.out = c->dims[l + 1]; L.Kp = pad16(L.in); L.Np = pad16(L.out);
      L.ld_in = L.Kp; L.ld_out = L.Np;
    }
    max_elems = std::max({max_elems, L.in_elems(), L.out_elems()});
    if (L.has_w()) {
      const size_t n = static_cast<size_t>(L.Np) * L.Kp;
      tps_status st;
      if ((st = alloc_t(p, &L.W, n, &p->mem_weights)) != TPS_OK) return cleanup(st);
      if ((st = alloc_t(p, &L.b, L.Np, &p->mem_weights)) != TPS_OK) return cleanup(st);
      if (p->mu != 0.f) {
        if ((st = alloc_t(p, &L.mW, n, &p->mem_optim)) != TPS_OK) return cleanup(st);
        if ((st = alloc_t(p, &L.mb, L.Np, &p->mem_optim)) != TPS_OK) return cleanup(st);
      }
      if (!p->fuse_update && (st = alloc_t(p, &L.dW, n, &p->mem_optim)) != TPS_OK) return cleanup(st);
      if ((st = alloc_t(p, &L.db, L.Np, &p->mem_optim)) != TPS_OK) return cleanup(st);
      L.ver.resize(p->R);
      for (int r = 0; r < p->R; ++r)
        if ((st = alloc_t(p, &L.ver[r], n * p->ew, r == 0 ? &p->mem_weights : &p->mem_stash)) != TPS_OK)
          return cleanup(st);
      p->ver_bytes += static_cast<int64_t>(n) * p->esz;
    }
    p->layers.push_back(L);
  }
  const int nl = p->nlayers();
  tps_status st;
  const Layer& L0 = p->layers[0];
  p->in0_elems = L0.im2col ? static_cast<int64_t>(L0.hw_in) * L0.Ci : L0.in_elems();
  p->act.assign(std::max(p->A0, p->Kmax), std::vector<uint16_t*>(nl, nullptr));
  for (int slot = 0; slot < static_cast<int>(p->act.size()); ++slot)
    for (int k = 0; k < nl; ++k) {
      const bool need = (k == 0) ? slot < p->A0 : slot < p->Kmax;
      if (need && (st = alloc_t(p, &p->act[slot][k], static_cast<size_t>(p->B) * p->layers[k].in_elems() * p->ew,
                                &p->mem_acts)) != TPS_OK)
        return cleanup(st);
    }
  if (L0.im2col) {
    p->x_stage.assign(p->A0, nullptr);
    for (int slot = 0; slot < p->A0; ++slot)
      if ((st = alloc_t(p, &p->x_stage[slot], static_cast<size_t>(p->B) * p->in0_elems, &p->mem_acts)) != TPS_OK)
        return cleanup(st);
  }
  const int64_t outL = p->layers[nl - 1].out_elems(), in0 = p->in0_elems;
  for (int i = 0; i < 2; ++i) {
    if (!p->last) {
      if ((st = alloc_t(p, &p->send_fwd[i], static_cast<size_t>(p->B) * outL * p->ew, &p->mem_comm)) != TPS_OK)
        return cleanup(st);
      if ((st = alloc_t(p, &p->gin[i], static_cast<size_t>(p->B) * outL * p->ew, &p->mem_comm)) != TPS_OK)
        return cleanup(st);
    }
    if (!p->first && (st = alloc_t(p, &p->gout[i], static_cast<size_t>(p->B) * in0 * p->ew, &p->mem_comm)) != TPS_OK)
      return cleanup(st);
    if (nl > 1 && (st = alloc_t(p, &p->gwork[i], static_cast<size_t>(p->B) * max_elems * p->ew, &p->mem_acts)) != TPS_OK)
      return cleanup(st);
  }
  {
    // default on (C5: +9.5 % A/B); TPS_SPLIT_W=0 keeps every backward kernel on the compute stream
    const char* e = std::getenv("TPS_SPLIT_W");
    p->split_w = !(e && e[0] == '0') && p->fuse_update && !p->graph && nl > 1;
  }
  {
    // opt-in (TPS_DUAL=1): the split backward's wgrad + update of layer k and dgrad of layer k-1
    // share one persistent launch (gemm_bwd_dual).  Off by default: the step runs at the 1 kW power
    // cap, so overlapping the two inside one launch only lowers the clock (dual 159 us at 1395 MHz
    // vs 166 us for the two launches at 1515 MHz; the C5 step unchanged)
    const char* e = std::getenv("TPS_DUAL");
    p->dual = p->split_w && e && e[0] == '1' && !p->tf;
  }
  if (p->split_w && (st = alloc_t(p, &p->gwork[2], static_cast<size_t>(p->B) * max_elems * p->ew, &p->mem_acts)) != TPS_OK)
    return cleanup(st);
  if (nl > 1 && !p->tf && std::getenv("TPS_COLSUM") && std::getenv("TPS_COLSUM")[0] == '1') {
    // column partial sums of the input gradients (bias gradients without another pass over G):
    // ceil(rows / 32) x cols floats for the largest input gradient of the stage.  Off by default:
    // the epilogue reduction costs more than the pass it saves (C5 589k vs 600k samples/s)
    int64_t pf = 0;
    for (int k = 1; k < nl; ++k) {
      const Layer& Lk = p->layers[k];
      if (Lk.kind == TPS_LAYER_MAXPOOL2) continue;
      const int64_t rows = static_cast<int64_t>(p->B) * Lk.hw_in;
      const int64_t cols = Lk.kind == TPS_LAYER_CONV3X3 ? Lk.Ci : Lk.Kp;
      pf = std::max(pf, (rows + 31) / 32 * cols);
    }
    for (int i = 0; i < (p->split_w ? 3 : 2) && pf > 0; ++i)
      if ((st = alloc_t(p, &p->bpart[i], static_cast<size_t>(pf), &p->mem_acts)) != TPS_OK) return cleanup(st);
  }
  if (p->split_w) {
    // SM partition of the concurrent pair (dgrad of layer k-1 | fused wgrad + update of layer k):
    // TPS_SPLIT_FRAC = the dgrad's fraction (default 0 = no partition, both grids full: measured
    // faster on C5, 573k vs 533k samples/s at 0.5, 486k at 0.4, 541k at 0.6)
    cudaDeviceGetAttribute(&p->nsm, cudaDevAttrMultiProcessorCount, p->device);
    double f = 0.0;
    if (const char* e = std::getenv("TPS_SPLIT_FRAC")) f = std::atof(e);
    p->part_dgrad = f > 0.0 && f < 1.0 ? std::max(2, static_cast<int>(f * p->nsm + 1.0) / 2 * 2) : 0;
  }
  if (p->last) {
    if (p->layers[nl - 1].kind != TPS_LAYER_LINEAR) return cleanup(fail(TPS_E_CONFIG, "the last layer must be the Linear head"));
    if ((st = alloc_t(p, &p->logits, static_cast<size_t>(p->B) * outL, &p->mem_acts)) != TPS_OK) return cleanup(st);
    if ((st = alloc_t(p, &p->gce, static_cast<size_t>(p->Kmax) * p->B * outL * p->ew, &p->mem_acts)) != TPS_OK)
      return cleanup(st);
    if ((st = alloc_t(p, &p->loss_rows, p->B, &p->mem_acts)) != TPS_OK) return cleanup(st);
    if ((st = alloc_t(p, &p->labels_dev, p->B, &p->mem_acts)) != TPS_OK) return cleanup(st);
    p->loss_cap = 1 << 20;
    if ((st = alloc_t(p, &p->losses, p->loss_cap, &p->mem_acts)) != TPS_OK) return cleanup(st);
    if ((st = alloc_t(p, &p->loss_ctr, 1, &p->mem_acts)) != TPS_OK) return cleanup(st);
  }
  int64_t scr = 0;
  for (auto& L : p->layers)
    if (L.has_w()) scr = std::max(scr, tps::bias_grad_scratch_floats(p->B * L.hw_out, L.Np));
  if ((st = alloc_t(p, &p->scratch, scr, &p->mem_optim)) != TPS_OK) return cleanup(st);
  if (p->fuse_update && (st = alloc_t(p, &p->scratch_side, scr, &p->mem_optim)) != TPS_OK) return cleanup(st);

  }
  const int nl = p->nlayers();
  if (p->dp > 1) {
    const tps_status fs = alloc_t(p, &p->dp_flags, static_cast<size_t>(nl) * 2 * p->dp, &p->mem_comm);
    if (fs != TPS_OK) return cleanup(fs);
  }
  if (p->transport == TPS_TRANSPORT_IPC) {
    const tps_status fs = alloc_t(p, &p->flags, 4, &p->mem_comm);
    if (fs != TPS_OK) return cleanup(fs);
    const char* e = std::getenv("TPS_IPC_DIRECT");
    p->ipc_direct = !p->graph && !(e && e[0] == '0');
  }
  {
    // split-K workspace for the weight-gradient GEMMs whose output tiles cannot fill the GPU
    // (TPS_FUSE_ALL=1: fuse the update into every weight gradient, as before)
    const char* fa = std::getenv("TPS_FUSE_ALL");
    const bool fuse_all = fa && fa[0] == '1';
    int64_t wsf = 0;
    bool any_unfused = false;
    for (Layer& L : p->layers) {
      if (!L.has_w() || L.kind == TPS_LAYER_BN) continue;
      const bool implicit = (L.kind == TPS_LAYER_CONV3X3 && !L.im2col) ||
                            (L.kind == TPS_LAYER_CONV && (L.conv_mode == 1 || L.conv_mode == 3));
      const int K = p->B * (L.kind == TPS_LAYER_LINEAR ? 1 : L.hw_out);
      const int64_t f =
          tps::gemm_splitk_floats(implicit ? tps::GEMM_CONV_WGRAD : tps::GEMM_WGRAD, L.Np, L.Kp, K, L.Kp);
      wsf = std::max(wsf, f);
      L.fuse = p->fuse_update && !p->graph && (f == 0 || p->tf || fuse_all);
      if (p->fuse_update && !p->graph && !L.fuse) {
        any_unfused = true;
        const tps_status dw_st = alloc_t(p, &L.dW, static_cast<size_t>(L.Np) * L.Kp, &p->mem_optim);
        if (dw_st != TPS_OK) return cleanup(dw_st);
      }
    }
    // forward / input-gradient split-K workspace (chain nets): the largest need over the
    // forward group sizes and the collective input gradient of every weight layer
    if (!p->graph && !p->tf) {
      int64_t fdf = 0;
      for (const Layer& L : p->layers) {
        if (!L.has_w() || L.kind == TPS_LAYER_BN) continue;
        const bool conv = L.kind == TPS_LAYER_CONV3X3 && !L.im2col;
        const int hw = L.kind == TPS_LAYER_LINEAR ? 1 : L.hw_out;
        const int fm = conv ? tps::GEMM_CONV_FWD : tps::GEMM_FWD;
        for (int g = 1; g <= p->m; ++g)
          fdf = std::max(fdf, tps::gemm_splitk_floats(fm, g * p->bsz * hw, L.Np, L.Kp, L.Np));
        if (L.kind == TPS_LAYER_LINEAR)
          fdf = std::max(fdf, tps::gemm_splitk_floats(tps::GEMM_DGRAD, p->B, L.Kp, L.Np, L.Kp));
        else if (conv)
          fdf = std::max(fdf, tps::gemm_splitk_floats(tps::GEMM_CONV_DGRAD, p->B * hw, L.Kp / 9, 9 * L.Np, L.Kp / 9));
      }
      if (fdf > 0) {
        const tps_status fd_st = alloc_t(p, &p->splitk_ws_fd, fdf, &p->mem_optim);
        if (fd_st != TPS_OK) return cleanup(fd_st);
        p->splitk_fd_floats = fdf;
      }
    }
    if (!p->fuse_update || p->graph || any_unfused) {
      const tps_status ws_st = alloc_t(p, &p->splitk_ws, wsf, &p->mem_optim);
      if (ws_st != TPS_OK) return cleanup(ws_st);
      p->splitk_floats = wsf;
    }
  }
  {
    size_t free1 = 0, total1 = 0;
    cudaDeviceSynchronize();
    cudaMemGetInfo(&free1, &total1);
    p->observed_bytes = static_cast<int64_t>(free0) - static_cast<int64_t>(free1);
  }
  // streams and events
  int prio_lo = 0, prio_hi = 0;   // least (0) and greatest (< 0) stream priority
  cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
  if (const char* e = std::getenv("TPS_PRIO"); e && e[0] == '0') prio_hi = prio_lo;
  if (const char* e = std::getenv("TPS_NVTX"); e && e[0] == '1') p->nvtx = true;
  p->ev_caller = new_event();
  if (c->compute_stream) {
    p->cs = reinterpret_cast<cudaStream_t>(c->compute_stream);
    p->caller = p->cs;
  } else {
    // the library-owned compute stream (forward GEMMs, the dgrad chain: the critical path) at
    // the greatest priority; the optimizer / weight-gradient streams stay at the least (= the
    // default, 0).  TPS_PRIO=0 puts every stream at the default priority.
    if (cudaStreamCreateWithPriority(&p->cs, cudaStreamNonBlocking, prio_hi) != cudaSuccess)
      return cleanup(fail(TPS_E_CUDA, "stream create"));
    p->own_cs = true;
  }
  for (cudaStream_t* sp : {&p->s_fin, &p->s_fout, &p->s_bin, &p->s_bout})
    if (cudaStreamCreateWithFlags(sp, cudaStreamNonBlocking) != cudaSuccess) return cleanup(fail(TPS_E_CUDA, "stream create"));
  if (cudaStreamCreateWithPriority(&p->s_upd, cudaStreamNonBlocking, prio_lo) != cudaSuccess)
    return cleanup(fail(TPS_E_CUDA, "stream create"));
  p->ev_fwd_ready.resize(2 * p->ng);
  p->ev_fwd_sent.resize(2 * p->ng);
  for (int i = 0; i < 2 * p->ng; ++i) {
    p->ev_fwd_ready[i] = new_event();
    p->ev_fwd_sent[i] = new_event();
  }
  p->ev_grad_ready.resize(nl);
  p->ev_upd_done.resize(nl);
  p->ev_bias_in = new_event();
  p->ev_bias_done = new_event();
  if (p->split_w) {
    p->ev_dg.resize(nl); p->ev_w_done.resize(nl); p->ev_bias_l.resize(nl);
    for (int k = 0; k < nl; ++k) {
      p->ev_dg[k] = new_event(); p->ev_w_done[k] = new_event(); p->ev_bias_l[k] = new_event();
    }
    // weight-gradient stream below the compute stream's dgrad chain (the critical path)
    if (cudaStreamCreateWithPriority(&p->s_w, cudaStreamNonBlocking, prio_lo) != cudaSuccess)
      return cleanup(fail(TPS_E_CUDA, "stream create"));
  }
  for (int k = 0; k < nl; ++k) {
    p->ev_grad_ready[k] = new_event();
    p->ev_upd_done[k] = new_event();
  }
  p->ev_act_free.resize(p->A0);
  for (auto& e : p->ev_act_free) e = new_event();
  p->ev_recv = new_event();
  p->ev_gout_ready = new_event();
  p->ev_gin_ready = new_event();
  for (int i = 0; i < 2; ++i) {
    p->ev_gin_free[i] = new_event();
    p->ev_bwd_sent[i] = new_event();
  }

  // NCCL edge communicators: edge e has a forward comm (ids[2e]) and a backward comm
  // (ids[2e+1]); in both, stage e is rank 0 and stage e+1 is rank 1.  Edges are joined
  // in increasing order so the blocking inits of neighbours pair up without deadlock.
  if (p->transport == TPS_TRANSPORT_NCCL) {
    const ncclUniqueId* ids = static_cast<const ncclUniqueId*>(c->nccl_ids);
    ncclResult_t r;
    if (!p->first) {
      const int e = p->s - 1;
      if ((r = ncclCommInitRank(&p->c_fin, 2, ids[2 * e], 1)) != ncclSuccess) return cleanup(fail(TPS_E_NCCL, "init fin: %s", ncclGetErrorString(r)));
      if ((r = ncclCommInitRank(&p->c_bout, 2, ids[2 * e + 1], 1)) != ncclSuccess) return cleanup(fail(TPS_E_NCCL, "init bout: %s", ncclGetErrorString(r)));
    }
    if (!p->last) {
      const int e = p->s;
      if ((r = ncclCommInitRank(&p->c_fout, 2, ids[2 * e], 0)) != ncclSuccess) return cleanup(fail(TPS_E_NCCL, "init fout: %s", ncclGetErrorString(r)));
      if ((r = ncclCommInitRank(&p->c_bin, 2, ids[2 * e + 1], 0)) != ncclSuccess) return cleanup(fail(TPS_E_NCCL, "init bin: %s", ncclGetErrorString(r)));
    }
  }
  if (cudaDeviceSynchronize() != cudaSuccess) return cleanup(fail(TPS_E_CUDA, "init sync: %s", cudaGetErrorString(cudaGetLastError())));
  *out = p;
  return TPS_OK;
}

tps_status tps_pipeline_destroy(tps_pipeline* p) {
  if (!p) return TPS_OK;
  cudaSetDevice(p->device);
  cudaDeviceSynchronize();
  for (ncclComm_t c : {p->c_fin, p->c_fout, p->c_bin, p->c_bout})
    if (c) ncclCommDestroy(c);
  for (void* a : p->ipc_opened) cudaIpcCloseMemHandle(a);
  for (void* a : p->allocs) {
    if (p->free_fn) p->free_fn(a, p->alloc_ctx);
    else cudaFree(a);
  }
  auto kill_ev = [](cudaEvent_t e) { if (e) cudaEventDestroy(e); };
  for (auto e : p->ev_fwd_ready) kill_ev(e);
  for (auto e : p->ev_fwd_sent) kill_ev(e);
  for (auto e : p->ev_act_free) kill_ev(e);
  kill_ev(p->ev_bias_in);
  kill_ev(p->ev_bias_done);
  for (auto v : {&p->ev_dg, &p->ev_w_done, &p->ev_bias_l})
    for (auto e : *v) kill_ev(e);
  if (p->s_w) cudaStreamDestroy(p->s_w);
  for (auto e : p->ev_grad_ready) kill_ev(e);
  for (auto e : p->ev_upd_done) kill_ev(e);
  for (auto e : p->ev_pool) kill_ev(e);
  for (auto& t : p->timed) { kill_ev(t.a); kill_ev(t.b); }
  for (auto& t : p->tl_pending) { kill_ev(t.a); kill_ev(t.b); }
  if (p->own_origin) kill_ev(p->tl_origin);
  for (cudaEvent_t e : {p->ev_caller, p->ev_recv, p->ev_gout_ready, p->ev_gin_ready, p->ev_gin_free[0], p->ev_gin_free[1],
                        p->ev_bwd_sent[0], p->ev_bwd_sent[1]})
    kill_ev(e);
  for (cudaStream_t s : {p->s_fin, p->s_fout, p->s_bin, p->s_bout, p->s_upd})
    if (s) cudaStreamDestroy(s);
  if (p->own_cs && p->cs) cudaStreamDestroy(p->cs);
  if (p->prev_local) p->prev_local->next_local = nullptr;
  if (p->next_local) p->next_local->prev_local = nullptr;
  delete p;
  return TPS_OK;
}

tps_status tps_local_link(tps_pipeline* const* st, int32_t n) {
  if (!st || n < 1) return fail(TPS_E_INVALID_ARG, "bad stage list");
  for (int i = 0; i < n; ++i) {
    if (!st[i]) return fail(TPS_E_INVALID_ARG, "null stage %d", i);
    if (st[i]->s != i || st[i]->S != n) return fail(TPS_E_CONFIG, "handle %d is stage %d of %d", i, st[i]->s, st[i]->S);
    if (n > 1 && st[i]->transport != TPS_TRANSPORT_LOCAL) return fail(TPS_E_CONFIG, "stage %d is not LOCAL transport", i);
  }
  for (int i = 0; i < n; ++i) {
    st[i]->prev_local = i > 0 ? st[i - 1] : nullptr;
    st[i]->next_local = i + 1 < n ? st[i + 1] : nullptr;
  }
  return TPS_OK;
}

namespace {
struct IpcBlob {
  int32_t magic, stage, num_stages, A0;
  int64_t in_bytes, gin_bytes;          // bytes of one input slot / one gradient receive buffer
  cudaIpcMemHandle_t flags, gin[2], in[16];
};
static_assert(sizeof(IpcBlob) <= TPS_IPC_BLOB_BYTES, "IPC descriptor too large");
constexpr int32_t IPC_MAGIC = 0x54505331;   // "TPS1"

tps_status ipc_open(tps_pipeline* p, const cudaIpcMemHandle_t& h, void** out) {
  CUDA_OK(cudaIpcOpenMemHandle(out, h, cudaIpcMemLazyEnablePeerAccess));
  p->ipc_opened.push_back(*out);
  return TPS_OK;
}
}  // namespace

tps_status tps_ipc_export(tps_pipeline* p, void* out, int64_t cap, int64_t* n) {
  TPS_TRY(check_usable(p));
  if (!out || !n) return fail(TPS_E_INVALID_ARG, "null argument");
  if (p->transport != TPS_TRANSPORT_IPC) return fail(TPS_E_CONFIG, "handle is not IPC transport");
  if (cap < static_cast<int64_t>(sizeof(IpcBlob))) return fail(TPS_E_INVALID_ARG, "cap < %zu", sizeof(IpcBlob));
  if (p->A0 > 16) return fail(TPS_E_UNSUPPORTED, "more than 16 input slots");
  IpcBlob b{};
  b.magic = IPC_MAGIC; b.stage = p->s; b.num_stages = p->S; b.A0 = p->A0;
  b.in_bytes = static_cast<int64_t>(p->B) * p->in0_elems * p->esz;
  b.gin_bytes = p->last ? 0 : static_cast<int64_t>(p->B) * p->layers[p->nlayers() - 1].out_elems() * p->esz;
  CUDA_OK(cudaIpcGetMemHandle(&b.flags, p->flags));
  if (!p->first)
    for (int i = 0; i < p->A0; ++i) CUDA_OK(cudaIpcGetMemHandle(&b.in[i], p->act[i][0]));
  if (!p->last)
    for (int i = 0; i < 2; ++i) CUDA_OK(cudaIpcGetMemHandle(&b.gin[i], p->gin[i]));
  std::memcpy(out, &b, sizeof(b));
  *n = sizeof(b);
  return TPS_OK;
}

tps_status tps_ipc_connect(tps_pipeline* p, const void* prev_blob, const void* next_blob) {
  TPS_TRY(check_usable(p));
  if (p->transport != TPS_TRANSPORT_IPC) return fail(TPS_E_CONFIG, "handle is not IPC transport");
  if (p->ipc_connected) return fail(TPS_E_STATE, "already connected");
  if (p->first != (prev_blob == nullptr) || p->last != (next_blob == nullptr))
    return fail(TPS_E_INVALID_ARG, "stage %d needs %s prev and %s next descriptors", p->s, p->first ? "no" : "a",
                p->last ? "no" : "a");
  if (prev_blob) {
    IpcBlob b;
    std::memcpy(&b, prev_blob, sizeof(b));
    const int64_t want = static_cast<int64_t>(p->B) * p->in0_elems * p->esz;
    if (b.magic != IPC_MAGIC || b.stage != p->s - 1 || b.num_stages != p->S || b.gin_bytes != want)
      return fail(TPS_E_CONFIG, "bad descriptor for stage %d (stage %d, %lld gradient bytes, want %lld)", p->s - 1,
                  b.stage, (long long)b.gin_bytes, (long long)want);
    void* v = nullptr;
    TPS_TRY(ipc_open(p, b.flags, &v));
    p->prev_flags = static_cast<uint64_t*>(v);
    for (int i = 0; i < 2; ++i) {
      TPS_TRY(ipc_open(p, b.gin[i], &v));
      p->prev_gin[i] = static_cast<uint16_t*>(v);
    }
  }
  if (next_blob) {
    IpcBlob b;
    std::memcpy(&b, next_blob, sizeof(b));
    const int64_t want = static_cast<int64_t>(p->B) * p->layers[p->nlayers() - 1].out_elems() * p->esz;
    if (b.magic != IPC_MAGIC || b.stage != p->s + 1 || b.num_stages != p->S || b.in_bytes != want || b.A0 < 1 ||
        b.A0 > 16)
      return fail(TPS_E_CONFIG, "bad descriptor for stage %d (stage %d, %lld input bytes, want %lld)", p->s + 1,
                  b.stage, (long long)b.in_bytes, (long long)want);
    void* v = nullptr;
    TPS_TRY(ipc_open(p, b.flags, &v));
    p->next_flags = static_cast<uint64_t*>(v);
    p->next_in.assign(b.A0, nullptr);
    for (int i = 0; i < b.A0; ++i) {
      TPS_TRY(ipc_open(p, b.in[i], &v));
      p->next_in[i] = static_cast<uint16_t*>(v);
    }
  }
  p->ipc_connected = true;
  return TPS_OK;
}

// ---- data parallelism: connect the R replicas of one stage
namespace {
tps_status dp_check_peer(tps_pipeline* p, int S, int s, int R, int r, int nl, const int64_t* np_kp) {
  if (S != p->S || s != p->s || R != p->dp || nl != p->nlayers())
    return fail(TPS_E_CONFIG, "replica %d is stage %d of %d with %d layers (R = %d); this is stage %d of %d with %d layers (R = %d)",
                r, s, S, nl, R, p->s, p->S, p->nlayers(), p->dp);
  for (int k = 0; k < nl; ++k) {
    const Layer& L = p->layers[k];
    const int64_t want = L.has_w() ? static_cast<int64_t>(L.Np) * L.Kp : 0;
    if (np_kp[k] != want) return fail(TPS_E_CONFIG, "replica %d: layer %d shape differs", r, k);
  }
  return TPS_OK;
}

void dp_alloc_tables(tps_pipeline* p) {
  p->dp_peer_flags.assign(p->dp, nullptr);
  p->dp_dW.assign(p->nlayers(), std::vector<float*>(p->dp, nullptr));
  p->dp_db.assign(p->nlayers(), std::vector<float*>(p->dp, nullptr));
}

struct DpBlobHead {
  int32_t magic, S, s, R, r, nl;
  cudaIpcMemHandle_t flags;
};
constexpr int32_t DP_MAGIC = 0x54505344;   // "TPSD"
}  // namespace

tps_status tps_dp_export(tps_pipeline* p, void* out, int64_t cap, int64_t* n) {
  TPS_TRY(check_usable(p));
  if (!n) return fail(TPS_E_INVALID_ARG, "null n");
  if (p->dp < 2) return fail(TPS_E_CONFIG, "dp_size < 2");
  const int nl = p->nlayers();
  const size_t bytes = sizeof(DpBlobHead) + static_cast<size_t>(nl) * (sizeof(int64_t) + 2 * sizeof(cudaIpcMemHandle_t));
  *n = static_cast<int64_t>(bytes);
  if (!out) return TPS_OK;
  if (cap < static_cast<int64_t>(bytes)) return fail(TPS_E_INVALID_ARG, "cap < %zu", bytes);
  uint8_t* o = static_cast<uint8_t*>(out);
  DpBlobHead h{};
  h.magic = DP_MAGIC; h.S = p->S; h.s = p->s; h.R = p->dp; h.r = p->dp_rank; h.nl = nl;
  CUDA_OK(cudaIpcGetMemHandle(&h.flags, p->dp_flags));
  std::memcpy(o, &h, sizeof(h));
  o += sizeof(h);
  for (int k = 0; k < nl; ++k) {
    const Layer& L = p->layers[k];
    const int64_t npk = L.has_w() ? static_cast<int64_t>(L.Np) * L.Kp : 0;
    cudaIpcMemHandle_t hw{}, hb{};
    if (L.has_w()) {
      CUDA_OK(cudaIpcGetMemHandle(&hw, L.dW));
      CUDA_OK(cudaIpcGetMemHandle(&hb, L.db));
    }
    std::memcpy(o, &npk, sizeof(npk)); o += sizeof(npk);
    std::memcpy(o, &hw, sizeof(hw)); o += sizeof(hw);
    std::memcpy(o, &hb, sizeof(hb)); o += sizeof(hb);
  }
  return TPS_OK;
}

tps_status tps_dp_connect(tps_pipeline* p, const void* const* blobs, int32_t R) {
  TPS_TRY(check_usable(p));
  if (!blobs || R != p->dp || R < 2) return fail(TPS_E_INVALID_ARG, "need dp_size descriptors");
  if (p->dp_connected) return fail(TPS_E_STATE, "already connected");
  const int nl = p->nlayers();
  dp_alloc_tables(p);
  for (int q = 0; q < R; ++q) {
    if (!blobs[q]) return fail(TPS_E_INVALID_ARG, "null descriptor %d", q);
    const uint8_t* b = static_cast<const uint8_t*>(blobs[q]);
    DpBlobHead h;
    std::memcpy(&h, b, sizeof(h));
    b += sizeof(h);
    if (h.magic != DP_MAGIC || h.r != q) return fail(TPS_E_CONFIG, "descriptor %d is not replica %d's", q, q);
    std::vector<int64_t> npk(std::max(0, h.nl));
    std::vector<cudaIpcMemHandle_t> hw(npk.size()), hb(npk.size());
    for (size_t k = 0; k < npk.size(); ++k) {
      std::memcpy(&npk[k], b, sizeof(int64_t)); b += sizeof(int64_t);
      std::memcpy(&hw[k], b, sizeof(cudaIpcMemHandle_t)); b += sizeof(cudaIpcMemHandle_t);
      std::memcpy(&hb[k], b, sizeof(cudaIpcMemHandle_t)); b += sizeof(cudaIpcMemHandle_t);
    }
    TPS_TRY(dp_check_peer(p, h.S, h.s, h.R, q, h.nl, npk.data()));
    if (q == p->dp_rank) {
      p->dp_peer_flags[q] = p->dp_flags;
      for (int k = 0; k < nl; ++k) {
        p->dp_dW[k][q] = p->layers[k].dW;
        p->dp_db[k][q] = p->layers[k].db;
      }
      continue;
    }
    void* v = nullptr;
    TPS_TRY(ipc_open(p, h.flags, &v));
    p->dp_peer_flags[q] = static_cast<uint64_t*>(v);
    for (int k = 0; k < nl; ++k) {
      if (!p->layers[k].has_w()) continue;
      TPS_TRY(ipc_open(p, hw[k], &v));
      p->dp_dW[k][q] = static_cast<float*>(v);
      TPS_TRY(ipc_open(p, hb[k], &v));
      p->dp_db[k][q] = static_cast<float*>(v);
    }
  }
  p->dp_connected = true;
  return TPS_OK;
}

tps_status tps_begin_run(tps_pipeline* p, int64_t first_mb, int64_t n_mb) {
  TPS_TRY(check_usable(p));
  return begin_run(p, first_mb, n_mb);
}

tps_status tps_stage_forward(tps_pipeline* p, int64_t mb, int32_t micro, int32_t count, const void* x,
                             const int32_t* labels) {
  TPS_TRY(check_usable(p));
  return bracket(p, TPS_EV_F, mb, [&] { return do_forward(p, mb, micro, count, x, labels); });
}

tps_status tps_stage_backward(tps_pipeline* p, int64_t mb, int32_t staleness) {
  TPS_TRY(check_usable(p));
  return bracket(p, TPS_EV_B, mb, [&] { return do_backward(p, mb, staleness); });
}

tps_status tps_stage_update(tps_pipeline* p, int64_t mb) {
  TPS_TRY(check_usable(p));
  return bracket(p, TPS_EV_U, mb, [&] { return do_update(p, mb); });
}

tps_status tps_run_schedule(tps_pipeline* p, int64_t first_mb, int64_t n_mb, const void* x_pool, const int32_t* y_pool,
                            int32_t pool) {
  TPS_TRY(check_usable(p));
  if (p->transport == TPS_TRANSPORT_LOCAL) return fail(TPS_E_CONFIG, "LOCAL transport: use tps_run_schedule_local");
  if (pool < 1) return fail(TPS_E_INVALID_ARG, "pool must be >= 1");
  if ((p->first && !x_pool) || (p->last && !y_pool)) return fail(TPS_E_INVALID_ARG, "missing input pool");
  TPS_TRY(begin_run(p, first_mb, n_mb));
  while (p->in_run) {
    const tps_event e = p->order[p->pos];
    TPS_TRY(fire(p, e, x_pool, y_pool, pool));
  }
  return join_update_stream(p);
}

namespace {
tps_status local_walk(tps_pipeline* const* st, int32_t n, int64_t first_mb, int64_t n_mb, const void* x_pool,
                      const int32_t* y_pool, int32_t pool);
}  // namespace

tps_status tps_run_schedule_local(tps_pipeline* const* st, int32_t n, int64_t first_mb, int64_t n_mb,
                                  const void* x_pool, const int32_t* y_pool, int32_t pool) {
  return local_walk(st, n, first_mb, n_mb, x_pool, y_pool, pool);
}

// ---- CUDA-graph capture / replay of whole runs
struct tps_graph {
  std::vector<tps_pipeline*> h;
  cudaGraphExec_t exec = nullptr;
  cudaStream_t origin = nullptr;
  int64_t n = 0, next = 0, replays = 0;
  cudaEvent_t done = nullptr;                  // recorded after every launch; the handles' streams wait on it
  std::vector<std::vector<tps_event>> slice;   // per handle: the captured run's trace
  std::vector<int64_t> launches, latest_after; // per handle: kernels per run, version after last run
};

namespace {
int64_t lcm64(int64_t a, int64_t b) {
  int64_t x = a, y = b;
  while (y) { const int64_t t = x % y; x = y; y = t; }
  return a / x * b;
}

// re-record every persistent event of the handle on `st` (inside a capture: later waits then
// refer to nodes of the graph, never to work recorded before the capture began)
tps_status rearm_events(tps_pipeline* p, cudaStream_t st) {
  auto rec = [&](cudaEvent_t e) -> tps_status {
    if (e) CUDA_OK(cudaEventRecord(e, st));
    return TPS_OK;
  };
  for (auto* v : {&p->ev_fwd_ready, &p->ev_fwd_sent, &p->ev_act_free, &p->ev_grad_ready, &p->ev_upd_done, &p->ev_dg,
                  &p->ev_w_done, &p->ev_bias_l})
    for (cudaEvent_t e : *v) TPS_TRY(rec(e));
  for (cudaEvent_t e : {p->ev_bias_in, p->ev_bias_done, p->ev_recv, p->ev_gout_ready, p->ev_gin_ready, p->ev_gin_free[0],
                        p->ev_gin_free[1], p->ev_bwd_sent[0], p->ev_bwd_sent[1]})
    TPS_TRY(rec(e));
  return TPS_OK;
}
}  // namespace

namespace {
// launch, then order every stream of every handle after the graph (later walks, readbacks and
// synchronisations of the handles see its work)
tps_status graph_launch(tps_graph* g) {
  CUDA_OK(cudaGraphLaunch(g->exec, g->origin));
  // events recorded inside the capture cannot be waited on by later (uncaptured) work: re-record
  // them after the graph so the next walk orders after it
  for (tps_pipeline* p : g->h) TPS_TRY(rearm_events(p, g->origin));
  CUDA_OK(cudaEventRecord(g->done, g->origin));
  for (tps_pipeline* p : g->h)
    for (cudaStream_t hs : {p->cs, p->s_upd, p->s_w, p->s_fin, p->s_fout, p->s_bin, p->s_bout})
      if (hs && hs != g->origin) CUDA_OK(cudaStreamWaitEvent(hs, g->done, 0));
  return TPS_OK;
}
}  // namespace

tps_status tps_graph_capture(tps_pipeline* const* st, int32_t n, int64_t first_mb, int64_t n_mb, const void* x_pool,
                             const int32_t* y_pool, int32_t pool, uint64_t stream, tps_graph** out) {
  if (!st || n < 1 || !out || stream == 0 || pool < 1) return fail(TPS_E_INVALID_ARG, "bad arguments (stream must not be 0)");
  *out = nullptr;
  cudaStream_t origin = reinterpret_cast<cudaStream_t>(stream);
  int64_t period = lcm64(2, pool);
  for (int i = 0; i < n; ++i) {
    tps_pipeline* p = st[i];
    TPS_TRY(check_usable(p));
    if (p->transport == TPS_TRANSPORT_IPC || p->transport == TPS_TRANSPORT_NCCL || p->dp > 1)
      return fail(TPS_E_UNSUPPORTED, "graph capture: LOCAL / single-stage handles only");
    if (p->profiling || p->timeline)
      return fail(TPS_E_STATE, "graph capture with per-launch profiling or the timeline enabled");
    if (p->in_run) return fail(TPS_E_ORDER, "handle %d is inside a run", i);
    period = lcm64(period, lcm64(lcm64(p->A0, p->Kmax), p->R));
  }
  if (n_mb < period || n_mb % period)
    return fail(TPS_E_CONFIG, "a replayable run covers a multiple of the schedule period %lld mini-batches", (long long)period);
  tps_graph* g = new tps_graph();
  g->h.assign(st, st + n);
  g->origin = origin;
  g->n = n_mb;
  std::vector<size_t> t0(n);
  std::vector<int64_t> l0(n);
  std::vector<cudaStream_t> callers(n);
  for (int i = 0; i < n; ++i) {
    t0[i] = st[i]->trace.size();
    l0[i] = st[i]->launches;
    callers[i] = st[i]->caller;
    st[i]->caller = origin;
  }
  // the capture starts once everything before it has finished (events recorded earlier are
  // re-armed inside the capture)
  CUDA_OK(cudaDeviceSynchronize());
  CUDA_OK(cudaStreamBeginCapture(origin, cudaStreamCaptureModeRelaxed));
  tps_status ws = TPS_OK;
  for (int i = 0; i < n && ws == TPS_OK; ++i) ws = rearm_events(st[i], origin);
  if (ws == TPS_OK) ws = local_walk(st, n, first_mb, n_mb, x_pool, y_pool, pool);
  for (int i = 0; i < n && ws == TPS_OK; ++i) ws = tps_join(st[i], stream);
  const std::string werr = g_err;
  cudaGraph_t graph = nullptr;
  const cudaError_t ce = cudaStreamEndCapture(origin, &graph);
  for (int i = 0; i < n; ++i) st[i]->caller = callers[i];
  if (ws != TPS_OK || ce != cudaSuccess) {
    if (graph) cudaGraphDestroy(graph);
    cudaGetLastError();
    delete g;
    if (ws != TPS_OK) return fail(ws, "graph capture: %s", werr.c_str());
    return fail(TPS_E_CUDA, "cudaStreamEndCapture: %s", cudaGetErrorString(ce));
  }
  const cudaError_t ie = cudaGraphInstantiate(&g->exec, graph, 0);
  cudaGraphDestroy(graph);
  if (ie != cudaSuccess) {
    delete g;
    return fail(TPS_E_CUDA, "cudaGraphInstantiate: %s", cudaGetErrorString(ie));
  }
  for (int i = 0; i < n; ++i) {
    tps_pipeline* p = st[i];
    g->slice.emplace_back(p->trace.begin() + static_cast<std::ptrdiff_t>(t0[i]), p->trace.end());
    g->launches.push_back(p->launches - l0[i]);
    g->latest_after.push_back(p->latest);
  }
  g->next = first_mb + n_mb;
  g->done = new_event();
  // the walk advanced the host state; now run the captured work once
  TPS_TRY(graph_launch(g));
  *out = g;
  return TPS_OK;
}

tps_status tps_graph_replay(tps_graph* g) {
  if (!g || !g->exec) return fail(TPS_E_INVALID_ARG, "null graph");
  for (size_t i = 0; i < g->h.size(); ++i) {
    tps_pipeline* p = g->h[i];
    TPS_TRY(check_usable(p));
    if (p->in_run || p->latest != g->latest_after[i])
      return fail(TPS_E_STATE, "handle %zu changed since the graph's last run (replay continues that run)", i);
  }
  TPS_TRY(graph_launch(g));
  g->replays += 1;
  const int64_t shift = g->replays * g->n;     // mini-batches and versions both advance by n per run
  for (size_t i = 0; i < g->h.size(); ++i) {
    tps_pipeline* p = g->h[i];
    for (tps_event e : g->slice[i]) {
      e.mb += shift;
      e.v_used += shift;
      e.v_latest += shift;
      p->trace.push_back(e);
    }
    p->latest += g->n;
    g->latest_after[i] = p->latest;
    if (p->last) p->loss_count += g->n;
    p->launches += g->launches[i];
  }
  g->next += g->n;
  return TPS_OK;
}

tps_status tps_graph_destroy(tps_graph* g) {
  if (!g) return TPS_OK;
  if (g->exec) {
    cudaStreamSynchronize(g->origin);
    cudaGraphExecDestroy(g->exec);
  }
  if (g->done) cudaEventDestroy(g->done);
  delete g;
  return TPS_OK;
}

namespace {
tps_status local_walk(tps_pipeline* const* st, int32_t n, int64_t first_mb, int64_t n_mb, const void* x_pool,
                      const int32_t* y_pool, int32_t pool) {
  if (!st || n < 1 || pool < 1 || !st[0]) return fail(TPS_E_INVALID_ARG, "bad arguments");
  // n = S handles of one pipeline, or R·S handles of R data-parallel replicas (replica-major)
  const int S = st[0]->S;
  if (n % S) return fail(TPS_E_CONFIG, "%d handles are not whole pipelines of %d stages", n, S);
  for (int i = 0; i < n; ++i) {
    if (!st[i] || st[i]->s != i % S || st[i]->S != S) return fail(TPS_E_CONFIG, "handle %d is not stage %d of %d", i, i % S, S);
    TPS_TRY(check_usable(st[i]));
    TPS_TRY(begin_run(st[i], first_mb, n_mb));
  }
  // Round-robin over handles; fire a handle's next static event once its cross-stage input
  // has been enqueued and the buffer it overwrites has been consumed downstream (neighbours
  // are the same replica's stages s-1 / s+1).  Replicas synchronise on the device only.
  std::vector<int64_t> fcount(n, 0), bcount(n, 0);
  const int ng = st[0]->ng;
  static const bool trace_fire = [] {
    const char* e = std::getenv("TPS_TRACE_FIRE");
    return e && e[0] == '1';
  }();
  for (;;) {
    bool all_done = true, progress = false;
    for (int i = 0; i < n; ++i) {
      tps_pipeline* p = st[i];
      const int s = i % S;
      if (!p->in_run) continue;
      all_done = false;
      const tps_event e = p->order[p->pos];
      const int64_t jr = e.mb - first_mb;
      if (e.kind == TPS_EV_F) {
        const int grp = e.micro / p->g;
        const int64_t idx = jr * ng + grp;
        if (s > 0 && fcount[i - 1] <= idx) continue;                          // input not produced
        if (s < S - 1 && jr >= 2 && fcount[i + 1] <= (jr - 2) * ng + grp) continue;  // send buffer busy
      } else if (e.kind == TPS_EV_B) {
        if (s < S - 1 && bcount[i + 1] <= jr) continue;                      // gradient not produced
        if (s > 0 && jr >= 2 && bcount[i - 1] <= jr - 2) continue;           // gout buffer busy
      }
      if (trace_fire) {
        std::fprintf(stderr, "[tps] fire h=%d s=%d kind=%d mb=%lld micro=%d\n", i, s, e.kind, (long long)e.mb, e.micro);
        std::fflush(stderr);
      }
      TPS_TRY(fire(p, e, x_pool, y_pool, pool));
      if (e.kind == TPS_EV_F) fcount[i] += 1;
      if (e.kind == TPS_EV_B) bcount[i] += 1;
      progress = true;
    }
    if (all_done) break;
    if (!progress) return fail(TPS_E_STATE, "local schedule deadlock");
  }
  for (int i = 0; i < n; ++i) TPS_TRY(join_update_stream(st[i]));
  return TPS_OK;
}
}  // namespace

tps_status tps_join(tps_pipeline* p, uint64_t stream) {
  TPS_TRY(check_usable(p));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  CUDA_OK(cudaStreamIsCapturing(st, &cap));
  // record the tail of every stream of the handle and make `st` wait for it (while `st` is being
  // captured, only the streams the capture pulled in: the others hold no work of the graph)
  for (cudaStream_t hs : {p->cs, p->s_upd, p->s_w, p->s_fin, p->s_fout, p->s_bin, p->s_bout}) {
    if (!hs || hs == st) continue;
    if (cap == cudaStreamCaptureStatusActive) {
      cudaStreamCaptureStatus hc = cudaStreamCaptureStatusNone;
      CUDA_OK(cudaStreamIsCapturing(hs, &hc));
      if (hc != cudaStreamCaptureStatusActive) continue;
    }
    CUDA_OK(cudaEventRecord(p->ev_caller, hs));
    CUDA_OK(cudaStreamWaitEvent(st, p->ev_caller, 0));
  }
  return TPS_OK;
}

tps_status tps_debug_progress(tps_pipeline* p, int64_t* pos, int64_t* n_events, int32_t* busy) {
  if (!p) return fail(TPS_E_INVALID_ARG, "null handle");
  if (pos) *pos = static_cast<int64_t>(p->pos);
  if (n_events) *n_events = static_cast<int64_t>(p->order.size());
  if (busy) {
    int b = 0, i = 0;
    for (cudaStream_t st : {p->cs, p->s_fin, p->s_fout, p->s_bin, p->s_bout, p->s_upd}) {
      if (st && cudaStreamQuery(st) == cudaErrorNotReady) b |= 1 << i;
      ++i;
    }
    cudaGetLastError();
    *busy = b;
  }
  return TPS_OK;
}

tps_status tps_synchronize(tps_pipeline* p) {
  if (!p) return fail(TPS_E_INVALID_ARG, "null handle");
  if (p->poisoned) return fail(TPS_E_STATE, "handle poisoned");
  cudaSetDevice(p->device);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    p->poisoned = true;
    return fail(TPS_E_CUDA, "device error: %s", cudaGetErrorString(e));
  }
  for (ncclComm_t c : {p->c_fin, p->c_fout, p->c_bin, p->c_bout}) {
    if (!c) continue;
    ncclResult_t ar = ncclSuccess;
    ncclCommGetAsyncError(c, &ar);
    if (ar != ncclSuccess) {
      p->poisoned = true;
      return fail(TPS_E_NCCL, "async NCCL error: %s", ncclGetErrorString(ar));
    }
  }
  return drain_timing(p);
}

tps_status tps_stash_info(tps_pipeline* p, int32_t* live, int64_t* stash, int64_t* peak) {
  if (!p) return fail(TPS_E_INVALID_ARG, "null handle");
  std::vector<int64_t> lv{p->latest};
  for (auto& kv : p->fwd_version)
    if (std::find(lv.begin(), lv.end(), kv.second) == lv.end()) lv.push_back(kv.second);
  const int64_t n_live = std::min<int64_t>(static_cast<int64_t>(lv.size()), p->R);   // V: R = 1
  if (live) *live = static_cast<int32_t>(n_live);
  if (stash) *stash = (n_live - 1) * p->ver_bytes;
  if (peak) *peak = p->peak_stash_live;
  return TPS_OK;
}

tps_status tps_intermediate_weight(tps_pipeline* p, int32_t layer, int32_t staleness, void* out_bf16) {
  TPS_TRY(check_usable(p));
  if (layer < 0 || layer >= p->nlayers() || !out_bf16) return fail(TPS_E_INVALID_ARG, "bad layer/out");
  if (staleness < 0 || staleness > p->latest || staleness >= p->R) return fail(TPS_E_STALENESS, "no live stash for staleness %d", staleness);
  float a, b;
  compute_coeffs(p->variant, p->blend, staleness, p->lambda, &a, &b);
  if (!p->layers[layer].has_w()) return fail(TPS_E_INVALID_ARG, "layer %d has no parameters", layer);
  Layer& L = p->layers[layer];
  if (L.kind == TPS_LAYER_BN) return fail(TPS_E_INVALID_ARG, "layer %d: BN γ versions are fp32 (use tps_get_weights)", layer);
  CUDA_OK(cudaStreamWaitEvent(p->cs, p->ev_upd_done[layer], 0));
  const int64_t vs = p->latest - staleness;
  if (p->tf)   // tf32 storage: fp32 out, tf32_rna(fp32(α·s) + fp32(β·l))
    CUDA_OK(tps::launch_blend_materialize_tf32(reinterpret_cast<const float*>(L.ver[vs % p->R]),
                                               reinterpret_cast<const float*>(L.ver[p->latest % p->R]),
                                               static_cast<float*>(out_bf16), static_cast<int64_t>(L.Np) * L.Kp, a, b,
                                               p->cs));
  else
    CUDA_OK(tps::launch_blend_materialize(L.ver[vs % p->R], L.ver[p->latest % p->R], static_cast<uint16_t*>(out_bf16),
                                          static_cast<int64_t>(L.Np) * L.Kp, a, b, p->cs));
  p->launches += 1;
  return TPS_OK;
}

tps_status tps_get_version(tps_pipeline* p, int32_t layer, int32_t staleness, void* out_bf16) {
  TPS_TRY(check_usable(p));
  if (layer < 0 || layer >= p->nlayers() || !out_bf16) return fail(TPS_E_INVALID_ARG, "bad layer/out");
  if (staleness < 0 || staleness > p->latest || staleness >= p->R) return fail(TPS_E_STALENESS, "no live version at staleness %d", staleness);
  if (!p->layers[layer].has_w()) return fail(TPS_E_INVALID_ARG, "layer %d has no parameters", layer);
  Layer& L = p->layers[layer];
  if (L.kind == TPS_LAYER_BN) return fail(TPS_E_INVALID_ARG, "layer %d: BN γ versions are fp32 (use tps_get_weights)", layer);
  CUDA_OK(cudaStreamWaitEvent(p->cs, p->ev_upd_done[layer], 0));
  CUDA_OK(cudaMemcpyAsync(out_bf16, L.ver[(p->latest - staleness) % p->R], static_cast<size_t>(L.Np) * L.Kp * p->esz,
                          cudaMemcpyDeviceToDevice, p->cs));
  TPS_TRY(sync_streams(p));
  return TPS_OK;
}

tps_status tps_get_weights(tps_pipeline* p, int32_t layer, float* w, float* b, float* mw, float* mb) {
  TPS_TRY(check_usable(p));
  if (layer < 0 || layer >= p->nlayers()) return fail(TPS_E_INVALID_ARG, "bad layer %d", layer);
  TPS_TRY(sync_streams(p));
  if (!p->layers[layer].has_w()) return fail(TPS_E_INVALID_ARG, "layer %d has no parameters", layer);
  Layer& L = p->layers[layer];
  const size_t rowb = static_cast<size_t>(L.in) * 4, ldb = static_cast<size_t>(L.Kp) * 4;
  if (w) CUDA_OK(cudaMemcpy2D(w, rowb, L.W, ldb, rowb, L.out, cudaMemcpyDeviceToHost));
  if (b) {
    if (L.b) CUDA_OK(cudaMemcpy(b, L.b, static_cast<size_t>(L.out) * 4, cudaMemcpyDeviceToHost));
    else std::memset(b, 0, static_cast<size_t>(L.out) * 4);
  }
  if (mw) {
    if (L.mW) CUDA_OK(cudaMemcpy2D(mw, rowb, L.mW, ldb, rowb, L.out, cudaMemcpyDeviceToHost));
    else std::memset(mw, 0, rowb * L.out);
  }
  if (mb) {
    if (L.mb) CUDA_OK(cudaMemcpy(mb, L.mb, static_cast<size_t>(L.out) * 4, cudaMemcpyDeviceToHost));
    else std::memset(mb, 0, static_cast<size_t>(L.out) * 4);
  }
  return TPS_OK;
}

tps_status tps_set_weights(tps_pipeline* p, int32_t layer, const float* w, const float* b) {
  TPS_TRY(check_usable(p));
  if (layer < 0 || layer >= p->nlayers()) return fail(TPS_E_INVALID_ARG, "bad layer %d", layer);
  TPS_TRY(sync_streams(p));
  if (!p->layers[layer].has_w()) return fail(TPS_E_INVALID_ARG, "layer %d has no parameters", layer);
  Layer& L = p->layers[layer];
  const size_t rowb = static_cast<size_t>(L.in) * 4, ldb = static_cast<size_t>(L.Kp) * 4;
  const size_t n = static_cast<size_t>(L.Np) * L.Kp;
  // stream-ordered on the compute stream: a synchronous cudaMemcpy from pageable memory may
  // return before its DMA lands, and the legacy stream does not order the handle's
  // non-blocking streams
  if (w) {
    CUDA_OK(cudaMemsetAsync(L.W, 0, n * 4, p->cs));
    CUDA_OK(cudaMemcpy2DAsync(L.W, ldb, w, rowb, rowb, L.out, cudaMemcpyHostToDevice, p->cs));
  }
  if (b && L.b) {
    CUDA_OK(cudaMemsetAsync(L.b, 0, static_cast<size_t>(L.Np) * 4, p->cs));
    CUDA_OK(cudaMemcpyAsync(L.b, b, static_cast<size_t>(L.out) * 4, cudaMemcpyHostToDevice, p->cs));
  }
  if (L.mW) CUDA_OK(cudaMemsetAsync(L.mW, 0, n * 4, p->cs));
  if (L.mb) CUDA_OK(cudaMemsetAsync(L.mb, 0, static_cast<size_t>(L.Np) * 4, p->cs));
  if (L.kind == TPS_LAYER_BN)
    CUDA_OK(cudaMemcpyAsync(L.verf[p->latest % p->R], L.W, n * 4, cudaMemcpyDeviceToDevice, p->cs));
  else if (p->tf)
    CUDA_OK(tps::launch_f32_to_tf32(L.W, reinterpret_cast<float*>(L.ver[p->latest % p->R]), static_cast<int64_t>(n), p->cs));
  else
    CUDA_OK(tps::launch_f32_to_bf16(L.W, L.ver[p->latest % p->R], static_cast<int64_t>(n), p->cs));
  p->launches += 1;
  TPS_TRY(sync_streams(p));
  return TPS_OK;
}

tps_status tps_init_weights_synthetic(tps_pipeline* p) {
  TPS_TRY(check_usable(p));
  for (auto& L : p->layers) {
    if (!L.has_w()) continue;
    if (L.kind == TPS_LAYER_BN) {   // γ = 1, β = 0
      std::vector<float> one(L.Np, 1.0f);
      CUDA_OK(cudaMemcpyAsync(L.W, one.data(), one.size() * 4, cudaMemcpyHostToDevice, p->cs));
      CUDA_OK(cudaMemsetAsync(L.b, 0, static_cast<size_t>(L.Np) * 4, p->cs));
      if (L.mW) CUDA_OK(cudaMemsetAsync(L.mW, 0, static_cast<size_t>(L.Np) * 4, p->cs));
      if (L.mb) CUDA_OK(cudaMemsetAsync(L.mb, 0, static_cast<size_t>(L.Np) * 4, p->cs));
      CUDA_OK(cudaMemcpyAsync(L.verf[p->latest % p->R], L.W, static_cast<size_t>(L.Np) * 4, cudaMemcpyDeviceToDevice, p->cs));
      CUDA_OK(cudaStreamSynchronize(p->cs));
      continue;
    }
    // round half to even, like synthgen (Python round): fan_in = 512 -> log2(sqrt) = 4.5 -> 4
    const int shift = static_cast<int>(std::nearbyint(std::log2(std::sqrt(static_cast<double>(L.in)))));
    CUDA_OK(cudaMemsetAsync(L.W, 0, static_cast<size_t>(L.Np) * L.Kp * 4, p->cs));
    CUDA_OK(tps::launch_fill_synthetic(3, p->seed, 0x0100 + static_cast<uint64_t>(L.gidx), L.out, L.in, L.Kp, 0, shift,
                                       L.W, p->cs));
    if (L.b) CUDA_OK(cudaMemsetAsync(L.b, 0, static_cast<size_t>(L.Np) * 4, p->cs));
    if (L.mW) CUDA_OK(cudaMemsetAsync(L.mW, 0, static_cast<size_t>(L.Np) * L.Kp * 4, p->cs));
    if (L.mb) CUDA_OK(cudaMemsetAsync(L.mb, 0, static_cast<size_t>(L.Np) * 4, p->cs));
    if (p->tf)
      CUDA_OK(tps::launch_f32_to_tf32(L.W, reinterpret_cast<float*>(L.ver[p->latest % p->R]),
                                      static_cast<int64_t>(L.Np) * L.Kp, p->cs));
    else
      CUDA_OK(tps::launch_f32_to_bf16(L.W, L.ver[p->latest % p->R], static_cast<int64_t>(L.Np) * L.Kp, p->cs));
    p->launches += 2;
  }
  TPS_TRY(sync_streams(p));
  return TPS_OK;
}

tps_status tps_get_losses(tps_pipeline* p, float* out, int64_t cap, int64_t* n) {
  TPS_TRY(check_usable(p));
  if (!n) return fail(TPS_E_INVALID_ARG, "null n");
  *n = p->last ? p->loss_count : 0;
  if (p->last && out && *n > 0) {
    TPS_TRY(sync_streams(p));
    CUDA_OK(cudaMemcpy(out, p->losses, sizeof(float) * static_cast<size_t>(std::min(cap, *n)), cudaMemcpyDeviceToHost));
  }
  return TPS_OK;
}

tps_status tps_read_losses_async(tps_pipeline* p, int64_t first, int64_t n, float* host_dst, uint64_t stream) {
  TPS_TRY(check_usable(p));
  if (!p->last) return fail(TPS_E_INVALID_ARG, "losses live on the last stage");
  if (!host_dst || first < 0 || n < 0 || first + n > p->loss_count)
    return fail(TPS_E_INVALID_ARG, "losses [%lld, +%lld) not produced (have %lld)", (long long)first, (long long)n,
                (long long)p->loss_count);
  if (n == 0) return TPS_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (st != p->cs) {   // the loss kernels run on the compute stream
    CUDA_OK(cudaEventRecord(p->ev_caller, p->cs));
    CUDA_OK(cudaStreamWaitEvent(st, p->ev_caller, 0));
  }
  CUDA_OK(cudaMemcpyAsync(host_dst, p->losses + first, static_cast<size_t>(n) * sizeof(float), cudaMemcpyDeviceToHost, st));
  return TPS_OK;
}

tps_status tps_get_trace(tps_pipeline* p, tps_event* out, int64_t cap, int64_t* n) {
  if (!p || !n) return fail(TPS_E_INVALID_ARG, "null argument");
  *n = static_cast<int64_t>(p->trace.size());
  if (out) std::memcpy(out, p->trace.data(), sizeof(tps_event) * static_cast<size_t>(std::min(cap, *n)));
  return TPS_OK;
}

tps_status tps_clear_trace(tps_pipeline* p) {
  if (!p) return fail(TPS_E_INVALID_ARG, "null handle");
  p->trace.clear();
  return TPS_OK;
}

tps_status tps_memory_stats(tps_pipeline* p, int64_t* weights, int64_t* stash, int64_t* acts, int64_t* optim,
                            int64_t* comm, int64_t* peak) {
  if (!p) return fail(TPS_E_INVALID_ARG, "null handle");
  if (weights) *weights = p->mem_weights;
  if (stash) *stash = p->mem_stash;
  if (acts) *acts = p->mem_acts;
  if (optim) *optim = p->mem_optim;
  if (comm) *comm = p->mem_comm;
  if (peak) *peak = p->mem_peak;
  return TPS_OK;
}

tps_status tps_memory_observed(tps_pipeline* p, int64_t* device_bytes) {
  if (!p || !device_bytes) return fail(TPS_E_INVALID_ARG, "null argument");
  *device_bytes = p->observed_bytes;
  return TPS_OK;
}

tps_status tps_set_profiling(tps_pipeline* p, int32_t enable) {
  TPS_TRY(check_usable(p));
  TPS_TRY(sync_streams(p));
  TPS_TRY(drain_timing(p));
  p->profiling = enable != 0;
  for (int k = 0; k < 6; ++k) { p->stat_ms[k] = 0; p->stat_work[k] = 0; p->stat_n[k] = 0; }
  return TPS_OK;
}

tps_status tps_set_timeline(tps_pipeline* p, int32_t enable, uint64_t origin_event) {
  TPS_TRY(check_usable(p));
  TPS_TRY(sync_streams(p));
  for (auto& t : p->tl_pending) { p->ev_pool.push_back(t.a); p->ev_pool.push_back(t.b); }
  p->tl_pending.clear();
  p->tl_done.clear();
  if (p->own_origin && p->tl_origin) cudaEventDestroy(p->tl_origin);
  p->tl_origin = nullptr;
  p->own_origin = false;
  p->timeline = enable != 0;
  if (!p->timeline) return TPS_OK;
  if (origin_event) {
    p->tl_origin = reinterpret_cast<cudaEvent_t>(origin_event);
  } else {
    CUDA_OK(cudaEventCreate(&p->tl_origin));
    p->own_origin = true;
    CUDA_OK(cudaEventRecord(p->tl_origin, p->cs));
  }
  return TPS_OK;
}

tps_status tps_get_timeline(tps_pipeline* p, tps_timeline_rec* out, int64_t cap, int64_t* n) {
  TPS_TRY(check_usable(p));
  if (!n || cap < 0 || (cap > 0 && !out)) return fail(TPS_E_INVALID_ARG, "bad timeline buffer");
  TPS_TRY(drain_timeline(p));
  *n = static_cast<int64_t>(p->tl_done.size());
  if (out) std::memcpy(out, p->tl_done.data(), sizeof(tps_timeline_rec) * static_cast<size_t>(std::min(cap, *n)));
  return TPS_OK;
}

tps_status tps_kernel_stats(tps_pipeline* p, int32_t which, int64_t* launches, double* ms, double* work) {
  TPS_TRY(check_usable(p));
  if (which < 0 || which > 5) return fail(TPS_E_INVALID_ARG, "bad kernel class");
  TPS_TRY(sync_streams(p));
  TPS_TRY(drain_timing(p));
  if (launches) *launches = p->stat_n[which];
  if (ms) *ms = p->stat_ms[which];
  if (work) *work = p->stat_work[which];
  return TPS_OK;
}

tps_status tps_launch_count(tps_pipeline* p, int64_t* n) {
  if (!p || !n) return fail(TPS_E_INVALID_ARG, "null argument");
  *n = p->launches;
  return TPS_OK;
}

tps_status tps_fill_synthetic(int32_t kind, uint64_t seed, uint64_t tid, int64_t rows, int64_t cols, int32_t classes,
                              void* dst, uint64_t stream) {
  if (!dst || rows < 0 || cols < 0 || kind < 0 || kind > 2) return fail(TPS_E_INVALID_ARG, "bad fill arguments");
  if (kind == 2 && classes < 1) return fail(TPS_E_INVALID_ARG, "classes must be >= 1");
  int dev = 0;
  CUDA_OK(cudaGetDevice(&dev));
  TPS_TRY(check_arch(dev));
  CUDA_OK(tps::launch_fill_synthetic(kind, seed, tid, rows, cols, cols, classes, 0, dst,
                                     reinterpret_cast<cudaStream_t>(stream)));
  return TPS_OK;
}

tps_status tps_partition(int32_t L, const double* pb, const double* ab, const double* fl, int32_t S, int32_t variant,
                         int32_t momentum, int32_t objective, int32_t* bounds, double* cost_out) {
  if (L < 1 || S < 1 || S > L || !bounds) return fail(TPS_E_INVALID_ARG, "need 1 <= S <= L and an output array");
  if (objective == 0 && (!pb || !ab)) return fail(TPS_E_INVALID_ARG, "memory objective needs param/act bytes");
  if (objective == 1 && !fl) return fail(TPS_E_INVALID_ARG, "time objective needs flops");
  if (objective != 0 && objective != 1) return fail(TPS_E_INVALID_ARG, "bad objective");
  // cost(s, i, j): cost of stage s holding layers [i, j)
  std::vector<double> P(L + 1, 0.0), A(L + 1, 0.0), F(L + 1, 0.0);
  for (int l = 0; l < L; ++l) {
    P[l + 1] = P[l] + (pb ? pb[l] : 0.0);
    A[l + 1] = A[l] + (ab ? ab[l] : 0.0);
    F[l + 1] = F[l] + (fl ? fl[l] : 0.0);
  }
  auto cost = [&](int s, int i, int j) {
    if (objective == 1) return F[j] - F[i];
    const double K = static_cast<double>(S - s);
    const double R = variant == TPS_I ? K : 1.0;
    return (P[j] - P[i]) * (1.0 + (momentum ? 1.0 : 0.0) + 0.5 * R) + K * (A[j] - A[i]);
  };
  const double INF = 1e300;
  // best[s][j]: minimal max-cost of placing layers [0, j) on stages 0..s-1
  std::vector<std::vector<double>> best(S + 1, std::vector<double>(L + 1, INF));
  std::vector<std::vector<int>> arg(S + 1, std::vector<int>(L + 1, -1));
  best[0][0] = 0.0;
  for (int s = 1; s <= S; ++s)
    for (int j = s; j <= L - (S - s); ++j)
      for (int i = s - 1; i < j; ++i) {
        if (best[s - 1][i] >= INF) continue;
        const double c = std::max(best[s - 1][i], cost(s - 1, i, j));
        if (c < best[s][j]) {
          best[s][j] = c;
          arg[s][j] = i;
        }
      }
  int j = L;
  bounds[S] = L;
  for (int s = S; s >= 1; --s) {
    const int i = arg[s][j];
    bounds[s - 1] = i;
    if (cost_out) cost_out[s - 1] = cost(s - 1, i, j);
    j = i;
  }
  return TPS_OK;
}

namespace {
// raw GEMM entry points: a stream-ordered split-K workspace when the shape splits
tps_status gemm_with_ws(int mode, const tps::GemmOperands& op, tps::GemmArgs ga, cudaStream_t st) {
  const int64_t wsf = ga.out_f32 ? tps::gemm_splitk_floats(mode, ga.M, ga.N, ga.K, ga.ldo) : 0;
  void* ws = nullptr;
  if (wsf > 0) CUDA_OK(cudaMallocAsync(&ws, static_cast<size_t>(wsf) * 4, st));
  ga.ws = static_cast<float*>(ws);
  ga.ws_floats = wsf;
  const cudaError_t e = tps::gemm_run(mode, op, ga, st);
  if (ws) CUDA_OK(cudaFreeAsync(ws, st));
  CUDA_OK(e);
  return TPS_OK;
}

tps_status op_prologue() {
  int dev = 0;
  CUDA_OK(cudaGetDevice(&dev));
  return check_arch(dev);
}
}  // namespace

tps_status tps_conv2d_gemm(int32_t mode, int32_t N, int32_t H, int32_t W, int32_t Ci, int32_t Co, int32_t k,
                           int32_t stride, int32_t pad, const void* A, const void* Wt, const void* W2, void* out,
                           int32_t out_f32, float alpha, float beta, uint64_t stream) {
  if (mode < 0 || mode > 3 || N < 1 || H < 1 || W < 1 || k < 1 || stride < 1 || stride > 8 || pad < 0 || !A || !Wt ||
      !out)
    return fail(TPS_E_INVALID_ARG, "bad conv operands");
  if (Ci % 64 || Co % 64) return fail(TPS_E_INVALID_ARG, "Ci and Co must be multiples of 64");
  if ((mode == 1 || mode == 3) && (k != 3 || stride != 1 || pad != 1)) return fail(TPS_E_INVALID_ARG, "dgrad: 3x3/1/1 only");
  if (mode == 3 && !W2) return fail(TPS_E_INVALID_ARG, "blend mode needs W2");
  const int Ho = (H + 2 * pad - k) / stride + 1, Wo = (W + 2 * pad - k) / stride + 1;
  if (Ho < 1 || Wo < 1) return fail(TPS_E_INVALID_ARG, "empty conv output");
  TPS_TRY(op_prologue());
  tps::GemmOperands op{};
  tps::GemmArgs ga{};
  ga.out = out; ga.out_f32 = out_f32; ga.alpha = 1.f; ga.xa = 1.f; ga.xb = 0.f;
  int gm;
  if (mode == 0) {
    op = tps::GemmOperands{A, 0, Wt, k * k * Ci, nullptr};
    op.cv = tps::ConvGeom{N, H, W, Ci, 1, k, stride, pad, Ho, Wo};
    ga.M = N * Ho * Wo; ga.N = Co; ga.K = k * k * Ci; ga.ldo = Co;
    gm = tps::GEMM_CONV_FWD;
  } else if (mode == 2) {
    op = tps::GemmOperands{A, Co, Wt, 0, nullptr};
    op.cv = tps::ConvGeom{N, H, W, Ci, 1, k, stride, pad, Ho, Wo};
    ga.M = Co; ga.N = k * k * Ci; ga.K = N * Ho * Wo; ga.ldo = k * k * Ci; ga.out_f32 = 1;
    gm = tps::GEMM_CONV_WGRAD;
  } else {
    op = tps::GemmOperands{A, Co, Wt, 9 * Ci, mode == 3 ? W2 : nullptr};
    op.cv = tps::ConvGeom{N, H, W, Co, 1, 3, 1, 1, H, W};
    op.Cw = Ci;
    ga.M = N * H * W; ga.N = Ci; ga.K = 9 * Co; ga.ldo = Ci;
    if (mode == 3) { ga.xa = alpha; ga.xb = beta; } else { ga.alpha = alpha; }
    gm = mode == 3 ? tps::GEMM_CONV_DGRAD_BLEND : tps::GEMM_CONV_DGRAD;
  }
  return gemm_with_ws(gm, op, ga, reinterpret_cast<cudaStream_t>(stream));
}

tps_status tps_conv_gemm(int32_t mode, int32_t N, int32_t H, int32_t W, int32_t Ci, int32_t Co, const void* A,
                         const void* Wt, const void* W2, void* out, int32_t out_f32, const float* bias, int32_t relu,
                         float alpha, float beta, const void* mask, uint64_t stream) {
  if (mode < 0 || mode > 3 || N < 1 || H < 1 || W < 1 || !A || !Wt || !out) return fail(TPS_E_INVALID_ARG, "bad conv operands");
  if (Ci % 64 || Co % 64) return fail(TPS_E_INVALID_ARG, "Ci and Co must be multiples of 64");
  if (mode == 3 && !W2) return fail(TPS_E_INVALID_ARG, "blend mode needs W2");
  int dev = 0;
  CUDA_OK(cudaGetDevice(&dev));
  TPS_TRY(check_arch(dev));
  const int P = N * H * W;
  tps::GemmOperands op{};
  tps::GemmArgs ga{};
  ga.out = out; ga.out_f32 = out_f32; ga.alpha = 1.f; ga.xa = 1.f; ga.xb = 0.f;
  int gm;
  if (mode == 0) {
    op = tps::GemmOperands{A, 0, Wt, 9 * Ci, nullptr};
    op.cv = tps::ConvGeom{N, H, W, Ci};
    ga.M = P; ga.N = Co; ga.K = 9 * Ci; ga.ldo = Co; ga.bias = bias; ga.relu = relu;
    gm = tps::GEMM_CONV_FWD;
  } else if (mode == 2) {
    op = tps::GemmOperands{A, Co, Wt, 0, nullptr};
    op.cv = tps::ConvGeom{N, H, W, Ci};
    ga.M = Co; ga.N = 9 * Ci; ga.K = P; ga.ldo = 9 * Ci; ga.out_f32 = 1;
    gm = tps::GEMM_CONV_WGRAD;
  } else {
    op = tps::GemmOperands{A, Co, Wt, 9 * Ci, mode == 3 ? W2 : nullptr};
    op.cv = tps::ConvGeom{N, H, W, Co};
    op.Cw = Ci;
    ga.M = P; ga.N = Ci; ga.K = 9 * Co; ga.ldo = Ci;
    ga.mask = static_cast<const uint16_t*>(mask); ga.ldm = Ci;
    if (mode == 3) { ga.xa = alpha; ga.xb = beta; } else { ga.alpha = alpha; }
    gm = mode == 3 ? tps::GEMM_CONV_DGRAD_BLEND : tps::GEMM_CONV_DGRAD;
  }
  return gemm_with_ws(gm, op, ga, reinterpret_cast<cudaStream_t>(stream));
}


tps_status tps_im2col(const void* X, void* P, int32_t N, int32_t H, int32_t W, int32_t C, int32_t k, int32_t stride,
                      int32_t pad, int32_t ldp, uint64_t stream) {
  if (!X || !P || N < 1 || H < 1 || W < 1 || C < 1 || k < 1 || stride < 1 || pad < 0 || ldp < k * k * C)
    return fail(TPS_E_INVALID_ARG, "bad im2col arguments");
  TPS_TRY(op_prologue());
  CUDA_OK(tps::launch_im2col(static_cast<const uint16_t*>(X), static_cast<uint16_t*>(P), N, H, W, C, k, stride, pad,
                             ldp, reinterpret_cast<cudaStream_t>(stream)));
  return TPS_OK;
}

tps_status tps_col2im(const float* dP, void* dX, const void* add, int32_t N, int32_t H, int32_t W, int32_t C,
                      int32_t k, int32_t stride, int32_t pad, int32_t ldp, uint64_t stream) {
  if (!dP || !dX || N < 1 || H < 1 || W < 1 || C < 1 || k < 1 || stride < 1 || pad < 0 || ldp < k * k * C)
    return fail(TPS_E_INVALID_ARG, "bad col2im arguments");
  TPS_TRY(op_prologue());
  CUDA_OK(tps::launch_col2im(dP, static_cast<uint16_t*>(dX), static_cast<const uint16_t*>(add), N, H, W, C, k, stride,
                             pad, ldp, reinterpret_cast<cudaStream_t>(stream)));
  return TPS_OK;
}

tps_status tps_bn_forward(const void* x, const void* res, void* y, const float* gamma, const float* beta, float* mean,
                          float* invstd, int32_t segs, int32_t seg_rows, int32_t C, int32_t relu, uint64_t stream) {
  if (!x || !y || !gamma || !beta || !mean || !invstd || segs < 1 || seg_rows < 1 || C < 1)
    return fail(TPS_E_INVALID_ARG, "bad bn_forward arguments");
  TPS_TRY(op_prologue());
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  void* scr = nullptr;
  CUDA_OK(cudaMallocAsync(&scr, sizeof(double) * tps::bn_scratch_doubles(segs, seg_rows, C), st));
  const cudaError_t e = tps::launch_bn_forward(static_cast<const uint16_t*>(x), static_cast<const uint16_t*>(res),
                                               static_cast<uint16_t*>(y), gamma, beta, mean, invstd, segs, seg_rows, C,
                                               relu, static_cast<double*>(scr), st);
  CUDA_OK(cudaFreeAsync(scr, st));
  CUDA_OK(e);
  return TPS_OK;
}

tps_status tps_bn_backward(const void* dy, const void* y, const void* x, const float* mean, const float* invstd,
                           const float* gamma_stash, const float* gamma_latest, float a, float b, int32_t segs,
                           int32_t seg_rows, int32_t C, int32_t relu, void* dx, void* dres, float* dgamma,
                           float* dbeta, uint64_t stream) {
  if (!dy || !y || !x || !mean || !invstd || !gamma_stash || !gamma_latest || !dx || !dgamma || !dbeta || segs < 1 ||
      seg_rows < 1 || C < 1)
    return fail(TPS_E_INVALID_ARG, "bad bn_backward arguments");
  TPS_TRY(op_prologue());
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  void* scr = nullptr;
  CUDA_OK(cudaMallocAsync(&scr, sizeof(double) * tps::bn_scratch_doubles(segs, seg_rows, C), st));
  const cudaError_t e = tps::launch_bn_backward(
      static_cast<const uint16_t*>(dy), static_cast<const uint16_t*>(y), static_cast<const uint16_t*>(x), mean, invstd,
      gamma_stash, gamma_latest, a, b, segs, seg_rows, C, relu, static_cast<uint16_t*>(dx),
      static_cast<uint16_t*>(dres), dgamma, dbeta, static_cast<double*>(scr), st);
  CUDA_OK(cudaFreeAsync(scr, st));
  CUDA_OK(e);
  return TPS_OK;
}

tps_status tps_pool_op(int32_t op, const void* a, const void* b, void* out, int32_t N, int32_t H, int32_t W, int32_t C,
                       uint64_t stream) {
  if (op < 0 || op > 5 || !out || N < 1 || H < 1 || W < 1 || C < 1) return fail(TPS_E_INVALID_ARG, "bad pool arguments");
  if ((op != 3 && !a) || (op != 0 && op != 2 && !b)) return fail(TPS_E_INVALID_ARG, "missing pool operand");
  if (op >= 4 && C % 8) return fail(TPS_E_INVALID_ARG, "recorded-tap max pool needs C %% 8 == 0");
  TPS_TRY(op_prologue());
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const uint16_t* A = static_cast<const uint16_t*>(a);
  const uint16_t* Bp = static_cast<const uint16_t*>(b);
  uint16_t* O = static_cast<uint16_t*>(out);
  if (op == 0) CUDA_OK(tps::launch_maxpool3_fwd(A, O, N, H, W, C, st));
  else if (op == 1) CUDA_OK(tps::launch_maxpool3_bwd(A, Bp, O, N, H, W, C, st));
  else if (op == 2) CUDA_OK(tps::launch_avgpool_fwd(A, O, N, H * W, C, st));
  else if (op == 3) CUDA_OK(tps::launch_avgpool_bwd(Bp, O, N, H * W, C, st));
  else if (op == 4) CUDA_OK(tps::launch_maxpool3_fwd_idx(A, O, static_cast<uint8_t*>(const_cast<void*>(b)), N, H, W, C, st));
  else CUDA_OK(tps::launch_maxpool3_bwd_idx(static_cast<const uint8_t*>(a), Bp, O, N, H, W, C, st));
  return TPS_OK;
}

tps_status tps_gemm_wgrad_sgd(int32_t M, int32_t N, int32_t K, const void* A, int32_t lda, const void* B, int32_t ldb,
                              float* w, float* v, void* ver, int32_t ldw, float lr, float mu, float wd,
                              uint64_t stream) {
  if (M < 1 || N < 1 || K < 1 || !A || !B || !w || !ver || (mu != 0.f && !v)) return fail(TPS_E_INVALID_ARG, "bad operands");
  if (N % 8 || lda % 8 || ldb % 8 || ldw % 8) return fail(TPS_E_INVALID_ARG, "N and leading dims must be multiples of 8");
  TPS_TRY(op_prologue());
  tps::GemmOperands op{A, lda, B, ldb, nullptr};
  tps::GemmArgs ga{};
  ga.M = M; ga.N = N; ga.K = K; ga.ldo = ldw; ga.out_f32 = 1; ga.alpha = 1.f; ga.xa = 1.f;
  ga.epi = tps::EPI_SGD; ga.w = w; ga.v = v; ga.ver = static_cast<uint16_t*>(ver);
  ga.lr = lr; ga.mu = mu; ga.wd = wd;
  CUDA_OK(tps::gemm_run(tps::GEMM_WGRAD, op, ga, reinterpret_cast<cudaStream_t>(stream)));
  return TPS_OK;
}

tps_status tps_gemm_bwd_dual(int32_t M, int32_t N, int32_t K, const void* A, int32_t lda, const void* B, int32_t ldb,
                             float* w, float* v, void* ver, int32_t ldw, float lr, float mu, float wd, int32_t Md,
                             int32_t Nd, int32_t Kd, const void* Ad, int32_t ldad, const void* Bd, int32_t ldbd,
                             void* outd, int32_t ldod, float alpha, const void* mask, int32_t ldm, uint64_t stream) {
  if (M < 1 || N < 1 || K < 1 || !A || !B || !w || !ver || (mu != 0.f && !v)) return fail(TPS_E_INVALID_ARG, "bad operands");
  if (Md < 1 || Nd < 1 || Kd < 1 || !Ad || !Bd || !outd) return fail(TPS_E_INVALID_ARG, "bad input-gradient operands");
  if (N % 8 || lda % 8 || ldb % 8 || ldw % 8 || Nd % 8 || ldad % 8 || ldbd % 8 || ldod % 8 || (mask && ldm % 8))
    return fail(TPS_E_INVALID_ARG, "N and leading dims must be multiples of 8");
  TPS_TRY(op_prologue());
  tps::GemmOperands opw{A, lda, B, ldb, nullptr};
  tps::GemmArgs ga{};
  ga.M = M; ga.N = N; ga.K = K; ga.ldo = ldw; ga.out_f32 = 1; ga.alpha = 1.f; ga.xa = 1.f;
  ga.epi = tps::EPI_SGD; ga.w = w; ga.v = v; ga.ver = static_cast<uint16_t*>(ver);
  ga.lr = lr; ga.mu = mu; ga.wd = wd;
  tps::GemmOperands opd{Ad, ldad, Bd, ldbd, nullptr};
  tps::DualArgs dg{Md, Nd, Kd, alpha, outd, ldod, static_cast<const uint16_t*>(mask), ldm};
  const cudaError_t e = tps::gemm_bwd_dual(opw, ga, opd, dg, reinterpret_cast<cudaStream_t>(stream));
  if (e == cudaErrorNotSupported) return fail(TPS_E_UNSUPPORTED, "shapes unsuited to the dual launch");
  CUDA_OK(e);
  return TPS_OK;
}

tps_status tps_gemm(int32_t mode, int32_t M, int32_t N, int32_t K, const void* A, int32_t lda, const void* B,
                    int32_t ldb, const void* B2, void* out, int32_t ldo, int32_t out_f32, const float* bias,
                    int32_t relu, float alpha, float beta, const void* mask, int32_t ldm, uint64_t stream) {
  const int tf = (mode & TPS_GEMM_TF32) != 0;
  mode &= ~TPS_GEMM_TF32;
  if (mode < 0 || mode > 3) return fail(TPS_E_INVALID_ARG, "bad mode");
  if (M < 0 || N < 0 || K < 0 || !A || !B || !out) return fail(TPS_E_INVALID_ARG, "bad operands");
  if (N % 8 || ldo % 8 || lda % 8 || ldb % 8 || (mask && ldm % 8)) return fail(TPS_E_INVALID_ARG, "N and leading dims must be multiples of 8");
  if (mode == 3 && !B2) return fail(TPS_E_INVALID_ARG, "blend mode needs B2");
  int dev = 0;
  CUDA_OK(cudaGetDevice(&dev));
  TPS_TRY(check_arch(dev));
  tps::GemmOperands op{A, lda, B, ldb, B2};
  tps::GemmArgs ga{};
  ga.M = M; ga.N = N; ga.K = K; ga.out = out; ga.ldo = ldo; ga.out_f32 = out_f32; ga.bias = bias; ga.relu = relu;
  ga.alpha = mode == 3 ? 1.f : alpha; ga.xa = alpha; ga.xb = beta;
  ga.mask = static_cast<const uint16_t*>(mask); ga.ldm = ldm;
  ga.tf32 = tf;
  return gemm_with_ws(mode, op, ga, reinterpret_cast<cudaStream_t>(stream));
}

}  // extern "C"

// gemm.h — host interface of the sm_100a stage GEMM (gemm_sm100.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace tps {

enum GemmMode {
  GEMM_FWD = 0, GEMM_DGRAD = 1, GEMM_WGRAD = 2, GEMM_DGRAD_BLEND = 3,
  // 3x3 / stride 1 / pad 1 convolutions as implicit GEMMs over NHWC tensors (4-D TMA boxes)
  GEMM_CONV_FWD = 4,          // Y[NHW, Co]   = im2col(X)[NHW, 9Ci] · W[Co, 9Ci]ᵀ
  GEMM_CONV_DGRAD = 5,        // dX[NHW, Ci]  = im2col(dY)[NHW, 9Co] · flip(W)[9Co, Ci]
  GEMM_CONV_DGRAD_BLEND = 6,  // same, flip(α·W_stash + β·W_latest) formed in shared memory
  GEMM_CONV_WGRAD = 7         // dW[Co, 9Ci]  = dY[NHW, Co]ᵀ · im2col(X)[NHW, 9Ci]
};
enum ConvKind { CONV_NONE = 0, CONV_FWD = 1, CONV_DGRAD = 2, CONV_WGRAD = 3 };

// geometry of the gathered NHWC tensor (stride 1, pad 1, 3x3): fwd: X (C = Ci);
// dgrad: dY (C = Co, also the K blocks of the flipped weight); wgrad: X (C = Ci).
struct ConvGeom {
  int N, H, W, C;
  // im2col != 0: the activation operand is read with TMA im2col-mode loads (any H, W; k x k
  // filter, stride s, zero padding p; output Ho x Wo) instead of whole-row pixel boxes
  int im2col, k, s, p, Ho, Wo;
};

struct GemmOperands {
  const void* A;  int lda;    // bf16
  const void* B;  int ldb;    // bf16
  const void* B2;             // bf16, BLEND only (the latest weight; same ld as B)
  ConvGeom cv;                // conv modes only
  int Cw;                     // conv dgrad: Ci of the weight [Co,3,3,Ci] (the GEMM N)
};

// Passed by value to the kernel.
struct GemmArgs {
  int M, N, K;
  void* out; int ldo; int out_f32;
  const float* bias; int relu;
  float alpha;                // epilogue scale (EQ1 α), 1 = none
  float xa, xb;               // BLEND operand coefficients
  const uint16_t* mask; int ldm;  // bf16 ReLU mask source (zero where <= 0), may be null
  const uint16_t* addend;     // bf16 [M, N] (ld = ldo) added before the bf16 store (gradient
                              // accumulation of a tensor with two consumers); may alias out
  // EPI_SGD (wgrad only): instead of storing dW, apply the PyTorch-order SGD/momentum update
  // to the fp32 master w / momentum v ([M, N], ld = ldo) and write bf16(w) to ver.
  int epi;
  float* w; float* v; uint16_t* ver;
  float lr, mu, wd;
  ConvGeom cv;                // copied from GemmOperands by gemm_run
  // split-K (weight gradients whose output tiles cannot fill the GPU): fp32 workspace of
  // ws_floats floats supplied by the caller; gemm_run sets splits / kper and reduces
  float* ws; int64_t ws_floats;
  int splits, kper;           // set by gemm_run
  // SMs this launch may occupy (0 = all).  The split backward runs layer k's fused wgrad +
  // update and layer k-1's input gradient CONCURRENTLY on two streams; capping both persistent
  // grids partitions the SMs between them so they co-run instead of queueing for SMs.
  int max_ctas;
  // column sums of the stored output (plain epilogue, no split-K): colsum[g·N + n] = Σ over rows
  // [32g, 32g+32) of out[·, n] (g < ceil(M/32)); with colsum_sq the Σx² plane follows at
  // colsum + ceil(M/32)·N.  Fed to the bias gradient of the next layer down and to batch-norm
  // statistics without another pass over the tensor.  Null = off.
  float* colsum; int colsum_sq;
  // tf32 storage (reading Z28): A, B (and B2, mask, a non-fp32 out, the fused update's version)
  // are fp32 arrays holding tf32 values, MMAs run kind::tf32, stores round RNA to tf32.
  // Linear modes only (GEMM_FWD / DGRAD / WGRAD / DGRAD_BLEND), no addend, no split-K.
  int tf32;
  // fused update (EPI_SGD) on 256-column CTA-pair tiles: split a last partial wave of tiles into
  // half tiles so no pair runs one whole HBM-bound update epilogue more than the others (set by
  // gemm_run: on unless TPS_SGD_SPLIT_TAIL=0)
  int split_tail;
};

// The input-gradient half of a dual backward launch (gemm_bwd_dual): dX[M, N] = α·(G·W)
// ⊙ 1[mask > 0], G [M, K] K-major (op.A, lda), W stored [K, N] (op.B, ldb), bf16 out.
struct DualArgs {
  int M, N, K;
  float alpha;
  void* out; int ldo;
  const uint16_t* mask; int ldm;
};

// One persistent launch computing layer k's weight gradient with the fused SGD/momentum update
// (opw / aw as gemm_run's GEMM_WGRAD with epi = EPI_SGD) AND layer k-1's input gradient (opd /
// dg as GEMM_DGRAD without blend): every CTA pair interleaves tiles of both, so the tensor
// pipe runs the input gradient's MMAs while the update epilogue streams w / v through HBM.
// Results are bit-identical to the two separate launches.  cudaErrorNotSupported when the
// shapes do not suit it (the caller then launches the two separately).
cudaError_t gemm_bwd_dual(const GemmOperands& opw, const GemmArgs& aw, const GemmOperands& opd, const DualArgs& dg,
                          cudaStream_t st);

// floats of split-K workspace gemm_run needs for this weight-gradient GEMM (0: no split)
int64_t gemm_splitk_floats(int mode, int M, int N, int K, int ldo);

enum GemmEpilogue { EPI_STORE = 0, EPI_SGD = 1 };

// whether the implicit-im2col conv modes (4-D TMA pixel boxes of whole image rows) support an
// H x W activation: 128- and 64-pixel tiles must be whole rows of one image or whole images
bool conv_implicit_ok(int H, int W);

cudaError_t gemm_run(int mode, const GemmOperands& op, const GemmArgs& args, cudaStream_t st, int* bn_out = nullptr);
const char* gemm_mode_name(int mode);

}  // namespace tps

// kernels.h — launchers of the non-GEMM kernels of the hot path (elementwise.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace tps {

// Fused SGD/momentum update + new bf16 version (row a10):
//   g' = g + wd·w ; v = μ·v + g' ; w = w - lr·v   (fp32, one rounding per op, PyTorch order)
//   ver = bf16_rne(w)  (skipped if ver == nullptr).  μ == 0 => v untouched (14 B/param).
// blocks_per_sm bounds the grid (a small grid lets the update run underneath a persistent GEMM).
// tf = 1: ver is an fp32 array that receives tf32_rna(w) (tf32 storage, reading Z28).
cudaError_t launch_sgd_update(float* w, float* v, const float* g, uint16_t* ver, int64_t n, float lr, float mu,
                              float wd, cudaStream_t st, int blocks_per_sm = 8, int tf = 0);

// Data parallelism (NEXT-2): the gradients of the R replicas of a stage (own + peers' mapped
// buffers), averaged in replica order g = (Σ_r g_r)·(1/R) and applied as launch_sgd_update does.
struct GradList {
  static constexpr int MAX = 8;
  const float* p[MAX];
  int n;
};
cudaError_t launch_sgd_update_dp(float* w, float* v, const GradList& g, uint16_t* ver, int64_t n, float lr, float mu,
                                 float wd, cudaStream_t st);

// db[c] = Σ_{r<rows} G[r, c] for c < cols (G bf16 [rows, ldg]); deterministic two-phase
// reduction using `scratch` (>= bias_grad_scratch_floats(rows, cols) floats).
int64_t bias_grad_scratch_floats(int rows, int cols);
// (tf = 1: G is an fp32 array of tf32 values, reading Z28; same for launch_bias_grad_sgd)
cudaError_t launch_bias_grad(const uint16_t* G, int rows, int cols, int ldg, float* db, float* scratch,
                             cudaStream_t st, int tf = 0);
// The same column sums in ONE launch (the last block of each column block finishes the
// fixed-order reduction; its arrival counters live at the end of `scratch` and reset
// themselves), followed, if b != nullptr, by the SGD/momentum step of launch_sgd_update on the
// fp32 bias b and its momentum vb (same operations, same bits).  Bit-identical db.
cudaError_t launch_bias_grad_sgd(const uint16_t* G, int rows, int cols, int ldg, float* db, float* scratch, float* b,
                                 float* vb, float lr, float mu, float wd, cudaStream_t st, int tf = 0);

// db[c] = Σ_g part[g·cols + c] (the 32-row column sums a GEMM epilogue wrote, GemmArgs.colsum;
// fixed order, fp64 accumulation), then the bias SGD/momentum step if b != nullptr.
cudaError_t launch_bias_from_colsum(const float* part, int groups, int cols, float* db, float* b, float* vb, float lr,
                                   float mu, float wd, cudaStream_t st);

// Softmax cross-entropy forward+backward for `rows` rows of fp32 logits [rows, ldl] with
// `classes` valid columns: loss_rows[r] = logsumexp(z) - z_y ;
// G[r, c] = bf16((softmax(z)_c - [c == y]) / batch) for c < classes, 0 for classes <= c < ldg.
// (tf = 1: G is an fp32 array receiving tf32_rna of the same value)
cudaError_t launch_softmax_xent(const float* logits, int ldl, const int32_t* labels, int rows, int classes,
                                int batch, float* loss_rows, uint16_t* G, int ldg, cudaStream_t st, int tf = 0);

// losses[*ctr] = (Σ_{r<rows} loss_rows[r]) / rows, then ++*ctr  (fixed-order fp64 reduction, one
// block; the device-side slot counter lets a replayed CUDA graph append)
cudaError_t launch_loss_mean(const float* loss_rows, int rows, float* losses, int64_t* ctr, cudaStream_t st);

// fp32 -> bf16 RNE, n elements
cudaError_t launch_f32_to_bf16(const float* in, uint16_t* out, int64_t n, cudaStream_t st);

// fp32 -> tf32 (RNA, fp32 container), n elements
cudaError_t launch_f32_to_tf32(const float* in, float* out, int64_t n, cudaStream_t st);
// K8 debug materialiser in tf32 storage: out = tf32_rna(fp32(α·s) + fp32(β·l))
cudaError_t launch_blend_materialize_tf32(const float* s, const float* l, float* out, int64_t n, float a, float b,
                                         cudaStream_t st);

// K8 debug materialiser: out = bf16(fp32(α·s) + fp32(β·l))
cudaError_t launch_blend_materialize(const uint16_t* s, const uint16_t* l, uint16_t* out, int64_t n, float a,
                                     float b, cudaStream_t st);

// image nets (NHWC bf16): 2x2/stride-2 max pool, its gradient (first maximum of each window,
// reading Z15), and explicit 3x3/pad-1 patches [(n,h,w), (kh,kw,c)] zero-padded to ldp columns.
cudaError_t launch_maxpool2_fwd(const uint16_t* X, uint16_t* Y, int N, int H, int W, int C, cudaStream_t st);
cudaError_t launch_maxpool2_bwd(const uint16_t* X, const uint16_t* dY, uint16_t* dX, int N, int H, int W, int C,
                                cudaStream_t st);
cudaError_t launch_im2col3x3(const uint16_t* X, uint16_t* P, int N, int H, int W, int C, int ldp, cudaStream_t st);

// ResNet (NHWC bf16):
//   general k x k / stride s / pad p patches P[(n,ho,wo), (kh,kw,c)] (zero padded to ldp) and
//   their adjoint (gather form, fp32 patch gradients, optional bf16 addend, bf16 out);
//   batch norm with per-micro-batch statistics over segments of seg_rows rows (biased
//   variance, ε = 1e-5), fused residual add + ReLU; its backward with the blended γ
//   (ga·γ_stash + gb·γ_latest) and the ReLU mask from the stored output;
//   3x3/2/1 max pool (first maximum), global average pool, bf16 accumulate.
cudaError_t launch_im2col(const uint16_t* X, uint16_t* P, int N, int H, int W, int C, int k, int s, int p, int ldp,
                          cudaStream_t st);
cudaError_t launch_col2im(const float* dP, uint16_t* dX, const uint16_t* add, int N, int H, int W, int C, int k, int s,
                          int p, int ldp, cudaStream_t st);
int64_t bn_scratch_doubles(int segs, int seg_rows, int C);
cudaError_t launch_bn_forward(const uint16_t* x, const uint16_t* res, uint16_t* y, const float* gamma,
                              const float* beta, float* mean, float* invstd, int segs, int seg_rows, int C, int relu,
                              double* scratch, cudaStream_t st, uint8_t* relu_mask = nullptr);
// relu_mask (optional, relu && C % 8 == 0): one byte per (row, 8-channel group), bit e = [y_e > 0],
// written by the forward and read by the backward in place of y (0.125 instead of 2 B per element)
// batch-norm forward whose statistics come from the producing convolution's epilogue column sums
// (GemmArgs.colsum + colsum_sq over the same rows: Σx plane, then Σx² plane; seg_rows % 32 == 0):
// same mean / invstd / y as launch_bn_forward up to the fp32 rounding of the 32-row partials
cudaError_t launch_bn_forward_colsum(const float* part, const uint16_t* x, const uint16_t* res, uint16_t* y,
                                    const float* gamma, const float* beta, float* mean, float* invstd, int segs,
                                    int seg_rows, int C, int relu, double* scratch, cudaStream_t st,
                                    uint8_t* relu_mask = nullptr);
cudaError_t launch_bn_backward(const uint16_t* dy, const uint16_t* y, const uint16_t* x, const float* mean,
                               const float* invstd, const float* gs, const float* gl, float ga, float gb, int segs,
                               int seg_rows, int C, int relu, uint16_t* dx, uint16_t* dres, float* dgamma,
                               float* dbeta, double* scratch, cudaStream_t st, const uint8_t* relu_mask = nullptr);
cudaError_t launch_maxpool3_fwd(const uint16_t* X, uint16_t* Y, int N, int H, int W, int C, cudaStream_t st);
cudaError_t launch_maxpool3_bwd(const uint16_t* X, const uint16_t* dY, uint16_t* dX, int N, int H, int W, int C,
                                cudaStream_t st);
// 3x3/2/1 max pool recording the first-max tap (uint8 [N, Ho, Wo, C]) and its gradient from
// the recorded taps (C % 8 == 0)
cudaError_t launch_maxpool3_fwd_idx(const uint16_t* X, uint16_t* Y, uint8_t* idx, int N, int H, int W, int C,
                                    cudaStream_t st);
cudaError_t launch_maxpool3_bwd_idx(const uint8_t* idx, const uint16_t* dY, uint16_t* dX, int N, int H, int W, int C,
                                    cudaStream_t st);
cudaError_t launch_avgpool_fwd(const uint16_t* X, uint16_t* Y, int N, int HW, int C, cudaStream_t st);
cudaError_t launch_avgpool_bwd(const uint16_t* dY, uint16_t* dX, int N, int HW, int C, cudaStream_t st);
cudaError_t launch_add_bf16(uint16_t* out, const uint16_t* add, int64_t n, cudaStream_t st);

// synthgen-identical counter-based generator (see synthgen/__init__.py)
//   kind 0/1: bf16 inputs into dst[rows, ld] (cols valid); kind 2: int32 labels[rows];
//   kind 3: fp32 weights [rows=out, ld] (cols=in valid), scale 2^-(23 + shift).
cudaError_t launch_fill_synthetic(int kind, uint64_t seed, uint64_t tid, int64_t rows, int64_t cols, int64_t ld,
                                  int classes, int shift, void* dst, cudaStream_t st);

}  // namespace tps

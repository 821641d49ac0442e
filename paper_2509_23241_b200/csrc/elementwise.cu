// elementwise.cu — HBM-bound kernels of the TiMePReSt step: fused SGD/momentum update
// + bf16 version write, bias gradient (a8), softmax
// cross-entropy at the last stage (a4), the K8 blend materialiser, and the
// synthetic-input generator shared with synthgen (counter-based splitmix64).
//
// All kernels use 16-byte vector accesses, grid-stride loops sized to a multiple of the
// SM count, and fixed-order reductions (bit-reproducible run to run).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>

#include "kernels.h"

namespace tps {

namespace {

int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

int grid_for(int64_t work_items, int threads, int per_sm = 8) {
  int64_t g = (work_items + threads - 1) / threads;
  int64_t cap = static_cast<int64_t>(sm_count()) * per_sm;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return static_cast<int>(g);
}

__device__ __forceinline__ uint16_t f2bf(float x) {
  __nv_bfloat16 h = __float2bfloat16_rn(x);
  return *reinterpret_cast<uint16_t*>(&h);
}
__device__ __forceinline__ float bf2f(uint32_t h) { return __uint_as_float(h << 16); }
// tf32 storage (reading Z28): nearest tf32 value, ties away from zero, in an fp32 container
__device__ __forceinline__ float rna_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// ------------------------------------------------------------------ SGD update
template <bool MOMENTUM, bool WRITE_VER, bool TF = false>
__global__ void __launch_bounds__(256) sgd_update_kernel(float* __restrict__ w, float* __restrict__ v,
                                                         const float* __restrict__ g, uint16_t* __restrict__ ver,
                                                         int64_t n4, float lr, float mu, float wd) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float4 wv = reinterpret_cast<float4*>(w)[i];
    const float4 gv = __ldcs(reinterpret_cast<const float4*>(g) + i);
    float ww[4] = {wv.x, wv.y, wv.z, wv.w};
    const float gg[4] = {gv.x, gv.y, gv.z, gv.w};
    float vv[4] = {0.f, 0.f, 0.f, 0.f};
    if (MOMENTUM) {
      const float4 t = reinterpret_cast<float4*>(v)[i];
      vv[0] = t.x; vv[1] = t.y; vv[2] = t.z; vv[3] = t.w;
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float gp = __fadd_rn(gg[e], __fmul_rn(wd, ww[e]));      // g' = g + wd·w
      float upd;
      if (MOMENTUM) {
        vv[e] = __fadd_rn(__fmul_rn(mu, vv[e]), gp);                 // v = μ·v + g'
        upd = vv[e];
      } else {
        upd = gp;                                                     // μ = 0: v = g'
      }
      ww[e] = __fsub_rn(ww[e], __fmul_rn(lr, upd));                  // w = w - lr·v
    }
    reinterpret_cast<float4*>(w)[i] = make_float4(ww[0], ww[1], ww[2], ww[3]);
    if (MOMENTUM) reinterpret_cast<float4*>(v)[i] = make_float4(vv[0], vv[1], vv[2], vv[3]);
    if (WRITE_VER && TF) {   // tf32 version (fp32 container)
      reinterpret_cast<float4*>(ver)[i] =
          make_float4(rna_tf32(ww[0]), rna_tf32(ww[1]), rna_tf32(ww[2]), rna_tf32(ww[3]));
    } else if (WRITE_VER) {
      uint2 o;
      o.x = static_cast<uint32_t>(f2bf(ww[0])) | (static_cast<uint32_t>(f2bf(ww[1])) << 16);
      o.y = static_cast<uint32_t>(f2bf(ww[2])) | (static_cast<uint32_t>(f2bf(ww[3])) << 16);
      reinterpret_cast<uint2*>(ver)[i] = o;
    }
  }
}

// ------------------------------------------------------------------ data-parallel reduce + update
// Pipeline x data parallelism (SURVEY §8(f) NEXT-2, P:75 / P:134): the R replicas of a stage
// hold the gradients of their own mini-batches; one pass reads all R of them (the peers' through
// NVLink peer mappings), averages them in replica order, g = (Σ_r g_r)·(1/R), and applies the
// SGD/momentum step of sgd_update_kernel (same operations, same order) — the all-reduce and the
// update fused, so the averaged gradient is never written.  Every replica computes the same
// sum in the same order, so the replicas' parameters stay bitwise identical.
template <bool MOMENTUM, bool WRITE_VER>
__global__ void __launch_bounds__(256) sgd_update_dp_kernel(float* __restrict__ w, float* __restrict__ v,
                                                            GradList gl, uint16_t* __restrict__ ver, int64_t n4,
                                                            float lr, float mu, float wd) {
  const float inv = 1.0f / static_cast<float>(gl.n);
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float4 gs = __ldcg(reinterpret_cast<const float4*>(gl.p[0]) + i);
    for (int r = 1; r < gl.n; ++r) {
      const float4 t = __ldcg(reinterpret_cast<const float4*>(gl.p[r]) + i);
      gs.x = __fadd_rn(gs.x, t.x); gs.y = __fadd_rn(gs.y, t.y); gs.z = __fadd_rn(gs.z, t.z); gs.w = __fadd_rn(gs.w, t.w);
    }
    const float gg[4] = {__fmul_rn(gs.x, inv), __fmul_rn(gs.y, inv), __fmul_rn(gs.z, inv), __fmul_rn(gs.w, inv)};
    float4 wv = reinterpret_cast<float4*>(w)[i];
    float ww[4] = {wv.x, wv.y, wv.z, wv.w};
    float vv[4] = {0.f, 0.f, 0.f, 0.f};
    if (MOMENTUM) {
      const float4 t = reinterpret_cast<float4*>(v)[i];
      vv[0] = t.x; vv[1] = t.y; vv[2] = t.z; vv[3] = t.w;
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float gp = __fadd_rn(gg[e], __fmul_rn(wd, ww[e]));
      float upd;
      if (MOMENTUM) {
        vv[e] = __fadd_rn(__fmul_rn(mu, vv[e]), gp);
        upd = vv[e];
      } else {
        upd = gp;
      }
      ww[e] = __fsub_rn(ww[e], __fmul_rn(lr, upd));
    }
    reinterpret_cast<float4*>(w)[i] = make_float4(ww[0], ww[1], ww[2], ww[3]);
    if (MOMENTUM) reinterpret_cast<float4*>(v)[i] = make_float4(vv[0], vv[1], vv[2], vv[3]);
    if (WRITE_VER) {
      uint2 o;
      o.x = static_cast<uint32_t>(f2bf(ww[0])) | (static_cast<uint32_t>(f2bf(ww[1])) << 16);
      o.y = static_cast<uint32_t>(f2bf(ww[2])) | (static_cast<uint32_t>(f2bf(ww[3])) << 16);
      reinterpret_cast<uint2*>(ver)[i] = o;
    }
  }
}

// ------------------------------------------------------------------ bias gradient
constexpr int BG_COLS = 256;   // columns per block at most (32 threads x 8 columns)
constexpr int BG_ROWS = 8;     // row lanes per block at the full width
// column threads per block (8 columns each): 32, or the largest power of two <= cols/8 for narrow
// gradients, the other threads becoming row lanes (block = tx x 256/tx).  A 64-column conv bias
// on 32 x 32 images with full-width blocks left 3/4 of the threads idle.
inline int bg_tx(int cols) {
  int tx = 32;
  while (tx > 1 && tx * 8 > cols) tx >>= 1;
  return tx;
}
constexpr int BG_CNT = 64;     // arrival counters at the head of the scratch (cols <= 64·BG_COLS)

template <bool TF>
__global__ void __launch_bounds__(256) bias_grad_partial(const uint16_t* __restrict__ G, int rows, int cols, int ldg,
                                                         int rows_per_split, float* __restrict__ part) {
  __shared__ float red[BG_ROWS * (BG_COLS + 4) + 1024];   // [ty][cbw + 4], ty = 256 / tx
  const int cbw = blockDim.x * 8, ty = blockDim.y, rs = cbw + 4;
  const int c0 = blockIdx.x * cbw + threadIdx.x * 8;
  const int r_begin = blockIdx.y * rows_per_split;
  const int r_end = min(rows, r_begin + rows_per_split);
  float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (c0 < cols) {
    for (int r = r_begin + threadIdx.y; r < r_end; r += ty) {
      if (TF) {   // fp32 (tf32) gradient: two 16-byte loads per 8 columns
        const float4* q =
            reinterpret_cast<const float4*>(reinterpret_cast<const float*>(G) + static_cast<size_t>(r) * ldg + c0);
        const float4 u0 = __ldg(q), u1 = __ldg(q + 1);
        const float f[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] += f[e];
      } else {
        const uint4 u = __ldg(reinterpret_cast<const uint4*>(G + static_cast<size_t>(r) * ldg + c0));
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] += bf2f((w[e >> 1] >> ((e & 1) * 16)) & 0xFFFFu);
      }
    }
  }
#pragma unroll
  for (int e = 0; e < 8; ++e) red[threadIdx.y * rs + threadIdx.x * 8 + e] = acc[e];
  __syncthreads();
  // fixed-order sum over the row lanes
  const int t = threadIdx.y * blockDim.x + threadIdx.x;   // 0..cbw-1 -> one column each
  const int c = blockIdx.x * cbw + t;
  if (t >= cbw) return;
  float s = 0.f;
  for (int y = 0; y < ty; ++y) s += red[y * rs + t];
  if (c < cols) part[static_cast<size_t>(blockIdx.y) * cols + c] = s;
}

// One launch for the bias of a Linear layer (rows a8 + a10): the partial column sums of
// bias_grad_partial, then the LAST block of each column block (arrival counter, self-resetting)
// sums the splits in fixed order (deterministic, same bits as bias_grad_final) and, if b != null,
// applies the SGD/momentum step of sgd_update_kernel to the fp32 bias and its momentum.
template <bool TF>
__global__ void __launch_bounds__(256) bias_grad_fused(const uint16_t* __restrict__ G, int rows, int cols, int ldg,
                                                       int rows_per_split, float* __restrict__ part,
                                                       unsigned int* __restrict__ cnt, float* __restrict__ db,
                                                       float* __restrict__ b, float* __restrict__ vb, float lr,
                                                       float mu, float wd) {
  __shared__ float red[BG_ROWS * (BG_COLS + 4) + 1024];   // [ty][cbw + 4], ty = 256 / tx
  __shared__ bool last;
  const int cbw = blockDim.x * 8, ty = blockDim.y, rs = cbw + 4;
  const int c0 = blockIdx.x * cbw + threadIdx.x * 8;
  const int r_begin = blockIdx.y * rows_per_split;
  const int r_end = min(rows, r_begin + rows_per_split);
  float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (c0 < cols) {
#pragma unroll 8
    for (int r = r_begin + threadIdx.y; r < r_end; r += ty) {   // unrolled: loads in flight, same add order
      if (TF) {   // fp32 (tf32) gradient: two 16-byte loads per 8 columns
        const float4* q =
            reinterpret_cast<const float4*>(reinterpret_cast<const float*>(G) + static_cast<size_t>(r) * ldg + c0);
        const float4 u0 = __ldg(q), u1 = __ldg(q + 1);
        const float f[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] += f[e];
      } else {
        const uint4 u = __ldg(reinterpret_cast<const uint4*>(G + static_cast<size_t>(r) * ldg + c0));
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] += bf2f((w[e >> 1] >> ((e & 1) * 16)) & 0xFFFFu);
      }
    }
  }
#pragma unroll
  for (int e = 0; e < 8; ++e) red[threadIdx.y * rs + threadIdx.x * 8 + e] = acc[e];
  __syncthreads();
  const int t = threadIdx.y * blockDim.x + threadIdx.x;   // 0..cbw-1 -> one column each
  const int c = blockIdx.x * cbw + t;
  if (t < cbw) {
    float s = 0.f;
    for (int y = 0; y < ty; ++y) s += red[y * rs + t];
    if (c < cols) part[static_cast<size_t>(blockIdx.y) * cols + c] = s;
  }
  __threadfence();
  __syncthreads();
  if (t == 0) last = atomicAdd(&cnt[blockIdx.x], 1u) == gridDim.y - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (t == 0) cnt[blockIdx.x] = 0u;               // ready for the next launch (stream-ordered)
  if (t >= cbw || c >= cols) return;
  float d = 0.f;
#pragma unroll 8
  for (int k = 0; k < static_cast<int>(gridDim.y); ++k) d += __ldcg(part + static_cast<size_t>(k) * cols + c);
  db[c] = d;
  if (!b) return;
  float w = b[c];
  const float gp = __fadd_rn(d, __fmul_rn(wd, w));
  float upd = gp;
  if (mu != 0.f) {
    const float v = __fadd_rn(__fmul_rn(mu, vb[c]), gp);
    vb[c] = v;
    upd = v;
  }
  b[c] = __fsub_rn(w, __fmul_rn(lr, upd));
}

// bias gradient from the column partial sums a GEMM epilogue wrote (GemmArgs.colsum: one row of
// 32-row sums per row group): db[c] = Σ_g part[g·cols + c] in fixed order (fp64 accumulation,
// rounded once), then, if b != null, the bias's SGD/momentum step (same operations as
// sgd_update_kernel).  Replaces a full pass over the activation gradient.
__global__ void __launch_bounds__(256) bias_from_colsum_kernel(const float* __restrict__ part, int groups, int cols,
                                                               float* __restrict__ db, float* __restrict__ b,
                                                               float* __restrict__ vb, float lr, float mu, float wd) {
  // block = 32 columns x 8 row lanes; lane ly sums groups ly, ly+8, ... (independent loads in
  // flight), then the 8 lane sums are added in fixed order: deterministic
  __shared__ double red[8][33];
  const int lx = threadIdx.x & 31, ly = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + lx;
  double acc = 0.0;
  if (c < cols) {
#pragma unroll 4
    for (int g = ly; g < groups; g += 8) acc += __ldcg(part + static_cast<size_t>(g) * cols + c);
  }
  red[ly][lx] = acc;
  __syncthreads();
  if (ly != 0 || c >= cols) return;
  double t = 0.0;
#pragma unroll
  for (int y = 0; y < 8; ++y) t += red[y][lx];
  const float d = static_cast<float>(t);
  db[c] = d;
  if (!b) return;
  const float w = b[c];
  const float gp = __fadd_rn(d, __fmul_rn(wd, w));
  float upd = gp;
  if (mu != 0.f) {
    const float v = __fadd_rn(__fmul_rn(mu, vb[c]), gp);
    vb[c] = v;
    upd = v;
  }
  b[c] = __fsub_rn(w, __fmul_rn(lr, upd));
}

__global__ void bias_grad_final(const float* __restrict__ part, int splits, int cols, float* __restrict__ db) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cols) return;
  float s = 0.f;
  for (int k = 0; k < splits; ++k) s += part[static_cast<size_t>(k) * cols + c];
  db[c] = s;
}

int bias_grad_splits(int rows, int cols) {
  // blocks per SM of the column-sum pass (TPS_BG_WAVES, default 2) and at least
  // TPS_BG_MIN_ROWS rows per split (default 64); read once, so the scratch sized at init fits
  static const int waves = std::getenv("TPS_BG_WAVES") ? std::max(1, std::atoi(std::getenv("TPS_BG_WAVES"))) : 2;
  static const int min_rows =
      std::getenv("TPS_BG_MIN_ROWS") ? std::max(8, std::atoi(std::getenv("TPS_BG_MIN_ROWS"))) : 64;
  const int cbw = bg_tx(cols) * 8;
  const int col_blocks = (cols + cbw - 1) / cbw;
  int splits = (waves * sm_count() + col_blocks - 1) / col_blocks;
  const int max_splits = (rows + min_rows - 1) / min_rows;
  if (splits > max_splits) splits = max_splits;
  if (splits < 1) splits = 1;
  return splits;
}

// ------------------------------------------------------------------ softmax cross-entropy
template <bool TF>
__global__ void __launch_bounds__(256) softmax_xent_kernel(const float* __restrict__ logits, int ldl,
                                                           const int32_t* __restrict__ labels, int rows, int classes,
                                                           int batch, float* __restrict__ loss_rows,
                                                           uint16_t* __restrict__ G, int ldg) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= rows) return;
  const float* z = logits + static_cast<size_t>(warp) * ldl;
  double mx = -1e300;
  for (int c = lane; c < classes; c += 32) mx = fmax(mx, static_cast<double>(z[c]));
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  double se = 0.0;
  for (int c = lane; c < classes; c += 32) se += exp(static_cast<double>(z[c]) - mx);
#pragma unroll
  for (int o = 16; o; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
  const int y = labels[warp];
  if (lane == 0) loss_rows[warp] = static_cast<float>(mx + log(se) - static_cast<double>(z[y]));
  for (int c = lane; c < ldg; c += 32) {
    float out = 0.f;
    if (c < classes) {
      double p = exp(static_cast<double>(z[c]) - mx) / se;
      if (c == y) p -= 1.0;
      out = static_cast<float>(p / batch);
    }
    if (TF) reinterpret_cast<float*>(G)[static_cast<size_t>(warp) * ldg + c] = rna_tf32(out);
    else G[static_cast<size_t>(warp) * ldg + c] = f2bf(out);
  }
}

__global__ void loss_mean_kernel(const float* __restrict__ loss_rows, int rows, float* __restrict__ losses,
                                 int64_t* __restrict__ ctr) {
  __shared__ double red[256];
  double s = 0.0;
  for (int r = threadIdx.x; r < rows; r += blockDim.x) s += loss_rows[r];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) {   // the slot index lives on the device so a replayed CUDA graph appends
    const int64_t idx = *ctr;
    losses[idx] = static_cast<float>(red[0] / rows);
    *ctr = idx + 1;
  }
}

// ------------------------------------------------------------------ conversions
__global__ void f32_to_bf16_kernel(const float* __restrict__ in, uint16_t* __restrict__ out, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = f2bf(in[i]);
}

__global__ void f32_to_tf32_kernel(const float* __restrict__ in, float* __restrict__ out, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = rna_tf32(in[i]);
}

__global__ void blend_materialize_tf32_kernel(const float* __restrict__ s, const float* __restrict__ l,
                                              float* __restrict__ out, int64_t n, float a, float b) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = rna_tf32(__fadd_rn(__fmul_rn(a, s[i]), __fmul_rn(b, l[i])));
}

__global__ void blend_materialize_kernel(const uint16_t* __restrict__ s, const uint16_t* __restrict__ l,
                                         uint16_t* __restrict__ out, int64_t n, float a, float b) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = f2bf(__fadd_rn(__fmul_rn(a, bf2f(s[i])), __fmul_rn(b, bf2f(l[i]))));
}

// ------------------------------------------------------------------ synthetic generator
__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void fill_synthetic_kernel(int kind, uint64_t key, int64_t rows, int64_t cols, int64_t ld, int classes,
                                      int shift, void* dst) {
  const int64_t n = (kind == 2) ? rows : rows * ld;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (kind == 2) {
      const uint64_t h = mix64(static_cast<uint64_t>(i) ^ key);
      reinterpret_cast<int32_t*>(dst)[i] = static_cast<int32_t>((h >> 8) % static_cast<uint64_t>(classes));
      continue;
    }
    const int64_t r = i / ld, c = i - r * ld;
    if (c >= cols) {
      if (kind == 3) reinterpret_cast<float*>(dst)[i] = 0.f;
      else reinterpret_cast<uint16_t*>(dst)[i] = 0;
      continue;
    }
    const uint64_t h = mix64(static_cast<uint64_t>(r * cols + c) ^ key);
    if (kind == 3) {
      const int64_t mant = static_cast<int64_t>(h >> 40) - (1ll << 23);
      reinterpret_cast<float*>(dst)[i] = static_cast<float>(ldexp(static_cast<double>(mant), -23 - shift));
    } else {
      const float b = static_cast<float>(h & 0xFFull);
      const float x = (kind == 0) ? (b - 128.0f) * (1.0f / 128.0f) : b * (1.0f / 256.0f);
      reinterpret_cast<uint16_t*>(dst)[i] = f2bf(x);
    }
  }
}

// ------------------------------------------------------------------ image-net helpers (NHWC, bf16)
// 2x2/stride-2 max pool; 8 channels (16 B) per thread
__global__ void maxpool2_fwd_kernel(const uint16_t* __restrict__ X, uint16_t* __restrict__ Y, int N, int H, int W,
                                    int C) {
  const int C8 = C / 8, Ho = H / 2, Wo = W / 2;
  const int64_t total = static_cast<int64_t>(N) * Ho * Wo * C8;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int c8 = static_cast<int>(i % C8);
    int64_t t = i / C8;
    const int wo = static_cast<int>(t % Wo);
    t /= Wo;
    const int ho = static_cast<int>(t % Ho);
    const int64_t n = t / Ho;
    const uint16_t* base = X + ((n * H + 2 * ho) * W + 2 * wo) * C + c8 * 8;
    uint4 q[4];
    q[0] = __ldg(reinterpret_cast<const uint4*>(base));
    q[1] = __ldg(reinterpret_cast<const uint4*>(base + C));
    q[2] = __ldg(reinterpret_cast<const uint4*>(base + static_cast<size_t>(W) * C));
    q[3] = __ldg(reinterpret_cast<const uint4*>(base + static_cast<size_t>(W) * C + C));
    uint32_t out[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      uint32_t packed = 0;
#pragma unroll
      for (int h2 = 0; h2 < 2; ++h2) {
        float best = -INFINITY;
        uint32_t bits = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t word = (&q[k].x)[e];
          const uint32_t hb = (word >> (16 * h2)) & 0xFFFFu;
          const float v = bf2f(hb);
          if (k == 0 || v > best) { best = v; bits = hb; }
        }
        packed |= bits << (16 * h2);
      }
      out[e] = packed;
    }
    reinterpret_cast<uint4*>(Y)[i] = make_uint4(out[0], out[1], out[2], out[3]);
  }
}

// gradient of the 2x2 max pool: dY goes to the FIRST maximum of the window in row-major
// order (reading Z15); the other three positions get 0.  Each thread owns one window x 8 ch.
__global__ void maxpool2_bwd_kernel(const uint16_t* __restrict__ X, const uint16_t* __restrict__ dY,
                                    uint16_t* __restrict__ dX, int N, int H, int W, int C) {
  const int C8 = C / 8, Ho = H / 2, Wo = W / 2;
  const int64_t total = static_cast<int64_t>(N) * Ho * Wo * C8;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int c8 = static_cast<int>(i % C8);
    int64_t t = i / C8;
    const int wo = static_cast<int>(t % Wo);
    t /= Wo;
    const int ho = static_cast<int>(t % Ho);
    const int64_t n = t / Ho;
    const size_t off[4] = {static_cast<size_t>(((n * H + 2 * ho) * W + 2 * wo) * C + c8 * 8),
                           static_cast<size_t>(((n * H + 2 * ho) * W + 2 * wo + 1) * C + c8 * 8),
                           static_cast<size_t>(((n * H + 2 * ho + 1) * W + 2 * wo) * C + c8 * 8),
                           static_cast<size_t>(((n * H + 2 * ho + 1) * W + 2 * wo + 1) * C + c8 * 8)};
    uint4 q[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) q[k] = __ldg(reinterpret_cast<const uint4*>(X + off[k]));
    const uint4 g = __ldg(reinterpret_cast<const uint4*>(dY) + i);
    uint32_t o[4][4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      uint32_t res[4] = {0, 0, 0, 0};
#pragma unroll
      for (int h2 = 0; h2 < 2; ++h2) {
        float best = -INFINITY;
        int arg = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float v = bf2f(((&q[k].x)[e] >> (16 * h2)) & 0xFFFFu);
          if (k == 0 || v > best) { best = v; arg = k; }
        }
        const uint32_t gb = ((&g.x)[e] >> (16 * h2)) & 0xFFFFu;
        res[arg] |= gb << (16 * h2);
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) o[k][e] = res[k];
    }
#pragma unroll
    for (int k = 0; k < 4; ++k)
      *reinterpret_cast<uint4*>(dX + off[k]) = make_uint4(o[k][0], o[k][1], o[k][2], o[k][3]);
  }
}

// explicit 3x3/pad-1 patches for a first layer with few channels: P[(n,h,w), (kh,kw,c)], zero
// padded columns up to ldp
__global__ void im2col3x3_kernel(const uint16_t* __restrict__ X, uint16_t* __restrict__ P, int N, int H, int W,
                                 int C, int ldp) {
  const int64_t total = static_cast<int64_t>(N) * H * W * ldp;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int col = static_cast<int>(i % ldp);
    const int64_t pix = i / ldp;
    uint16_t v = 0;
    if (col < 9 * C) {
      const int khw = col / C, c = col - khw * C;
      const int w = static_cast<int>(pix % W);
      const int64_t t = pix / W;
      const int h = static_cast<int>(t % H);
      const int64_t n = t / H;
      const int hh = h + khw / 3 - 1, ww = w + khw % 3 - 1;
      if (hh >= 0 && hh < H && ww >= 0 && ww < W) v = X[((n * H + hh) * W + ww) * C + c];
    }
    P[i] = v;
  }
}

// ------------------------------------------------------------------ ResNet helpers (NHWC, bf16)
// adjoint of im2col (gather form, fixed (kh, kw) order, fp32 sum of fp32 patch gradients):
// dX[n,h,w,c] = Σ dP[(n,(h+p-kh)/s,(w+p-kw)/s), (kh,kw,c)] over valid (kh, kw); optional bf16 addend
__global__ void col2im_kernel(const float* __restrict__ dP, uint16_t* __restrict__ dX, const uint16_t* __restrict__ add,
                              int N, int H, int W, int C, int k, int s, int p, int Ho, int Wo, int ldp) {
  const int64_t total = static_cast<int64_t>(N) * H * W * C;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(i % C);
    int64_t t = i / C;
    const int w = static_cast<int>(t % W);
    t /= W;
    const int h = static_cast<int>(t % H);
    const int64_t n = t / H;
    float acc = 0.f;
    for (int kh = 0; kh < k; ++kh) {
      const int hy = h + p - kh;
      if (hy < 0 || hy % s) continue;
      const int ho = hy / s;
      if (ho >= Ho) continue;
      for (int kw = 0; kw < k; ++kw) {
        const int wy = w + p - kw;
        if (wy < 0 || wy % s) continue;
        const int wo = wy / s;
        if (wo >= Wo) continue;
        acc += dP[((n * Ho + ho) * Wo + wo) * static_cast<int64_t>(ldp) + (kh * k + kw) * C + c];
      }
    }
    if (add) acc += bf2f(add[i]);
    dX[i] = f2bf(acc);
  }
}

// batch-norm statistics per (segment, channel) over `seg_rows` rows of x[rows, C] (bf16):
// fp64 sums per (segment, row chunk, channel), then a fixed-order final pass -> mean, invstd
__global__ void bn_stats_partial(const uint16_t* __restrict__ x, int seg_rows, int C, int chunks,
                                 double* __restrict__ part) {
  // grid: (ceil(C/32), chunks, segments); block (32, 8)
  const int c = blockIdx.x * 32 + threadIdx.x;
  const int seg = blockIdx.z;
  const int64_t r0 = static_cast<int64_t>(seg) * seg_rows;
  const int per = (seg_rows + chunks - 1) / chunks;
  const int a = blockIdx.y * per, b = min(seg_rows, a + per);
  __shared__ double red[2][8][33];
  double s1 = 0.0, s2 = 0.0;
  if (c < C)
    for (int r = a + threadIdx.y; r < b; r += 8) {
      const double v = bf2f(x[(r0 + r) * C + c]);
      s1 += v;
      s2 += v * v;
    }
  red[0][threadIdx.y][threadIdx.x] = s1;
  red[1][threadIdx.y][threadIdx.x] = s2;
  __syncthreads();
  if (threadIdx.y == 0 && c < C) {
    double t1 = 0.0, t2 = 0.0;
    for (int y = 0; y < 8; ++y) { t1 += red[0][y][threadIdx.x]; t2 += red[1][y][threadIdx.x]; }
    const size_t o = (static_cast<size_t>(seg) * chunks + blockIdx.y) * C + c;
    part[2 * o] = t1;
    part[2 * o + 1] = t2;
  }
}

// one warp per (segment, channel): lanes stride the chunks, fixed shuffle tree
__global__ void bn_stats_final(const double* __restrict__ part, int chunks, int C, int seg_rows, int segs,
                               float* __restrict__ mean, float* __restrict__ invstd, float eps) {
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;   // (segment, channel)
  const int lane = threadIdx.x & 31;
  if (i >= segs * C) return;
  const int seg = i / C, c = i - seg * C;
  double s1 = 0.0, s2 = 0.0;
#pragma unroll 8
  for (int k = lane; k < chunks; k += 32) {
    const size_t o = (static_cast<size_t>(seg) * chunks + k) * C + c;
    s1 += __ldcg(part + 2 * o);
    s2 += __ldcg(part + 2 * o + 1);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    s1 += __shfl_xor_sync(0xffffffffu, s1, off);
    s2 += __shfl_xor_sync(0xffffffffu, s2, off);
  }
  if (lane) return;
  const double m = s1 / seg_rows;
  const double var = fmax(s2 / seg_rows - m * m, 0.0);
  mean[i] = static_cast<float>(m);
  invstd[i] = static_cast<float>(1.0 / sqrt(var + eps));
}

// batch-norm statistics from the column partial sums the producing convolution's epilogue wrote
// (GemmArgs.colsum with colsum_sq: Σx plane then Σx² plane, one row per 32 output rows; segment
// `seg` = groups [seg·gps, (seg+1)·gps)): per (segment, row-group chunk, 32 channels) fp64 sums in
// the layout bn_stats_final reads (the same chunking as the statistics pass it replaces, over
// 1/32 of the rows)
__global__ void __launch_bounds__(256) bn_colsum_partial(const float* __restrict__ part, int64_t groups_total,
                                                         int gps, int C, int chunks, double* __restrict__ out) {
  __shared__ double red[2][8][33];
  const int lx = threadIdx.x & 31, ly = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + lx;
  const int seg = blockIdx.z;
  const int per = (gps + chunks - 1) / chunks;
  const int lo = blockIdx.y * per, hi = min(gps, lo + per);
  double s1 = 0.0, s2 = 0.0;
  if (c < C) {
#pragma unroll 4
    for (int g = lo + ly; g < hi; g += 8) {
      const size_t o = static_cast<size_t>(seg) * gps + g;
      s1 += __ldcg(part + o * C + c);
      s2 += __ldcg(part + (groups_total + o) * C + c);
    }
  }
  red[0][ly][lx] = s1;
  red[1][ly][lx] = s2;
  __syncthreads();
  if (ly != 0 || c >= C) return;
  double t1 = 0.0, t2 = 0.0;
#pragma unroll
  for (int y = 0; y < 8; ++y) { t1 += red[0][y][lx]; t2 += red[1][y][lx]; }
  const size_t o = (static_cast<size_t>(seg) * chunks + blockIdx.y) * C + c;
  out[2 * o] = t1;
  out[2 * o + 1] = t2;
}

// y = act(γ·(x - μ_seg)·invstd_seg + β (+ res)) -> bf16
__global__ void bn_apply_kernel(const uint16_t* __restrict__ x, const uint16_t* __restrict__ res,
                                uint16_t* __restrict__ y, const float* __restrict__ gamma, const float* __restrict__ beta,
                                const float* __restrict__ mean, const float* __restrict__ invstd, int64_t rows, int C,
                                int seg_rows, int relu) {
  const int64_t total = rows * C;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(i % C);
    const int64_t r = i / C;
    const int si = static_cast<int>(r / seg_rows) * C + c;
    float v = gamma[c] * ((bf2f(x[i]) - mean[si]) * invstd[si]) + beta[c];
    if (res) v += bf2f(res[i]);
    if (relu) v = fmaxf(v, 0.f);
    y[i] = f2bf(v);
  }
}

// backward sums per (segment, channel): Σ dy', Σ dy'·x̂ with dy' = dy ⊙ [y > 0] if relu (fp64)
__global__ void bn_bwd_partial(const uint16_t* __restrict__ dy, const uint16_t* __restrict__ y,
                               const uint16_t* __restrict__ x, const float* __restrict__ mean,
                               const float* __restrict__ invstd, int seg_rows, int C, int chunks, int relu,
                               double* __restrict__ part) {
  const int c = blockIdx.x * 32 + threadIdx.x;
  const int seg = blockIdx.z;
  const int64_t r0 = static_cast<int64_t>(seg) * seg_rows;
  const int per = (seg_rows + chunks - 1) / chunks;
  const int a = blockIdx.y * per, b = min(seg_rows, a + per);
  __shared__ double red[2][8][33];
  double s1 = 0.0, s2 = 0.0;
  if (c < C) {
    const double m = mean[seg * C + c], is = invstd[seg * C + c];
    for (int r = a + threadIdx.y; r < b; r += 8) {
      const int64_t o = (r0 + r) * C + c;
      double d = bf2f(dy[o]);
      if (relu && !(bf2f(y[o]) > 0.f)) d = 0.0;
      s1 += d;
      s2 += d * ((bf2f(x[o]) - m) * is);
    }
  }
  red[0][threadIdx.y][threadIdx.x] = s1;
  red[1][threadIdx.y][threadIdx.x] = s2;
  __syncthreads();
  if (threadIdx.y == 0 && c < C) {
    double t1 = 0.0, t2 = 0.0;
    for (int yy = 0; yy < 8; ++yy) { t1 += red[0][yy][threadIdx.x]; t2 += red[1][yy][threadIdx.x]; }
    const size_t o = (static_cast<size_t>(seg) * chunks + blockIdx.y) * C + c;
    part[2 * o] = t1;
    part[2 * o + 1] = t2;
  }
}

// per (segment, channel) sums -> sdy, sdyx (fp64); dγ = Σ_seg sdyx, dβ = Σ_seg sdy (fp32)
__global__ void bn_bwd_final(const double* __restrict__ part, int chunks, int C, int segs, double* __restrict__ sums,
                             float* __restrict__ dgamma, float* __restrict__ dbeta) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  double tg = 0.0, tb = 0.0;
  for (int seg = 0; seg < segs; ++seg) {
    double s1 = 0.0, s2 = 0.0;
    for (int k = 0; k < chunks; ++k) {
      const size_t o = (static_cast<size_t>(seg) * chunks + k) * C + c;
      s1 += part[2 * o];
      s2 += part[2 * o + 1];
    }
    sums[2 * (static_cast<size_t>(seg) * C + c)] = s1;
    sums[2 * (static_cast<size_t>(seg) * C + c) + 1] = s2;
    tb += s1;
    tg += s2;
  }
  dgamma[c] = static_cast<float>(tg);
  dbeta[c] = static_cast<float>(tb);
}

// dx = γ_res·invstd·(dy' - Σdy'/m - x̂·Σ(dy'x̂)/m) (bf16), γ_res = a·γ_stash + b·γ_latest;
// d_res = dy' written to `dres` (bf16) when the layer adds a residual
__global__ void bn_bwd_apply(const uint16_t* __restrict__ dy, const uint16_t* __restrict__ y,
                             const uint16_t* __restrict__ x, const float* __restrict__ mean,
                             const float* __restrict__ invstd, const double* __restrict__ sums,
                             const float* __restrict__ gs, const float* __restrict__ gl, float ga, float gb, int64_t rows,
                             int C, int seg_rows, int relu, uint16_t* __restrict__ dx, uint16_t* __restrict__ dres) {
  const int64_t total = rows * C;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(i % C);
    const int64_t r = i / C;
    const int seg = static_cast<int>(r / seg_rows);
    const int si = seg * C + c;
    float d = bf2f(dy[i]);
    if (relu && !(bf2f(y[i]) > 0.f)) d = 0.f;
    if (dres) dres[i] = f2bf(d);
    const float g = __fadd_rn(__fmul_rn(ga, gs[c]), __fmul_rn(gb, gl[c]));
    const float xh = (bf2f(x[i]) - mean[si]) * invstd[si];
    const double s1 = sums[2 * static_cast<size_t>(si)], s2 = sums[2 * static_cast<size_t>(si) + 1];
    const float v = g * invstd[si] * (d - static_cast<float>(s1 / seg_rows) - xh * static_cast<float>(s2 / seg_rows));
    dx[i] = f2bf(v);
  }
}

// 3x3 / stride 2 / pad 1 max pool (padding never wins), and its gradient in gather form: an
// input pixel collects dY of every window whose FIRST maximum it is (fixed window order)
__global__ void maxpool3_fwd_kernel(const uint16_t* __restrict__ X, uint16_t* __restrict__ Y, int N, int H, int W,
                                    int C, int Ho, int Wo) {
  const int64_t total = static_cast<int64_t>(N) * Ho * Wo * C;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(i % C);
    int64_t t = i / C;
    const int wo = static_cast<int>(t % Wo);
    t /= Wo;
    const int ho = static_cast<int>(t % Ho);
    const int64_t n = t / Ho;
    float best = -INFINITY;
    uint16_t bits = 0;
    for (int kh = 0; kh < 3; ++kh)
      for (int kw = 0; kw < 3; ++kw) {
        const int h = 2 * ho + kh - 1, w = 2 * wo + kw - 1;
        if (h < 0 || h >= H || w < 0 || w >= W) continue;
        const uint16_t hb = X[((n * H + h) * W + w) * C + c];
        const float v = bf2f(hb);
        if (v > best) { best = v; bits = hb; }
      }
    Y[i] = bits;
  }
}

__device__ __forceinline__ int maxpool3_first(const uint16_t* X, int64_t n, int ho, int wo, int c, int H, int W,
                                              int C) {
  float best = -INFINITY;
  int arg = -1;
  for (int kh = 0; kh < 3; ++kh)
    for (int kw = 0; kw < 3; ++kw) {
      const int h = 2 * ho + kh - 1, w = 2 * wo + kw - 1;
      if (h < 0 || h >= H || w < 0 || w >= W) continue;
      const float v = bf2f(X[((n * H + h) * W + w) * C + c]);
      if (v > best) { best = v; arg = h * W + w; }
    }
  return arg;
}

__global__ void maxpool3_bwd_kernel(const uint16_t* __restrict__ X, const uint16_t* __restrict__ dY,
                                    uint16_t* __restrict__ dX, int N, int H, int W, int C, int Ho, int Wo) {
  const int64_t total = static_cast<int64_t>(N) * H * W * C;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(i % C);
    int64_t t = i / C;
    const int w = static_cast<int>(t % W);
    t /= W;
    const int h = static_cast<int>(t % H);
    const int64_t n = t / H;
    float acc = 0.f;
    for (int ho = max(0, h / 2 - 1); ho <= min(Ho - 1, (h + 1) / 2); ++ho) {
      if (h < 2 * ho - 1 || h > 2 * ho + 1) continue;
      for (int wo = max(0, w / 2 - 1); wo <= min(Wo - 1, (w + 1) / 2); ++wo) {
        if (w < 2 * wo - 1 || w > 2 * wo + 1) continue;
        if (maxpool3_first(X, n, ho, wo, c, H, W, C) == h * W + w) acc += bf2f(dY[((n * Ho + ho) * Wo + wo) * C + c]);
      }
    }
    dX[i] = f2bf(acc);
  }
}

// global average pool [N, H*W, C] -> [N, C] (fp32 sum in fixed order, bf16 out) and its gradient
__global__ void avgpool_fwd_kernel(const uint16_t* __restrict__ X, uint16_t* __restrict__ Y, int N, int HW, int C) {
  const int64_t total = static_cast<int64_t>(N) * C;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(i % C);
    const int64_t n = i / C;
    double acc = 0.0;
    for (int p = 0; p < HW; ++p) acc += bf2f(X[(n * HW + p) * C + c]);
    Y[i] = f2bf(static_cast<float>(acc / HW));
  }
}

__global__ void avgpool_bwd_kernel(const uint16_t* __restrict__ dY, uint16_t* __restrict__ dX, int N, int HW, int C) {
  const int64_t total = static_cast<int64_t>(N) * HW * C;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(i % C);
    const int64_t n = i / (static_cast<int64_t>(HW) * C);
    dX[i] = f2bf(bf2f(dY[n * C + c]) / HW);
  }
}

// out = bf16(out + add)   (gradient accumulation of a tensor with two consumers)
__global__ void add_bf16_kernel(uint16_t* __restrict__ out, const uint16_t* __restrict__ add, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = f2bf(bf2f(out[i]) + bf2f(add[i]));
}

// ------------------------------------------------------------------ vectorised ResNet kernels
// 8 channels (16 bytes) per thread; used when C % 8 == 0 (every ResNet-50 layer)
__device__ __forceinline__ void unpack8(const uint4& v, float (&f)[8]) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int e = 0; e < 8; ++e) f[e] = bf2f((w[e >> 1] >> ((e & 1) * 16)) & 0xFFFFu);
}

__device__ __forceinline__ uint4 pack8(const float (&f)[8]) {
  uint4 o;
  o.x = static_cast<uint32_t>(f2bf(f[0])) | (static_cast<uint32_t>(f2bf(f[1])) << 16);
  o.y = static_cast<uint32_t>(f2bf(f[2])) | (static_cast<uint32_t>(f2bf(f[3])) << 16);
  o.z = static_cast<uint32_t>(f2bf(f[4])) | (static_cast<uint32_t>(f2bf(f[5])) << 16);
  o.w = static_cast<uint32_t>(f2bf(f[6])) | (static_cast<uint32_t>(f2bf(f[7])) << 16);
  return o;
}

// bit e = [bf16 element e of v > 0] (0 < bits <= 0x7F80: positive, +inf included, NaN excluded)
__device__ __forceinline__ uint8_t relu_bits8(const uint4& v) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
  uint32_t m = 0;
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const uint32_t h = (w[e >> 1] >> ((e & 1) * 16)) & 0xFFFFu;
    m |= static_cast<uint32_t>(h - 1u < 0x7F80u) << e;
  }
  return static_cast<uint8_t>(m);
}

__device__ __forceinline__ void load8f(const float* p, float (&f)[8]) {
  const float4 a = *reinterpret_cast<const float4*>(p), b = *reinterpret_cast<const float4*>(p + 4);
  f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w; f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
}

// gradient of the global average pool over 8 channels per thread (C % 8 == 0): 16-byte stores
__global__ void avgpool_bwd_vec(const uint4* __restrict__ dY, uint4* __restrict__ dX, int N, int HW, int C8) {
  const int64_t total = static_cast<int64_t>(N) * HW * C8;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int cv = static_cast<int>(i % C8);
    const int64_t n = i / (static_cast<int64_t>(HW) * C8);
    float d[8];
    unpack8(__ldg(dY + n * C8 + cv), d);
#pragma unroll
    for (int e = 0; e < 8; ++e) d[e] = d[e] / HW;
    dX[i] = pack8(d);
  }
}

// Row-mapped BN apply kernels: a thread owns one 8-channel group and walks rows, so the
// per-channel parameters (γ, β, and the current segment's statistics / backward coefficients)
// stay in registers; a warp covers 512 contiguous bytes of a row (or of 32/tx adjacent rows).
// block = tx channel groups x ty rows (tx = min(C8, 32)), grid = (ceil(C8/tx), row blocks).
template <bool MASK>   // MASK: also write the ReLU bit mask (compile-time)
__global__ void __launch_bounds__(256) bn_apply_rows(const uint4* __restrict__ x, const uint4* __restrict__ res,
                                                     uint4* __restrict__ y, const float* __restrict__ gamma,
                                                     const float* __restrict__ beta, const float* __restrict__ mean,
                                                     const float* __restrict__ invstd, int rows, int C8, int seg_rows,
                                                     int relu, uint8_t* __restrict__ mask) {
  const int tx = min(C8, 32), ty = blockDim.x / tx;
  const int cg = blockIdx.x * tx + static_cast<int>(threadIdx.x) % tx;
  if (cg >= C8 || static_cast<int>(threadIdx.x) >= tx * ty) return;
  const int C = C8 * 8, c0 = cg * 8;
  float g[8], bt[8], m[8], is[8];
  load8f(gamma + c0, g);
  load8f(beta + c0, bt);
  int cur = -1;
  const int step = gridDim.y * ty;
#pragma unroll 4
  for (int r = blockIdx.y * ty + static_cast<int>(threadIdx.x) / tx; r < rows; r += step) {   // loads of 4 rows in flight
    const int seg = r / seg_rows;
    if (seg != cur) {
      cur = seg;
      load8f(mean + seg * C + c0, m);
      load8f(invstd + seg * C + c0, is);
    }
    const size_t o = static_cast<size_t>(r) * C8 + cg;
    float xv[8], v[8];
    unpack8(x[o], xv);
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] = g[e] * ((xv[e] - m[e]) * is[e]) + bt[e];
    if (res) {
      float rv[8];
      unpack8(res[o], rv);
#pragma unroll
      for (int e = 0; e < 8; ++e) v[e] += rv[e];
    }
    if (relu) {
#pragma unroll
      for (int e = 0; e < 8; ++e) v[e] = fmaxf(v[e], 0.f);
    }
    const uint4 py = pack8(v);
    y[o] = py;
    if (MASK) mask[o] = relu_bits8(py);
  }
}

template <bool MASK>   // MASK: ReLU mask from the forward's bit mask (compile-time, see bn_partial_vec)
__global__ void __launch_bounds__(256) bn_bwd_apply_rows(const uint4* __restrict__ dy, const uint4* __restrict__ yv,
                                                         const uint4* __restrict__ xv, const float4* __restrict__ coef,
                                                         const float* __restrict__ invstd, int rows, int C8,
                                                         int seg_rows, int relu, uint4* __restrict__ dx,
                                                         uint4* __restrict__ dres, const uint8_t* __restrict__ mask) {
  const int tx = min(C8, 32), ty = blockDim.x / tx;
  const int cg = blockIdx.x * tx + static_cast<int>(threadIdx.x) % tx;
  if (cg >= C8 || static_cast<int>(threadIdx.x) >= tx * ty) return;
  const int C = C8 * 8, c0 = cg * 8;
  float ka[8], kb[8], kc[8], km[8], is[8];
  int cur = -1;
  const int step = gridDim.y * ty;
#pragma unroll 4
  for (int r = blockIdx.y * ty + static_cast<int>(threadIdx.x) / tx; r < rows; r += step) {   // loads of 4 rows in flight
    const int seg = r / seg_rows;
    if (seg != cur) {
      cur = seg;
      const int sc = seg * C + c0;
      load8f(invstd + sc, is);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float4 k = coef[sc + e];
        ka[e] = k.x; kb[e] = k.y; kc[e] = k.z; km[e] = k.w;
      }
    }
    const size_t o = static_cast<size_t>(r) * C8 + cg;
    float d[8], xx[8], out[8];
    unpack8(dy[o], d);
    unpack8(xv[o], xx);
    if (MASK) {
      const uint32_t mb = mask[o];
#pragma unroll
      for (int e = 0; e < 8; ++e)
        if (!((mb >> e) & 1u)) d[e] = 0.f;
    } else if (relu) {
      float yy[8];
      unpack8(yv[o], yy);
#pragma unroll
      for (int e = 0; e < 8; ++e)
        if (!(yy[e] > 0.f)) d[e] = 0.f;
    }
    if (dres) dres[o] = pack8(d);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float xh = (xx[e] - km[e]) * is[e];
      out[e] = ka[e] * (d[e] - kb[e] - xh * kc[e]);
    }
    dx[o] = pack8(out);
  }
}

// per (segment, chunk) partial sums over 8 channels per thread, fp64:
//   MODE 0 (statistics): Σx, Σx²;  MODE 1 (backward): Σdy', Σdy'·x̂ (dy' = dy ⊙ [y > 0] if relu);
//   MODE 2: MODE 1 with the ReLU mask from the forward's bit mask (compile-time, so the unrolled
//   loop keeps its loads in flight: a run-time choice between the two mask sources serialised them)
// block: tx = min(C8, 32) channel groups x ty = 256 / tx rows; grid (ceil(C8/tx), chunks, segs)
template <int MODE>
__global__ void __launch_bounds__(256) bn_partial_vec(const uint4* __restrict__ a, const uint4* __restrict__ yv,
                                                      const uint4* __restrict__ xv, const float* __restrict__ mean,
                                                      const float* __restrict__ invstd, int seg_rows, int C8,
                                                      int chunks, int relu, double* __restrict__ part,
                                                      const uint8_t* __restrict__ mask) {
  extern __shared__ double red[];            // [ty][tx][16]
  const int tx = min(C8, 32), ty = blockDim.x / tx;
  const int lx = threadIdx.x % tx, ly = threadIdx.x / tx;
  const int cg = blockIdx.x * tx + lx;       // channel group
  const int seg = blockIdx.z;
  const int C = C8 * 8;
  const int64_t r0 = static_cast<int64_t>(seg) * seg_rows;
  const int per = (seg_rows + chunks - 1) / chunks;
  const int lo = blockIdx.y * per, hi = min(seg_rows, lo + per);
  double s1[8], s2[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) s1[e] = s2[e] = 0.0;
  if (cg < C8) {
    float m[8], is[8];
    if (MODE != 0) {
      load8f(mean + seg * C + cg * 8, m);
      load8f(invstd + seg * C + cg * 8, is);
    }
#pragma unroll 8
    for (int r = lo + ly; r < hi; r += ty) {   // 8 rows of loads in flight per thread
      const int64_t o = (r0 + r) * C8 + cg;
      float v[8];
      unpack8(a[o], v);
      if (MODE == 0) {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          s1[e] += v[e];
          s2[e] += static_cast<double>(v[e]) * v[e];
        }
      } else {
        float yy[8], xx[8];
        unpack8(xv[o], xx);
        if (MODE == 2) {
          const uint32_t mb = mask[o];
#pragma unroll
          for (int e = 0; e < 8; ++e) yy[e] = ((mb >> e) & 1u) ? 1.f : 0.f;
        } else if (relu) {
          unpack8(yv[o], yy);
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const double d = ((MODE == 2 || relu) && !(yy[e] > 0.f)) ? 0.0 : static_cast<double>(v[e]);
          s1[e] += d;
          s2[e] += d * ((static_cast<double>(xx[e]) - m[e]) * is[e]);
        }
      }
    }
  }
  double* mine = red + (static_cast<size_t>(ly) * tx + lx) * 16;
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    mine[e] = s1[e];
    mine[8 + e] = s2[e];
  }
  __syncthreads();
  if (ly == 0 && cg < C8) {
    for (int yy = 1; yy < ty; ++yy) {
      const double* o = red + (static_cast<size_t>(yy) * tx + lx) * 16;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        s1[e] += o[e];
        s2[e] += o[8 + e];
      }
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const size_t o = (static_cast<size_t>(seg) * chunks + blockIdx.y) * C + cg * 8 + e;
      part[2 * o] = s1[e];
      part[2 * o + 1] = s2[e];
    }
  }
}

// backward coefficients per (segment, channel), packed float4 {γ_r·invstd, Σdy'/m, Σdy'x̂/m, mean}
// with γ_r = a·γ_stash + b·γ_latest; and dγ, dβ summed over segments in segment order.
// One block per channel, one warp per segment (warps stride the segments): lanes stride the
// chunks, fixed shuffle tree, lane 0 parks the segment's sums in shared memory; thread 0 then
// adds them in segment order.  (One warp per channel walking the segments serially left the
// grid at C/8 blocks and ran ~29 µs per launch, latency-bound, on ResNet-50's 64-channel layers.)
constexpr int kBnCoefWarps = 8;
__global__ void __launch_bounds__(32 * kBnCoefWarps) bn_bwd_coef(
    const double* __restrict__ part, int chunks, int C, int segs, int seg_rows, const float* __restrict__ mean,
    const float* __restrict__ invstd, const float* __restrict__ gs, const float* __restrict__ gl, float ga, float gb,
    float4* __restrict__ coef, float* __restrict__ dgamma, float* __restrict__ dbeta) {
  extern __shared__ double seg_sums[];   // [segs][2]
  const int c = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const float g = __fadd_rn(__fmul_rn(ga, gs[c]), __fmul_rn(gb, gl[c]));
  for (int seg = warp; seg < segs; seg += blockDim.x >> 5) {
    double s1 = 0.0, s2 = 0.0;
#pragma unroll 8
    for (int k = lane; k < chunks; k += 32) {
      const size_t o = (static_cast<size_t>(seg) * chunks + k) * C + c;
      s1 += __ldcg(part + 2 * o);
      s2 += __ldcg(part + 2 * o + 1);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      s1 += __shfl_xor_sync(0xffffffffu, s1, off);
      s2 += __shfl_xor_sync(0xffffffffu, s2, off);
    }
    if (lane) continue;
    seg_sums[2 * seg] = s1;
    seg_sums[2 * seg + 1] = s2;
    const int sc = seg * C + c;
    coef[sc] = make_float4(g * invstd[sc], static_cast<float>(s1 / seg_rows), static_cast<float>(s2 / seg_rows),
                           mean[sc]);
  }
  __syncthreads();
  if (threadIdx.x) return;
  double tg = 0.0, tb = 0.0;
  for (int seg = 0; seg < segs; ++seg) {
    tb += seg_sums[2 * seg];
    tg += seg_sums[2 * seg + 1];
  }
  dgamma[c] = static_cast<float>(tg);
  dbeta[c] = static_cast<float>(tb);
}

// 3x3/2/1 max pool over 8 channels per thread, recording the first-max tap (0..8) per output
__global__ void maxpool3_fwd_vec(const uint4* __restrict__ X, uint4* __restrict__ Y, uint2* __restrict__ idx, int N,
                                 int H, int W, int C8, int Ho, int Wo) {
  const int64_t total = static_cast<int64_t>(N) * Ho * Wo * C8;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int cv = static_cast<int>(i % C8);
    int64_t t = i / C8;
    const int wo = static_cast<int>(t % Wo);
    t /= Wo;
    const int ho = static_cast<int>(t % Ho);
    const int64_t n = t / Ho;
    float best[8];
    uint32_t bits[8], arg[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) { best[e] = -INFINITY; bits[e] = 0; arg[e] = 0; }
    for (int kh = 0; kh < 3; ++kh) {
      const int h = 2 * ho + kh - 1;
      if (h < 0 || h >= H) continue;
      for (int kw = 0; kw < 3; ++kw) {
        const int w = 2 * wo + kw - 1;
        if (w < 0 || w >= W) continue;
        const uint4 v = X[((n * H + h) * W + w) * C8 + cv];
        const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const uint32_t hb = (wv[e >> 1] >> ((e & 1) * 16)) & 0xFFFFu;
          const float f = bf2f(hb);
          if (f > best[e]) { best[e] = f; bits[e] = hb; arg[e] = kh * 3 + kw; }
        }
      }
    }
    uint4 o;
    o.x = bits[0] | (bits[1] << 16); o.y = bits[2] | (bits[3] << 16);
    o.z = bits[4] | (bits[5] << 16); o.w = bits[6] | (bits[7] << 16);
    Y[i] = o;
    idx[i] = make_uint2(arg[0] | (arg[1] << 8) | (arg[2] << 16) | (arg[3] << 24),
                        arg[4] | (arg[5] << 8) | (arg[6] << 16) | (arg[7] << 24));
  }
}

// gradient in gather form from the recorded taps: dX[n,h,w,c] = Σ dY of windows whose first max
// is (h, w), windows in (ho, wo) order
__global__ void maxpool3_bwd_vec(const uint2* __restrict__ idx, const uint4* __restrict__ dY, uint4* __restrict__ dX,
                                 int N, int H, int W, int C8, int Ho, int Wo) {
  const int64_t total = static_cast<int64_t>(N) * H * W * C8;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int cv = static_cast<int>(i % C8);
    int64_t t = i / C8;
    const int w = static_cast<int>(t % W);
    t /= W;
    const int h = static_cast<int>(t % H);
    const int64_t n = t / H;
    float acc[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] = 0.f;
    for (int ho = max(0, h / 2 - 1); ho <= min(Ho - 1, (h + 1) / 2); ++ho) {
      const int kh = h - (2 * ho - 1);
      if (kh < 0 || kh > 2) continue;
      for (int wo = max(0, w / 2 - 1); wo <= min(Wo - 1, (w + 1) / 2); ++wo) {
        const int kw = w - (2 * wo - 1);
        if (kw < 0 || kw > 2) continue;
        const uint32_t tap = kh * 3 + kw;
        const int64_t o = ((n * Ho + ho) * Wo + wo) * C8 + cv;
        const uint2 a = idx[o];
        const uint32_t av[2] = {a.x, a.y};
        float g[8];
        unpack8(dY[o], g);
#pragma unroll
        for (int e = 0; e < 8; ++e)
          if (((av[e >> 2] >> ((e & 3) * 8)) & 0xFFu) == tap) acc[e] += g[e];
      }
    }
    dX[i] = pack8(acc);
  }
}

// patch gradients back to the image, 4 channels per thread (C % 4 == 0)
__global__ void col2im_vec4(const float* __restrict__ dP, uint2* __restrict__ dX, const uint2* __restrict__ add, int N,
                            int H, int W, int C, int k, int s, int p, int Ho, int Wo, int ldp) {
  const int C4 = C / 4;
  const int64_t total = static_cast<int64_t>(N) * H * W * C4;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(i % C4) * 4;
    int64_t t = i / C4;
    const int w = static_cast<int>(t % W);
    t /= W;
    const int h = static_cast<int>(t % H);
    const int64_t n = t / H;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int kh = 0; kh < k; ++kh) {
      const int hy = h + p - kh;
      if (hy < 0 || hy % s) continue;
      const int ho = hy / s;
      if (ho >= Ho) continue;
      for (int kw = 0; kw < k; ++kw) {
        const int wy = w + p - kw;
        if (wy < 0 || wy % s) continue;
        const int wo = wy / s;
        if (wo >= Wo) continue;
        const float4 v = *reinterpret_cast<const float4*>(
            dP + ((n * Ho + ho) * Wo + wo) * static_cast<int64_t>(ldp) + (kh * k + kw) * C + c);
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
      }
    }
    if (add) {
      const uint2 a = add[i];
      acc.x += bf2f(a.x & 0xFFFFu); acc.y += bf2f(a.x >> 16); acc.z += bf2f(a.y & 0xFFFFu); acc.w += bf2f(a.y >> 16);
    }
    dX[i] = make_uint2(static_cast<uint32_t>(f2bf(acc.x)) | (static_cast<uint32_t>(f2bf(acc.y)) << 16),
                       static_cast<uint32_t>(f2bf(acc.z)) | (static_cast<uint32_t>(f2bf(acc.w)) << 16));
  }
}

// col2im_vec4 with the kernel size and stride fixed at compile time (the strided ResNet-50
// convolutions: 3x3/2 and 1x1/2): every tap's load is issued before the first add (predicated,
// up to ceil(K/S)^2 live), where the generic loop's data-dependent branches serialised them; the
// adds keep the generic kernel's order (kh, kw ascending), so the result is bitwise the same
template <int K, int S>
__global__ void __launch_bounds__(256) col2im_vec4_ks(const float* __restrict__ dP, uint2* __restrict__ dX,
                                                      const uint2* __restrict__ add, int N, int H, int W, int C,
                                                      int p, int Ho, int Wo, int ldp) {
  const int C4 = C / 4;
  const int64_t total = static_cast<int64_t>(N) * H * W * C4;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(i % C4) * 4;
    int64_t t = i / C4;
    const int w = static_cast<int>(t % W);
    t /= W;
    const int h = static_cast<int>(t % H);
    const int64_t n = t / H;
    float4 v[K * K];
    bool ok[K * K];
#pragma unroll
    for (int kh = 0; kh < K; ++kh) {
#pragma unroll
      for (int kw = 0; kw < K; ++kw) {
        const int hy = h + p - kh, wy = w + p - kw;
        const int ho = hy / S, wo = wy / S;
        const bool o = hy >= 0 && hy % S == 0 && ho < Ho && wy >= 0 && wy % S == 0 && wo < Wo;
        ok[kh * K + kw] = o;
        v[kh * K + kw] = o ? __ldcs(reinterpret_cast<const float4*>(
                                 dP + ((n * Ho + ho) * Wo + wo) * static_cast<int64_t>(ldp) + (kh * K + kw) * C + c))
                           : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
    const uint2 a = add ? __ldcs(add + i) : make_uint2(0u, 0u);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int q = 0; q < K * K; ++q)
      if (ok[q]) { acc.x += v[q].x; acc.y += v[q].y; acc.z += v[q].z; acc.w += v[q].w; }
    if (add) {
      acc.x += bf2f(a.x & 0xFFFFu); acc.y += bf2f(a.x >> 16); acc.z += bf2f(a.y & 0xFFFFu); acc.w += bf2f(a.y >> 16);
    }
    dX[i] = make_uint2(static_cast<uint32_t>(f2bf(acc.x)) | (static_cast<uint32_t>(f2bf(acc.y)) << 16),
                       static_cast<uint32_t>(f2bf(acc.z)) | (static_cast<uint32_t>(f2bf(acc.w)) << 16));
  }
}

// explicit patches, 8 consecutive columns per thread (one 16-byte store), ldp % 8 == 0
__global__ void im2col_vec8(const uint16_t* __restrict__ X, uint4* __restrict__ P, int H, int W, int C, int k, int s,
                            int p, int Ho, int Wo, int ldp8, int64_t nvec) {
  const int kkC = k * k * C;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nvec;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / ldp8;
    const int col0 = static_cast<int>(i - r * ldp8) * 8;
    const int wo = static_cast<int>(r % Wo);
    const int64_t t = r / Wo;
    const int ho = static_cast<int>(t % Ho);
    const int64_t n = t / Ho;
    const uint16_t* xb = X + n * H * W * static_cast<int64_t>(C);
    int tap = col0 / C, c = col0 - tap * C;
    int kh = tap / k, kw = tap - kh * k;
    uint32_t v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      uint32_t val = 0;
      if (col0 + e < kkC) {
        const int hh = ho * s + kh - p, ww = wo * s + kw - p;
        if (hh >= 0 && hh < H && ww >= 0 && ww < W) val = xb[(hh * W + ww) * C + c];
      }
      v[e] = val;
      if (++c == C) {
        c = 0;
        if (++kw == k) { kw = 0; ++kh; }
      }
    }
    P[i] = make_uint4(v[0] | (v[1] << 16), v[2] | (v[3] << 16), v[4] | (v[5] << 16), v[6] | (v[7] << 16));
  }
}

// explicit patches for one output row (n, ho) per block: the k input rows it reads are staged in
// shared memory with the zero padding materialised, a per-column offset table maps patch
// column (kh, kw, c) to its smem element, and the patch rows are written as 16-byte vectors
__global__ void __launch_bounds__(256) im2col_rowtile(const uint16_t* __restrict__ X, uint4* __restrict__ P, int H,
                                                      int W, int C, int k, int s, int p, int Ho, int Wo, int ldp) {
  extern __shared__ uint16_t sm[];
  const int Wp = W + 2 * p;                       // padded row length (pixels)
  const int rowlen = Wp * C;
  uint16_t* tile = sm;                            // [k][Wp][C]
  int* off = reinterpret_cast<int*>(sm + ((k * rowlen + 1) & ~1));   // [ldp]
  const int n = blockIdx.x / Ho, ho = blockIdx.x - n * Ho;
  const int h0 = ho * s - p;
  for (int i = threadIdx.x; i < k * rowlen; i += blockDim.x) {
    const int kh = i / rowlen, rem = i - kh * rowlen;
    const int wp = rem / C, c = rem - wp * C;
    const int h = h0 + kh, w = wp - p;
    uint16_t v = 0;
    if (h >= 0 && h < H && w >= 0 && w < W) v = X[((static_cast<int64_t>(n) * H + h) * W + w) * C + c];
    tile[i] = v;
  }
  const int kkC = k * k * C;
  for (int col = threadIdx.x; col < ldp; col += blockDim.x) {
    int o = -1;
    if (col < kkC) {
      const int kh = col / (k * C), rem = col - kh * k * C;    // rem = kw·C + c
      o = kh * rowlen + rem;
    }
    off[col] = o;
  }
  __syncthreads();
  const int v8 = ldp / 8;
  uint4* prow = P + (static_cast<int64_t>(n) * Ho + ho) * Wo * v8;
  for (int i = threadIdx.x; i < Wo * v8; i += blockDim.x) {
    const int wo = i / v8, cv = i - wo * v8;
    const int base = wo * s * C;
    uint32_t v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int o = off[cv * 8 + e];
      v[e] = o >= 0 ? tile[o + base] : 0u;
    }
    prow[i] = make_uint4(v[0] | (v[1] << 16), v[2] | (v[3] << 16), v[4] | (v[5] << 16), v[6] | (v[7] << 16));
  }
}

// im2col_rowtile with the k input rows staged by 16-byte loads (W·C % 8 == 0: every input row
// starts 16-byte aligned).  Tile row layout: [lead zeros | W·C data at D0 | trail zeros], D0 =
// p·C rounded up to 8 elements, so padded pixel wp, channel c sits at D0 − p·C + wp·C + c; rows
// outside the image are all zeros.  The scalar fill of im2col_rowtile issued its 2-byte loads
// one after another (integer divisions between them) and dominated that kernel.
__global__ void __launch_bounds__(256) im2col_rowtile_v(const uint16_t* __restrict__ X, uint4* __restrict__ P, int H,
                                                        int W, int C, int k, int s, int p, int Ho, int Wo, int ldp,
                                                        int D0, int rowlen, int staged) {
  extern __shared__ __align__(16) uint16_t smv[];
  uint16_t* tile = smv;                                    // [k][rowlen], rowlen % 8 == 0
  int* off = reinterpret_cast<int*>(smv + k * rowlen);     // [ldp]
  const int n = blockIdx.x / Ho, ho = blockIdx.x - n * Ho;
  const int h0 = ho * s - p;
  const int WC8 = W * C / 8, row8 = rowlen / 8, D08 = D0 / 8;
  uint4* tile4 = reinterpret_cast<uint4*>(tile);
  const uint4* X4 = reinterpret_cast<const uint4*>(X);
  for (int i = threadIdx.x; i < k * row8; i += blockDim.x) {
    const int kh = i / row8, q = i - kh * row8;
    const int h = h0 + kh, d = q - D08;
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    if (h >= 0 && h < H && d >= 0 && d < WC8) v = __ldg(X4 + (static_cast<int64_t>(n) * H + h) * WC8 + d);
    tile4[i] = v;
  }
  const int kkC = k * k * C, shift = D0 - p * C;
  for (int col = threadIdx.x; col < ldp; col += blockDim.x) {
    int o = -1;
    if (col < kkC) {
      const int kh = col / (k * C), rem = col - kh * k * C;    // rem = kw·C + c
      o = kh * rowlen + shift + rem;
    }
    off[col] = o;
  }
  __syncthreads();
  const int v8 = ldp / 8;
  uint4* prow = P + (static_cast<int64_t>(n) * Ho + ho) * Wo * v8;
  if (staged) {
    // the block's patch rows assembled element by element in shared memory (consecutive threads
    // read consecutive tile elements and write consecutive outputs), then streamed out as
    // 16-byte stores (opt-in: measured slower than the direct 8-element gather below)
    uint16_t* outs = reinterpret_cast<uint16_t*>(off + ldp);   // [Wo][ldp]
    for (int i = threadIdx.x; i < Wo * ldp; i += blockDim.x) {
      const int wo = i / ldp, col = i - wo * ldp;
      const int o = off[col];
      outs[i] = o >= 0 ? tile[o + wo * s * C] : static_cast<uint16_t>(0);
    }
    __syncthreads();
    const uint4* outs4 = reinterpret_cast<const uint4*>(outs);
    for (int i = threadIdx.x; i < Wo * v8; i += blockDim.x) __stcs(prow + i, outs4[i]);
    return;
  }
  for (int i = threadIdx.x; i < Wo * v8; i += blockDim.x) {
    const int wo = i / v8, cv = i - wo * v8;
    const int base = wo * s * C;
    uint32_t v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int o = off[cv * 8 + e];
      v[e] = o >= 0 ? tile[o + base] : 0u;
    }
    __stcs(prow + i, make_uint4(v[0] | (v[1] << 16), v[2] | (v[3] << 16), v[4] | (v[5] << 16), v[6] | (v[7] << 16)));
  }
}

// explicit patches, one output pixel row per block iteration (32-bit index math per element)
__global__ void im2col_rows(const uint16_t* __restrict__ X, uint16_t* __restrict__ P, int N, int H, int W, int C,
                            int k, int s, int p, int Ho, int Wo, int ldp, int64_t rows) {
  const int kkC = k * k * C;
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    const int wo = static_cast<int>(r % Wo);
    const int64_t t = r / Wo;
    const int ho = static_cast<int>(t % Ho);
    const int64_t n = t / Ho;
    const uint16_t* xb = X + n * H * W * static_cast<int64_t>(C);
    uint16_t* pr = P + r * ldp;
    for (int col = threadIdx.x; col < ldp; col += blockDim.x) {
      uint16_t v = 0;
      if (col < kkC) {
        const int tap = col / C, c = col - tap * C;
        const int kh = tap / k, kw = tap - kh * k;
        const int hh = ho * s + kh - p, ww = wo * s + kw - p;
        if (hh >= 0 && hh < H && ww >= 0 && ww < W) v = xb[(hh * W + ww) * C + c];
      }
      pr[col] = v;
    }
  }
}

uint64_t host_mix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

}  // namespace

cudaError_t launch_sgd_update(float* w, float* v, const float* g, uint16_t* ver, int64_t n, float lr, float mu,
                              float wd, cudaStream_t st, int blocks_per_sm, int tf) {
  if (n <= 0) return cudaSuccess;
  if (n % 4) return cudaErrorInvalidValue;
  const int64_t n4 = n / 4;
  const int grid = grid_for(n4, 256, blocks_per_sm);
  const bool mom = mu != 0.0f;
  if (tf && ver) {
    if (mom) sgd_update_kernel<true, true, true><<<grid, 256, 0, st>>>(w, v, g, ver, n4, lr, mu, wd);
    else sgd_update_kernel<false, true, true><<<grid, 256, 0, st>>>(w, v, g, ver, n4, lr, mu, wd);
  } else if (mom && ver) sgd_update_kernel<true, true><<<grid, 256, 0, st>>>(w, v, g, ver, n4, lr, mu, wd);
  else if (mom) sgd_update_kernel<true, false><<<grid, 256, 0, st>>>(w, v, g, ver, n4, lr, mu, wd);
  else if (ver) sgd_update_kernel<false, true><<<grid, 256, 0, st>>>(w, v, g, ver, n4, lr, mu, wd);
  else sgd_update_kernel<false, false><<<grid, 256, 0, st>>>(w, v, g, ver, n4, lr, mu, wd);
  return cudaGetLastError();
}

cudaError_t launch_sgd_update_dp(float* w, float* v, const GradList& g, uint16_t* ver, int64_t n, float lr, float mu,
                                 float wd, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  if (n % 4 || g.n < 1 || g.n > GradList::MAX) return cudaErrorInvalidValue;
  const int64_t n4 = n / 4;
  const int grid = grid_for(n4, 256, 8);
  const bool mom = mu != 0.0f;
  if (mom && ver) sgd_update_dp_kernel<true, true><<<grid, 256, 0, st>>>(w, v, g, ver, n4, lr, mu, wd);
  else if (mom) sgd_update_dp_kernel<true, false><<<grid, 256, 0, st>>>(w, v, g, ver, n4, lr, mu, wd);
  else if (ver) sgd_update_dp_kernel<false, true><<<grid, 256, 0, st>>>(w, v, g, ver, n4, lr, mu, wd);
  else sgd_update_dp_kernel<false, false><<<grid, 256, 0, st>>>(w, v, g, ver, n4, lr, mu, wd);
  return cudaGetLastError();
}

cudaError_t launch_bias_from_colsum(const float* part, int groups, int cols, float* db, float* b, float* vb, float lr,
                                   float mu, float wd, cudaStream_t st) {
  if (cols <= 0) return cudaSuccess;
  bias_from_colsum_kernel<<<(cols + 31) / 32, 256, 0, st>>>(part, groups, cols, db, b, vb, lr, mu, wd);
  return cudaGetLastError();
}

int64_t bias_grad_scratch_floats(int rows, int cols) {
  // BG_CNT arrival counters of bias_grad_fused (zero at allocation, self-resetting) at a fixed
  // offset, then the partial sums
  return BG_CNT + static_cast<int64_t>(bias_grad_splits(rows, cols)) * cols;
}

cudaError_t launch_bias_grad_sgd(const uint16_t* G, int rows, int cols, int ldg, float* db, float* scratch, float* b,
                                 float* vb, float lr, float mu, float wd, cudaStream_t st, int tf) {
  if (cols <= 0) return cudaSuccess;
  if (cols % 8 || ldg % 8) return cudaErrorInvalidValue;
  const int splits = bias_grad_splits(rows, cols);
  const int rps = (rows + splits - 1) / splits;
  const int tx = bg_tx(cols);
  dim3 grid((cols + tx * 8 - 1) / (tx * 8), splits), block(tx, 256 / tx);
  if (static_cast<int>(grid.x) > BG_CNT) return cudaErrorInvalidValue;
  unsigned int* cnt = reinterpret_cast<unsigned int*>(scratch);
  if (tf)
    bias_grad_fused<true><<<grid, block, 0, st>>>(G, rows, cols, ldg, rps, scratch + BG_CNT, cnt, db, b, vb, lr, mu, wd);
  else
    bias_grad_fused<false><<<grid, block, 0, st>>>(G, rows, cols, ldg, rps, scratch + BG_CNT, cnt, db, b, vb, lr, mu, wd);
  return cudaGetLastError();
}

cudaError_t launch_bias_grad(const uint16_t* G, int rows, int cols, int ldg, float* db, float* scratch,
                             cudaStream_t st, int tf) {
  if (cols <= 0) return cudaSuccess;
  if (cols % 8 || ldg % 8) return cudaErrorInvalidValue;
  const int splits = bias_grad_splits(rows, cols);
  const int rps = (rows + splits - 1) / splits;
  const int tx = bg_tx(cols);
  dim3 grid((cols + tx * 8 - 1) / (tx * 8), splits), block(tx, 256 / tx);
  if (tf) bias_grad_partial<true><<<grid, block, 0, st>>>(G, rows, cols, ldg, rps, scratch + BG_CNT);
  else bias_grad_partial<false><<<grid, block, 0, st>>>(G, rows, cols, ldg, rps, scratch + BG_CNT);
  bias_grad_final<<<(cols + 255) / 256, 256, 0, st>>>(scratch + BG_CNT, splits, cols, db);
  return cudaGetLastError();
}

cudaError_t launch_softmax_xent(const float* logits, int ldl, const int32_t* labels, int rows, int classes, int batch,
                                float* loss_rows, uint16_t* G, int ldg, cudaStream_t st, int tf) {
  if (rows <= 0) return cudaSuccess;
  const int warps_per_block = 8;
  if (tf) {
    softmax_xent_kernel<true><<<(rows + warps_per_block - 1) / warps_per_block, 32 * warps_per_block, 0, st>>>(
        logits, ldl, labels, rows, classes, batch, loss_rows, G, ldg);
    return cudaGetLastError();
  }
  softmax_xent_kernel<false><<<(rows + warps_per_block - 1) / warps_per_block, 32 * warps_per_block, 0, st>>>(
      logits, ldl, labels, rows, classes, batch, loss_rows, G, ldg);
  return cudaGetLastError();
}

cudaError_t launch_loss_mean(const float* loss_rows, int rows, float* losses, int64_t* ctr, cudaStream_t st) {
  loss_mean_kernel<<<1, 256, 0, st>>>(loss_rows, rows, losses, ctr);
  return cudaGetLastError();
}

cudaError_t launch_f32_to_bf16(const float* in, uint16_t* out, int64_t n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  f32_to_bf16_kernel<<<grid_for(n, 256), 256, 0, st>>>(in, out, n);
  return cudaGetLastError();
}

cudaError_t launch_f32_to_tf32(const float* in, float* out, int64_t n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  f32_to_tf32_kernel<<<grid_for(n, 256), 256, 0, st>>>(in, out, n);
  return cudaGetLastError();
}

cudaError_t launch_blend_materialize_tf32(const float* s, const float* l, float* out, int64_t n, float a, float b,
                                         cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  blend_materialize_tf32_kernel<<<grid_for(n, 256), 256, 0, st>>>(s, l, out, n, a, b);
  return cudaGetLastError();
}

cudaError_t launch_blend_materialize(const uint16_t* s, const uint16_t* l, uint16_t* out, int64_t n, float a, float b,
                                     cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  blend_materialize_kernel<<<grid_for(n, 256), 256, 0, st>>>(s, l, out, n, a, b);
  return cudaGetLastError();
}

cudaError_t launch_maxpool2_fwd(const uint16_t* X, uint16_t* Y, int N, int H, int W, int C, cudaStream_t st) {
  if (C % 8 || H % 2 || W % 2) return cudaErrorInvalidValue;
  const int64_t total = static_cast<int64_t>(N) * (H / 2) * (W / 2) * (C / 8);
  if (total <= 0) return cudaSuccess;
  maxpool2_fwd_kernel<<<grid_for(total, 256), 256, 0, st>>>(X, Y, N, H, W, C);
  return cudaGetLastError();
}

cudaError_t launch_maxpool2_bwd(const uint16_t* X, const uint16_t* dY, uint16_t* dX, int N, int H, int W, int C,
                                cudaStream_t st) {
  if (C % 8 || H % 2 || W % 2) return cudaErrorInvalidValue;
  const int64_t total = static_cast<int64_t>(N) * (H / 2) * (W / 2) * (C / 8);
  if (total <= 0) return cudaSuccess;
  maxpool2_bwd_kernel<<<grid_for(total, 256), 256, 0, st>>>(X, dY, dX, N, H, W, C);
  return cudaGetLastError();
}

cudaError_t launch_im2col3x3(const uint16_t* X, uint16_t* P, int N, int H, int W, int C, int ldp, cudaStream_t st) {
  const int64_t total = static_cast<int64_t>(N) * H * W * ldp;
  if (total <= 0) return cudaSuccess;
  im2col3x3_kernel<<<grid_for(total, 256), 256, 0, st>>>(X, P, N, H, W, C, ldp);
  return cudaGetLastError();
}

cudaError_t launch_im2col(const uint16_t* X, uint16_t* P, int N, int H, int W, int C, int k, int s, int p, int ldp,
                          cudaStream_t st) {
  const int Ho = (H + 2 * p - k) / s + 1, Wo = (W + 2 * p - k) / s + 1;
  const int64_t rows = static_cast<int64_t>(N) * Ho * Wo;
  if (rows <= 0) return cudaSuccess;
  if (ldp % 8 == 0 && (W * C) % 8 == 0) {
    // right padding: the last window reaches padded pixel (Wo−1)·s + k − 1 < W + 2p
    const int D0 = (p * C + 7) / 8 * 8;
    const int rowlen = (D0 + W * C + p * C + 7) / 8 * 8;
    const size_t smem_v = static_cast<size_t>(k) * rowlen * 2 + static_cast<size_t>(ldp) * 4;
    const size_t smem_s = smem_v + static_cast<size_t>(Wo) * ldp * 2;   // + the staged patch rows
    if (smem_v <= 48 * 1024) {
      // staging the patch rows through shared memory measured slower at the ResNet-50 stem
      // (639 vs 549 us per launch): opt-in TPS_IM2COL_STAGED=1
      static const bool want_staged = std::getenv("TPS_IM2COL_STAGED") && std::getenv("TPS_IM2COL_STAGED")[0] == '1';
      const int staged = want_staged && smem_s <= 48 * 1024 ? 1 : 0;
      im2col_rowtile_v<<<static_cast<unsigned>(static_cast<int64_t>(N) * Ho), 256, staged ? smem_s : smem_v, st>>>(
          X, reinterpret_cast<uint4*>(P), H, W, C, k, s, p, Ho, Wo, ldp, D0, rowlen, staged);
      return cudaGetLastError();
    }
  }
  const size_t smem = static_cast<size_t>((k * (W + 2 * p) * C + 1) & ~1) * 2 + static_cast<size_t>(ldp) * 4;
  if (ldp % 8 == 0 && smem <= 48 * 1024) {
    im2col_rowtile<<<static_cast<unsigned>(static_cast<int64_t>(N) * Ho), 256, smem, st>>>(
        X, reinterpret_cast<uint4*>(P), H, W, C, k, s, p, Ho, Wo, ldp);
    return cudaGetLastError();
  }
  if (ldp % 8 == 0) {
    const int64_t nvec = rows * (ldp / 8);
    im2col_vec8<<<grid_for(nvec, 256), 256, 0, st>>>(X, reinterpret_cast<uint4*>(P), H, W, C, k, s, p, Ho, Wo, ldp / 8,
                                                     nvec);
    return cudaGetLastError();
  }
  const int threads = ldp >= 256 ? 256 : (ldp >= 128 ? 128 : 64);
  const int blocks = static_cast<int>(std::min<int64_t>(rows, 148LL * 16));
  im2col_rows<<<blocks, threads, 0, st>>>(X, P, N, H, W, C, k, s, p, Ho, Wo, ldp, rows);
  return cudaGetLastError();
}

cudaError_t launch_col2im(const float* dP, uint16_t* dX, const uint16_t* add, int N, int H, int W, int C, int k, int s,
                          int p, int ldp, cudaStream_t st) {
  const int Ho = (H + 2 * p - k) / s + 1, Wo = (W + 2 * p - k) / s + 1;
  const int64_t total = static_cast<int64_t>(N) * H * W * C;
  if (total <= 0) return cudaSuccess;
  static const bool generic = std::getenv("TPS_COL2IM_GENERIC") != nullptr;   // A/B of the specialised kernel
  if (C % 4 == 0 && ldp % 4 == 0 && s == 2 && (k == 3 || k == 1) && !generic) {
    auto* kern = k == 3 ? col2im_vec4_ks<3, 2> : col2im_vec4_ks<1, 2>;
    kern<<<grid_for(total / 4, 256), 256, 0, st>>>(dP, reinterpret_cast<uint2*>(dX), reinterpret_cast<const uint2*>(add),
                                                   N, H, W, C, p, Ho, Wo, ldp);
  } else if (C % 4 == 0 && ldp % 4 == 0) {
    col2im_vec4<<<grid_for(total / 4, 256), 256, 0, st>>>(dP, reinterpret_cast<uint2*>(dX),
                                                          reinterpret_cast<const uint2*>(add), N, H, W, C, k, s, p, Ho,
                                                          Wo, ldp);
  } else {
    col2im_kernel<<<grid_for(total, 256), 256, 0, st>>>(dP, dX, add, N, H, W, C, k, s, p, Ho, Wo, ldp);
  }
  return cudaGetLastError();
}

// row chunks per segment: enough blocks to fill the GPU with >= 64 rows per chunk
dim3 bn_rows_grid(int rows, int C8) {
  const int tx = std::min(C8, 32), ty = 256 / tx;
  const int gx = (C8 + tx - 1) / tx;
  const int gy = std::max(1, std::min((rows + ty - 1) / ty, (148 * 8 + gx - 1) / gx));
  return dim3(gx, gy);
}

// row chunks per (segment, channel block) of the partial-sum kernels: enough blocks to fill the
// GPU (~8 per SM), but at least 16 rows per thread so the per-block fp64 shared-memory
// reduction stays small next to the streaming loop (64-row chunks made it dominate)
int bn_chunks(int segs, int seg_rows, int C) {
  const int C8 = C / 8;
  const int tx = (C % 8 == 0) ? std::min(C8, 32) : 32, ty = (C % 8 == 0) ? 256 / tx : 8;
  const int gx = (C % 8 == 0) ? (C8 + tx - 1) / tx : (C + 31) / 32;
  const int want = (8 * 148 + gx * segs - 1) / (gx * segs);
  const int cap = std::max(1, seg_rows / (16 * ty));
  return std::max(1, std::min({256, want, cap}));
}

int64_t bn_scratch_doubles(int segs, int seg_rows, int C) {
  return static_cast<int64_t>(segs) * bn_chunks(segs, seg_rows, C) * C * 2 + static_cast<int64_t>(segs) * C * 2;
}

cudaError_t launch_bn_forward(const uint16_t* x, const uint16_t* res, uint16_t* y, const float* gamma,
                              const float* beta, float* mean, float* invstd, int segs, int seg_rows, int C, int relu,
                              double* scratch, cudaStream_t st, uint8_t* relu_mask) {
  const int chunks = bn_chunks(segs, seg_rows, C);
  const int64_t rows = static_cast<int64_t>(segs) * seg_rows;
  if (!relu || C % 8) relu_mask = nullptr;
  if (C % 8 == 0) {
    const int C8 = C / 8, tx = std::min(C8, 32);
    dim3 grid((C8 + tx - 1) / tx, chunks, segs);
    bn_partial_vec<0><<<grid, tx * (256 / tx), 256 * 16 * sizeof(double), st>>>(reinterpret_cast<const uint4*>(x), nullptr,
                                                                     nullptr, nullptr, nullptr, seg_rows, C8, chunks,
                                                                     0, scratch, nullptr);
    bn_stats_final<<<(segs * C * 32 + 255) / 256, 256, 0, st>>>(scratch, chunks, C, seg_rows, segs, mean, invstd, 1e-5f);
    {
      const int C8r = C8, tx = std::min(C8r, 32);
      auto* apply = relu_mask ? bn_apply_rows<true> : bn_apply_rows<false>;
      apply<<<bn_rows_grid(static_cast<int>(rows), C8r), tx * (256 / tx), 0, st>>>(
          reinterpret_cast<const uint4*>(x), reinterpret_cast<const uint4*>(res), reinterpret_cast<uint4*>(y), gamma,
          beta, mean, invstd, static_cast<int>(rows), C8r, seg_rows, relu, relu_mask);
    }
    return cudaGetLastError();
  }
  dim3 grid((C + 31) / 32, chunks, segs);
  bn_stats_partial<<<grid, dim3(32, 8), 0, st>>>(x, seg_rows, C, chunks, scratch);
  bn_stats_final<<<(segs * C * 32 + 255) / 256, 256, 0, st>>>(scratch, chunks, C, seg_rows, segs, mean, invstd, 1e-5f);
  bn_apply_kernel<<<grid_for(rows * C, 256), 256, 0, st>>>(x, res, y, gamma, beta, mean, invstd, rows, C, seg_rows, relu);
  return cudaGetLastError();
}

cudaError_t launch_bn_forward_colsum(const float* part, const uint16_t* x, const uint16_t* res, uint16_t* y,
                                    const float* gamma, const float* beta, float* mean, float* invstd, int segs,
                                    int seg_rows, int C, int relu, double* scratch, cudaStream_t st,
                                    uint8_t* relu_mask) {
  if (seg_rows % 32 || C % 8) return cudaErrorInvalidValue;
  if (!relu) relu_mask = nullptr;
  const int gps = seg_rows / 32;
  const int64_t rows = static_cast<int64_t>(segs) * seg_rows;
  const int chunks = std::min(bn_chunks(segs, seg_rows, C), gps);
  bn_colsum_partial<<<dim3((C + 31) / 32, chunks, segs), 256, 0, st>>>(part, static_cast<int64_t>(segs) * gps, gps, C,
                                                                        chunks, scratch);
  bn_stats_final<<<(segs * C * 32 + 255) / 256, 256, 0, st>>>(scratch, chunks, C, seg_rows, segs, mean, invstd, 1e-5f);
  const int C8 = C / 8, tx = std::min(C8, 32);
  auto* apply = relu_mask ? bn_apply_rows<true> : bn_apply_rows<false>;
  apply<<<bn_rows_grid(static_cast<int>(rows), C8), tx * (256 / tx), 0, st>>>(
      reinterpret_cast<const uint4*>(x), reinterpret_cast<const uint4*>(res), reinterpret_cast<uint4*>(y), gamma, beta,
      mean, invstd, static_cast<int>(rows), C8, seg_rows, relu, relu_mask);
  return cudaGetLastError();
}

cudaError_t launch_bn_backward(const uint16_t* dy, const uint16_t* y, const uint16_t* x, const float* mean,
                               const float* invstd, const float* gs, const float* gl, float ga, float gb, int segs,
                               int seg_rows, int C, int relu, uint16_t* dx, uint16_t* dres, float* dgamma,
                               float* dbeta, double* scratch, cudaStream_t st, const uint8_t* relu_mask) {
  const int chunks = bn_chunks(segs, seg_rows, C);
  if (!relu || C % 8) relu_mask = nullptr;
  double* sums = scratch + static_cast<int64_t>(segs) * chunks * C * 2;
  if (C % 8 == 0) {
    const int C8 = C / 8, tx = std::min(C8, 32);
    const int64_t rows = static_cast<int64_t>(segs) * seg_rows;
    dim3 grid((C8 + tx - 1) / tx, chunks, segs);
    auto* partial = relu_mask ? bn_partial_vec<2> : bn_partial_vec<1>;
    partial<<<grid, tx * (256 / tx), 256 * 16 * sizeof(double), st>>>(
        reinterpret_cast<const uint4*>(dy), reinterpret_cast<const uint4*>(y), reinterpret_cast<const uint4*>(x), mean,
        invstd, seg_rows, C8, chunks, relu, scratch, relu_mask);
    float4* coef = reinterpret_cast<float4*>(sums);   // segs·C float4 = the sums region
    bn_bwd_coef<<<C, 32 * std::min(segs, kBnCoefWarps), 2 * segs * sizeof(double), st>>>(
        scratch, chunks, C, segs, seg_rows, mean, invstd, gs, gl, ga,
                                                      gb, coef, dgamma, dbeta);
    {
      const int C8r = C8, tx = std::min(C8r, 32);
      auto* apply = relu_mask ? bn_bwd_apply_rows<true> : bn_bwd_apply_rows<false>;
      apply<<<bn_rows_grid(static_cast<int>(rows), C8r), tx * (256 / tx), 0, st>>>(
          reinterpret_cast<const uint4*>(dy), reinterpret_cast<const uint4*>(y), reinterpret_cast<const uint4*>(x),
          coef, invstd, static_cast<int>(rows), C8r, seg_rows, relu, reinterpret_cast<uint4*>(dx),
          reinterpret_cast<uint4*>(dres), relu_mask);
    }
    return cudaGetLastError();
  }
  dim3 grid((C + 31) / 32, chunks, segs);
  bn_bwd_partial<<<grid, dim3(32, 8), 0, st>>>(dy, y, x, mean, invstd, seg_rows, C, chunks, relu, scratch);
  bn_bwd_final<<<(C + 255) / 256, 256, 0, st>>>(scratch, chunks, C, segs, sums, dgamma, dbeta);
  const int64_t rows = static_cast<int64_t>(segs) * seg_rows;
  bn_bwd_apply<<<grid_for(rows * C, 256), 256, 0, st>>>(dy, y, x, mean, invstd, sums, gs, gl, ga, gb, rows, C, seg_rows,
                                                        relu, dx, dres);
  return cudaGetLastError();
}

cudaError_t launch_maxpool3_fwd(const uint16_t* X, uint16_t* Y, int N, int H, int W, int C, cudaStream_t st) {
  const int Ho = (H - 1) / 2 + 1, Wo = (W - 1) / 2 + 1;
  const int64_t total = static_cast<int64_t>(N) * Ho * Wo * C;
  if (total <= 0) return cudaSuccess;
  maxpool3_fwd_kernel<<<grid_for(total, 256), 256, 0, st>>>(X, Y, N, H, W, C, Ho, Wo);
  return cudaGetLastError();
}

cudaError_t launch_maxpool3_bwd(const uint16_t* X, const uint16_t* dY, uint16_t* dX, int N, int H, int W, int C,
                                cudaStream_t st) {
  const int Ho = (H - 1) / 2 + 1, Wo = (W - 1) / 2 + 1;
  const int64_t total = static_cast<int64_t>(N) * H * W * C;
  if (total <= 0) return cudaSuccess;
  maxpool3_bwd_kernel<<<grid_for(total, 256), 256, 0, st>>>(X, dY, dX, N, H, W, C, Ho, Wo);
  return cudaGetLastError();
}

cudaError_t launch_maxpool3_fwd_idx(const uint16_t* X, uint16_t* Y, uint8_t* idx, int N, int H, int W, int C,
                                    cudaStream_t st) {
  if (C % 8) return cudaErrorInvalidValue;
  const int Ho = (H - 1) / 2 + 1, Wo = (W - 1) / 2 + 1;
  const int64_t total = static_cast<int64_t>(N) * Ho * Wo * (C / 8);
  if (total <= 0) return cudaSuccess;
  maxpool3_fwd_vec<<<grid_for(total, 256), 256, 0, st>>>(reinterpret_cast<const uint4*>(X), reinterpret_cast<uint4*>(Y),
                                                         reinterpret_cast<uint2*>(idx), N, H, W, C / 8, Ho, Wo);
  return cudaGetLastError();
}

cudaError_t launch_maxpool3_bwd_idx(const uint8_t* idx, const uint16_t* dY, uint16_t* dX, int N, int H, int W, int C,
                                    cudaStream_t st) {
  if (C % 8) return cudaErrorInvalidValue;
  const int Ho = (H - 1) / 2 + 1, Wo = (W - 1) / 2 + 1;
  const int64_t total = static_cast<int64_t>(N) * H * W * (C / 8);
  if (total <= 0) return cudaSuccess;
  maxpool3_bwd_vec<<<grid_for(total, 256), 256, 0, st>>>(reinterpret_cast<const uint2*>(idx),
                                                         reinterpret_cast<const uint4*>(dY), reinterpret_cast<uint4*>(dX),
                                                         N, H, W, C / 8, Ho, Wo);
  return cudaGetLastError();
}

cudaError_t launch_avgpool_fwd(const uint16_t* X, uint16_t* Y, int N, int HW, int C, cudaStream_t st) {
  avgpool_fwd_kernel<<<grid_for(static_cast<int64_t>(N) * C, 256), 256, 0, st>>>(X, Y, N, HW, C);
  return cudaGetLastError();
}

cudaError_t launch_avgpool_bwd(const uint16_t* dY, uint16_t* dX, int N, int HW, int C, cudaStream_t st) {
  if (C % 8 == 0) {
    avgpool_bwd_vec<<<grid_for(static_cast<int64_t>(N) * HW * (C / 8), 256), 256, 0, st>>>(
        reinterpret_cast<const uint4*>(dY), reinterpret_cast<uint4*>(dX), N, HW, C / 8);
    return cudaGetLastError();
  }
  avgpool_bwd_kernel<<<grid_for(static_cast<int64_t>(N) * HW * C, 256), 256, 0, st>>>(dY, dX, N, HW, C);
  return cudaGetLastError();
}

cudaError_t launch_add_bf16(uint16_t* out, const uint16_t* add, int64_t n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  add_bf16_kernel<<<grid_for(n, 256), 256, 0, st>>>(out, add, n);
  return cudaGetLastError();
}

cudaError_t launch_fill_synthetic(int kind, uint64_t seed, uint64_t tid, int64_t rows, int64_t cols, int64_t ld,
                                  int classes, int shift, void* dst, cudaStream_t st) {
  const uint64_t key = host_mix64(host_mix64(seed) ^ tid);
  const int64_t n = (kind == 2) ? rows : rows * ld;
  if (n <= 0) return cudaSuccess;
  fill_synthetic_kernel<<<grid_for(n, 256), 256, 0, st>>>(kind, key, rows, cols, ld, classes, shift, dst);
  return cudaGetLastError();
}

}  // namespace tps

// elementwise.cu — HBM-bound kernels of the TiMePReSt step: fused SGD/momentum update
// + bf16 version write, bias gradient (a8), softmax
// cross-entropy at the last stage (a4), the K8 blend materialiser, and the
// synthetic-input generator shared with synthgen (counter-based splitmix64).
//
// All kernels use 16-byte vector accesses, grid-stride loops sized to a multiple of the
// SM count, and fixed-order reductions (bit-reproducible run to run).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

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

// ------------------------------------------------------------------ SGD update
template <bool MOMENTUM, bool WRITE_VER>
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
    if (WRITE_VER) {
      uint2 o;
      o.x = static_cast<uint32_t>(f2bf(ww[0])) | (static_cast<uint32_t>(f2bf(ww[1])) << 16);
      o.y = static_cast<uint32_t>(f2bf(ww[2])) | (static_cast<uint32_t>(f2bf(ww[3])) << 16);
      reinterpret_cast<uint2*>(ver)[i] = o;
    }
  }
}

// ------------------------------------------------------------------ bias gradient
constexpr int BG_COLS = 256;   // columns per block (32 threads x 8 columns)
constexpr int BG_ROWS = 8;     // row lanes per block

__global__ void __launch_bounds__(256) bias_grad_partial(const uint16_t* __restrict__ G, int rows, int cols, int ldg,
                                                         int rows_per_split, float* __restrict__ part) {
  __shared__ float red[BG_ROWS][BG_COLS + 4];
  const int c0 = blockIdx.x * BG_COLS + threadIdx.x * 8;
  const int r_begin = blockIdx.y * rows_per_split;
  const int r_end = min(rows, r_begin + rows_per_split);
  float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (c0 < cols) {
    for (int r = r_begin + threadIdx.y; r < r_end; r += BG_ROWS) {
      const uint4 u = __ldg(reinterpret_cast<const uint4*>(G + static_cast<size_t>(r) * ldg + c0));
      const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] += bf2f((w[e >> 1] >> ((e & 1) * 16)) & 0xFFFFu);
    }
  }
#pragma unroll
  for (int e = 0; e < 8; ++e) red[threadIdx.y][threadIdx.x * 8 + e] = acc[e];
  __syncthreads();
  // fixed-order sum over the row lanes
  const int t = threadIdx.y * 32 + threadIdx.x;   // 0..255 -> one column each
  const int c = blockIdx.x * BG_COLS + t;
  float s = 0.f;
#pragma unroll
  for (int y = 0; y < BG_ROWS; ++y) s += red[y][t];
  if (c < cols) part[static_cast<size_t>(blockIdx.y) * cols + c] = s;
}

__global__ void bias_grad_final(const float* __restrict__ part, int splits, int cols, float* __restrict__ db) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cols) return;
  float s = 0.f;
  for (int k = 0; k < splits; ++k) s += part[static_cast<size_t>(k) * cols + c];
  db[c] = s;
}

int bias_grad_splits(int rows, int cols) {
  const int col_blocks = (cols + BG_COLS - 1) / BG_COLS;
  int splits = (2 * sm_count() + col_blocks - 1) / col_blocks;
  const int max_splits = (rows + 63) / 64;
  if (splits > max_splits) splits = max_splits;
  if (splits < 1) splits = 1;
  return splits;
}

// ------------------------------------------------------------------ softmax cross-entropy
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
  uint16_t* g = G + static_cast<size_t>(warp) * ldg;
  for (int c = lane; c < ldg; c += 32) {
    float out = 0.f;
    if (c < classes) {
      double p = exp(static_cast<double>(z[c]) - mx) / se;
      if (c == y) p -= 1.0;
      out = static_cast<float>(p / batch);
    }
    g[c] = f2bf(out);
  }
}

__global__ void loss_mean_kernel(const float* __restrict__ loss_rows, int rows, float* __restrict__ losses,
                                 int64_t idx) {
  __shared__ double red[256];
  double s = 0.0;
  for (int r = threadIdx.x; r < rows; r += blockDim.x) s += loss_rows[r];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) losses[idx] = static_cast<float>(red[0] / rows);
}

// ------------------------------------------------------------------ conversions
__global__ void f32_to_bf16_kernel(const float* __restrict__ in, uint16_t* __restrict__ out, int64_t n) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = f2bf(in[i]);
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

uint64_t host_mix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

}  // namespace

cudaError_t launch_sgd_update(float* w, float* v, const float* g, uint16_t* ver, int64_t n, float lr, float mu,
                              float wd, cudaStream_t st, int blocks_per_sm) {
  if (n <= 0) return cudaSuccess;
  if (n % 4) return cudaErrorInvalidValue;
  const int64_t n4 = n / 4;
  const int grid = grid_for(n4, 256, blocks_per_sm);
  const bool mom = mu != 0.0f;
  if (mom && ver) sgd_update_kernel<true, true><<<grid, 256, 0, st>>>(w, v, g, ver, n4, lr, mu, wd);
  else if (mom) sgd_update_kernel<true, false><<<grid, 256, 0, st>>>(w, v, g, ver, n4, lr, mu, wd);
  else if (ver) sgd_update_kernel<false, true><<<grid, 256, 0, st>>>(w, v, g, ver, n4, lr, mu, wd);
  else sgd_update_kernel<false, false><<<grid, 256, 0, st>>>(w, v, g, ver, n4, lr, mu, wd);
  return cudaGetLastError();
}

int64_t bias_grad_scratch_floats(int rows, int cols) {
  return static_cast<int64_t>(bias_grad_splits(rows, cols)) * cols;
}

cudaError_t launch_bias_grad(const uint16_t* G, int rows, int cols, int ldg, float* db, float* scratch,
                             cudaStream_t st) {
  if (cols <= 0) return cudaSuccess;
  if (cols % 8 || ldg % 8) return cudaErrorInvalidValue;
  const int splits = bias_grad_splits(rows, cols);
  const int rps = (rows + splits - 1) / splits;
  dim3 grid((cols + BG_COLS - 1) / BG_COLS, splits);
  bias_grad_partial<<<grid, dim3(32, BG_ROWS), 0, st>>>(G, rows, cols, ldg, rps, scratch);
  bias_grad_final<<<(cols + 255) / 256, 256, 0, st>>>(scratch, splits, cols, db);
  return cudaGetLastError();
}

cudaError_t launch_softmax_xent(const float* logits, int ldl, const int32_t* labels, int rows, int classes, int batch,
                                float* loss_rows, uint16_t* G, int ldg, cudaStream_t st) {
  if (rows <= 0) return cudaSuccess;
  const int warps_per_block = 8;
  softmax_xent_kernel<<<(rows + warps_per_block - 1) / warps_per_block, 32 * warps_per_block, 0, st>>>(
      logits, ldl, labels, rows, classes, batch, loss_rows, G, ldg);
  return cudaGetLastError();
}

cudaError_t launch_loss_mean(const float* loss_rows, int rows, float* losses, int64_t idx, cudaStream_t st) {
  loss_mean_kernel<<<1, 256, 0, st>>>(loss_rows, rows, losses, idx);
  return cudaGetLastError();
}

cudaError_t launch_f32_to_bf16(const float* in, uint16_t* out, int64_t n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  f32_to_bf16_kernel<<<grid_for(n, 256), 256, 0, st>>>(in, out, n);
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

cudaError_t launch_fill_synthetic(int kind, uint64_t seed, uint64_t tid, int64_t rows, int64_t cols, int64_t ld,
                                  int classes, int shift, void* dst, cudaStream_t st) {
  const uint64_t key = host_mix64(host_mix64(seed) ^ tid);
  const int64_t n = (kind == 2) ? rows : rows * ld;
  if (n <= 0) return cudaSuccess;
  fill_synthetic_kernel<<<grid_for(n, 256), 256, 0, st>>>(kind, key, rows, cols, ld, classes, shift, dst);
  return cudaGetLastError();
}

}  // namespace tps

// gemm_sm100.cu — the stage GEMMs of the TiMePReSt hot path on 5th-gen tensor cores.
//
// One persistent, warp-specialised kernel template serves the three contractions of
// a Linear layer (PAPER P:134 forward / backward):
//   forward  Y  = act(X·Wᵀ + b)             A = X  [M,K] K-major,  B = W  [N,K] K-major
//   dgrad    dX = (G·W_res) ⊙ 1[X_in > 0]    A = G  [M,K] K-major,  B = W  stored [K,N] (MN-major)
//   wgrad    dW = Gᵀ·X                       A = G  stored [K,M],   B = X  stored [K,N] (both MN-major)
// so no transpose is ever materialised.  For I-TiMePReSt the dgrad weight is the
// intermediate weight (Eq. 1, reading Z1): either α applied in the epilogue
// (EQ1: α·(G·W_stash), exact in real arithmetic) or, with BLEND, W_res = α·W_stash +
// β·W_latest formed by transform warps from two TMA-staged tiles straight into the MMA
// operand buffer — the blended weight never exists in HBM.
//
// Roles (one CTA per SM, persistent over output tiles 128 x BN):
//   warp 0      TMA producer (one elected lane): A/B tiles -> 128B-swizzled smem ring
//   warp 1      MMA issuer (one lane): tcgen05.mma kind::f16, fp32 accumulators in TMEM
//   warps 2..9  epilogue: tcgen05.ld TMEM -> registers -> smem transpose -> bias/ReLU/α/mask
//               (or the fused SGD update) -> coalesced global row segments
//   warps 10..17 (BLEND only) operand transform warps (blend in place on the stash tile)
// TMEM holds two accumulators (2·BN columns) so the epilogue of tile i overlaps the
// MMAs of tile i+1.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "gemm.h"
#include "ptx.cuh"

namespace tps {

namespace {

constexpr int BM = 128;
constexpr int BK = 64;                     // 64 bf16 = 128 B = one swizzle atom row
constexpr int A_BYTES = BM * BK * 2;       // 16 KiB
constexpr int SMEM_BUDGET = 227 * 1024;
constexpr int EPI_WARPS = 8;
// fused-update epilogue: 4 warps, each with SGD_NB buffers of one 32x32 chunk of w, v (fp32,
// 128B-swizzled TMA boxes) and the new bf16 version (64B-swizzled), refilled SGD_NB-1 chunks ahead
// fused-update epilogue warps: 4 (one per TMEM lane quarter) or 8 (two per quarter, each taking
// every other column chunk, so each SM sub-partition has two update warps to hide latency)
#ifndef TPS_SGD_WARPS
#define TPS_SGD_WARPS 4
#endif
constexpr int SGD_WARPS = TPS_SGD_WARPS;
static_assert(SGD_WARPS == 4 || SGD_WARPS == 8, "4 or 8 fused-update warps");
#ifndef TPS_SGD_NB
#define TPS_SGD_NB 2
#endif
constexpr int SGD_NB = TPS_SGD_NB;
#ifndef TPS_SGD_L2HINT
#define TPS_SGD_L2HINT 1   // fused update: w / v streamed evict-first, GEMM operands evict-last in L2
#endif
#ifndef TPS_SGD_STG
#define TPS_SGD_STG 1      // fused update: coalesced STG write-back (0 = TMA stores)
#endif
// diagnostics only (never set in a product build): 1 = skip the blend arithmetic / the
// fused-update memory traffic, to measure what the rest of the kernel costs
#ifndef TPS_DBG_XF
#define TPS_DBG_XF 0
#endif
#ifndef TPS_DBG_NOMAIN
#define TPS_DBG_NOMAIN 0   // diagnostics: no operand loads and no MMAs (times the epilogue alone)
#endif
#ifndef TPS_DBG_SGD
#define TPS_DBG_SGD 0
#endif
#ifndef TPS_SGD_PF
#define TPS_SGD_PF 0       // fused update: L2 prefetch distance in chunks (0 = off)
#endif
// (Register-staged alternatives to the TMA-fed fused-update epilogue were measured and
// dropped: w / v streamed global -> registers row per thread 142.9 us, or coalesced through a
// transposed accumulator 163.8 us, vs 88.3 us TMA-fed, at 4096 x 4096 x 2048.)
// w, v fp32 32x32 boxes (+ the bf16 version box when it is TMA-stored)
// fused update: columns per w / v chunk (32: 128B-swizzled 32x32 fp32 boxes; 16: 64B-swizzled
// 32x16 boxes, half the bytes per buffer, so twice the buffers fit the same shared memory and
// more chunks are in flight per warp)
#ifndef TPS_SGD_PF0
#define TPS_SGD_PF0 0      // fused update: L2 prefetch of the first N tiles' w / v at kernel start
#endif
#ifndef TPS_SGD_CW
#define TPS_SGD_CW 32
#endif
#ifndef TPS_SGD_LDGSTS
#define TPS_SGD_LDGSTS 1   // fused update: w / v chunks loaded by per-lane cp.async (LSU path); 0 = TMA boxes
#endif
constexpr int SGD_CW = TPS_SGD_CW;
static_assert(SGD_CW == 32 || (SGD_CW == 16 && TPS_SGD_STG), "16-column chunks need the STG write-back");
constexpr int SGD_WBYTES = 32 * SGD_CW * 4;                 // one 32-row chunk of w (or v)
constexpr int SGD_BUF = 2 * SGD_WBYTES + (TPS_SGD_STG ? 0 : 32 * 32 * 2);
constexpr int XF_WARPS = 8;                                // BLEND operand transform warps

// MH = 2 (BLEND on CTA pairs): each CTA stages TWO 128-row A blocks per K step and the pair
// computes a 512 x BN tile as two 256 x BN accumulators that share one blended B tile, so the
// blend's shared-memory passes (stash + latest read, blend written) are spread over twice the MMA
// work.  Single accumulator buffer (2·BN·MH = all 512 TMEM columns).
template <int BN, int BLEND, int SGD = 0, int CG = 1, int MH = 1>
struct Cfg {
  static_assert(MH == 1 || (MH == 2 && !SGD && CG == 2 && BN == 256), "MH = 2: plain epilogue, CTA pairs, BN 256");
  static constexpr int NEPI = SGD ? SGD_WARPS : EPI_WARPS;            // epilogue warps
  // fused-update buffers (SGD = 1: TMA-fed shared-memory chunks; SGD = 2: register-staged, none)
  static constexpr int EPI = SGD ? SGD_WARPS * SGD_NB * SGD_BUF : 0;  // fused-update buffers
  static constexpr int B_BYTES = (BN / CG) * BK * 2;   // this CTA's share of the B tile
  static constexpr int STAGE_BYTES = A_BYTES * MH + B_BYTES * (BLEND ? 2 : 1);
  static constexpr int STAGES_RAW = (SMEM_BUDGET - 2048 - EPI) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_RAW > 8 ? 8 : STAGES_RAW;
  static constexpr int THREADS = 32 * (2 + NEPI + (BLEND ? XF_WARPS : 0));
  // accumulator stages in TMEM: the fused-update variant keeps up to 4 so the MMAs can run
  // several tiles ahead of its HBM-bound epilogue
  static constexpr int ACC = MH == 2 ? 1 : ((SGD && 512 / BN >= 4) ? 4 : 2);
  static constexpr int TMEM_COLS = ACC * BN * MH;
  static constexpr int SMEM = 1024 + STAGES * STAGE_BYTES + 1024 + EPI;   // ring | barriers | epilogue
  // bytes the leader's full barrier waits for per stage: both CTAs' A (and, without BLEND, B)
  // land on it; with BLEND each CTA counts its own stash + latest B tiles on its own barrier
  static constexpr uint32_t TX = A_BYTES * MH * CG + (BLEND ? 2 * B_BYTES : B_BYTES * CG);
};

__device__ __forceinline__ void tile_coords(int t, int num_m, int num_n, int& mb, int& nb) {
  constexpr int G = 8;                      // group m-blocks so B tiles are reused from L2
  const int group = G * num_n;
  const int g = t / group;
  const int first_m = g * G;
  const int gm = min(G, num_m - first_m);
  const int r = t - g * group;
  mb = first_m + r % gm;
  nb = r / gm;
}

__device__ __forceinline__ void tile_split(int t, int num_m, int num_n, int num_k, int kper, int& mb, int& nb,
                                           int& kb0, int& kb1) {
  const int tiles = num_m * num_n;
  const int ks = t / tiles;
  tile_coords(t - ks * tiles, num_m, num_n, mb, nb);
  kb0 = ks * kper;
  kb1 = min(num_k, kb0 + kper);
}


// a[i] holds row `lane`, column i of a 32 x 32 block; afterwards a[0] of lane j = Σ_rows of
// column j.  Five butterfly rounds, each halving the columns a lane keeps (lane bit b picks the
// upper or lower half), fixed order: deterministic.
__device__ __forceinline__ void warp_transpose_sum(float (&a)[32], int lane) {
#pragma unroll
  for (int w = 16; w >= 1; w >>= 1) {
    const bool upper = (lane & w) != 0;
#pragma unroll
    for (int i = 0; i < w; ++i) {
      const float send = upper ? a[i] : a[i + w];          // the half this lane gives away
      const float keep = upper ? a[i + w] : a[i];
      a[i] = keep + __shfl_xor_sync(0xffffffffu, send, w);
    }
  }
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// TPS_HANG_DETECT (debug builds only): every mbarrier wait gives up after ~20 s of spinning,
// prints which barrier of which GEMM it was stuck on and traps, turning a hang into an error
#ifndef TPS_HANG_DETECT
#define TPS_HANG_DETECT 0
#endif
#if TPS_HANG_DETECT
#define MBAR_WAIT(tag, bar, par)                                                                             \
  do {                                                                                                       \
    const long long t0_ = clock64();                                                                         \
    while (!ptx::mbar_try_wait((bar), (par))) {                                                              \
      if (clock64() - t0_ > 40000000000LL) {                                                                 \
        printf("TPS HANG gemm<BN=%d A_MN=%d B_MN=%d BLEND=%d SGD=%d CG=%d CONV=%d> M=%d N=%d K=%d splits=%d "  \
               "im2col=%d tag=%d block=%d warp=%d par=%u\n", BN, A_MN, B_MN, BLEND, SGD, CG, CONV, args.M,      \
               args.N, args.K, args.splits, args.cv.im2col, (tag), blockIdx.x, threadIdx.x >> 5, (par));     \
        __trap();                                                                                            \
      }                                                                                                      \
    }                                                                                                        \
  } while (0)
#else
#define MBAR_WAIT(tag, bar, par) ptx::mbar_wait((bar), (par))
#endif

template <int BN, int A_MN, int B_MN, int BLEND, int SGD, int CG, int CONV, int MH = 1, int TF = 0>
__global__ void __launch_bounds__(Cfg<BN, BLEND, SGD, CG, MH>::THREADS, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ CUtensorMap tmB2, const __grid_constant__ CUtensorMap tmW,
                const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmQ, const GemmArgs args) {
  // CG = 2: a cluster of two CTAs on one TPC computes a 256 x BN tile with one
  // tcgen05.mma.cta_group::2 stream issued by the leader; each CTA stages its own 128 rows
  // of A and half of the B tile, so per-SM operand traffic drops by a third.
  using C = Cfg<BN, BLEND, SGD, CG, MH>;
  static_assert(CG == 1 || BN / CG >= 64, "pair mode: >= 64 B columns per CTA");
  constexpr int MROWS = BM * CG * MH;                 // output rows per tile
  // TF = 1 (tf32 storage, reading Z28): fp32 containers holding tf32 values, kind::tf32 MMAs.
  // A stage still holds one 128-byte swizzle row per operand row, so it covers 32 K elements
  // instead of 64 and every byte count of the ring is unchanged.
  static_assert(!TF || (CONV == CONV_NONE && TPS_SGD_STG), "tf32: Linear GEMMs, STG update write-back");
  constexpr int ESZ = TF ? 4 : 2;                     // operand element bytes
  constexpr int BKE = 128 / ESZ;                      // K elements per stage
  constexpr int MNC = 128 / ESZ;                      // MN elements per MN-major swizzle row
  constexpr int CHB = MNC * BKE * ESZ;                // bytes of one MN-major box (MNC x BKE)
  constexpr int KSTEP_MN = (TF ? 8 : 16) * 128;       // MN-major descriptor advance per MMA (K rows x 128 B)
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1 KiB alignment by pointer arithmetic on the __shared__ array itself, so every derived
  // pointer keeps the shared address space (LDS/STS rather than generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* stages = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* xform = empty + C::STAGES;
  uint64_t* tmem_full = xform + C::STAGES;
  uint64_t* tmem_empty = tmem_full + C::ACC;
  uint64_t* sgd_bar = tmem_empty + C::ACC;                                  // SGD_WARPS * SGD_NB
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sgd_bar + SGD_WARPS * SGD_NB);
  uint8_t* epi_smem = smem + C::STAGES * C::STAGE_BYTES + 1024;       // 1 KiB aligned

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = CG == 2 ? ptx::cluster_rank() : 0;
  const int cid = blockIdx.x / CG, ncl = gridDim.x / CG;
  const int num_m = (args.M + MROWS - 1) / MROWS;
  const int num_n = (args.N + BN - 1) / BN;
  const int num_k = (args.K + BKE - 1) / BKE;
  // split-K (args.splits > 1, plain fp32 epilogue only): tile t covers K blocks
  // [ks·kper, min(num_k, (ks+1)·kper)) of output tile t mod (num_m·num_n), ks = t / (num_m·num_n)
  const int num_tiles = num_m * num_n * args.splits;
  // split tail (fused update, args.split_tail): the HBM-bound update epilogue makes a tile's time
  // ~ its epilogue, so a last partial wave of R <= pairs/2 full tiles would leave R pairs doing
  // one tile more than the rest.  Those R tiles are split into 2R half tiles (N = BN/2) dealt to
  // 2R different pairs: work item i < n_full is tile i, item n_full + h is half (h & 1) of tile
  // n_full + h/2.  Every pair's half item (if any) is its last.
  constexpr bool ST_OK = SGD && CG == 2 && BN == 256 && MH == 1 && B_MN && !CONV;
  const int st_waves = num_tiles / ncl, st_rem = num_tiles - st_waves * ncl;
  const bool split_tail = ST_OK && args.split_tail && args.splits <= 1 && st_waves >= 1 && st_rem > 0 &&
                          2 * st_rem <= ncl;
  const int n_full = split_tail ? st_waves * ncl : num_tiles;
  const int n_items = split_tail ? n_full + 2 * st_rem : num_tiles;
  auto item = [&](int i, int& t, int& noff, int& nw) {
    if (i < n_full) { t = i; noff = 0; nw = BN; }
    else { const int h = i - n_full; t = n_full + h / 2; noff = (h & 1) * (BN / 2); nw = BN / 2; }
  };

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmA);
    ptx::prefetch_tmap(&tmB);
    if (BLEND) ptx::prefetch_tmap(&tmB2);
    for (int s = 0; s < C::STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
      ptx::mbar_init(&xform[s], XF_WARPS * CG);   // one arrival per transform warp (leader's is used)
    }
    for (int a = 0; a < C::ACC; ++a) {
      ptx::mbar_init(&tmem_full[a], 1);
      ptx::mbar_init(&tmem_empty[a], C::NEPI * CG);
    }
    if (SGD)
      for (int i = 0; i < SGD_WARPS * SGD_NB; ++i) ptx::mbar_init(&sgd_bar[i], TPS_SGD_LDGSTS ? 32 : 1);
    ptx::fence_barrier_init();
  }
  // CTA pairs: the cta_group::2 TMEM allocation handshakes through the PEER's shared memory
  // (reserved words + a barrier), so both CTAs must be running before either allocates; without
  // this cluster barrier a leader that starts first can arrive before its peer exists and the
  // peer then waits for that arrival forever (the rare multi-stream hang, found with cuda-gdb)
  if (CG == 2) ptx::cluster_sync();
  if (warp == 1) {
    if (CG == 2) ptx::tmem_alloc_cg2(tmem_slot, C::TMEM_COLS);
    else ptx::tmem_alloc(tmem_slot, C::TMEM_COLS);
  }
  ptx::tc_fence_before();
  if (CG == 2) ptx::cluster_sync();
  else __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // programmatic dependent launch: everything above (barrier init, TMEM allocation, tensor-map
  // prefetch) may overlap the tail of the previous kernel on the stream; no global memory is
  // read or written before that kernel has completed and flushed
  ptx::grid_dep_wait();

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      const uint64_t pol_keep = (SGD && TPS_SGD_L2HINT) ? ptx::policy_evict_last() : 0ull;
      int stage = 0;
      uint32_t phase = 0;
      for (int wi = cid; wi < n_items; wi += ncl) {
        int t, noff, nw;
        item(wi, t, noff, nw);
        int mb, nb, kb0, kb1;
        tile_split(t, num_m, num_n, num_k, args.kper, mb, nb, kb0, kb1);
        const int n0 = nb * BN + noff + static_cast<int>(rank) * (nw / CG);   // this CTA's B share
        for (int kb = kb0; kb < (TPS_DBG_NOMAIN ? kb0 : kb1); ++kb) {
          MBAR_WAIT(1, &empty[stage], phase ^ 1);
          uint8_t* const sA0 = stages + stage * C::STAGE_BYTES;
          uint8_t* sB = sA0 + MH * A_BYTES;
          if (rank == 0) ptx::mbar_expect_tx(&full[stage], C::TX - (BN - nw) * BK * 2);   // (half item: half of B)
          else if (BLEND) ptx::mbar_expect_tx(&full[stage], 2 * C::B_BYTES);   // own B tiles, own barrier
          // every load of this stage completes on the leader CTA's full barrier
          const uint32_t fb = CG == 2 ? ptx::mapa(ptx::smem_u32(&full[stage]), 0) : 0u;
          auto ld2 = [&](void* dst, const CUtensorMap* m, int x, int y) {
            if (SGD && TPS_SGD_L2HINT) {   // keep the operands resident while w / v stream through L2
              if (CG == 2) ptx::tma_load_2d_cg2_hint(dst, m, fb, x, y, pol_keep);
              else ptx::tma_load_2d_hint(dst, m, &full[stage], x, y, pol_keep);
            } else if (CG == 2) {
              ptx::tma_load_2d_cg2(dst, m, fb, x, y);
            } else {
              ptx::tma_load_2d(dst, m, &full[stage], x, y);
            }
          };
          auto ld4 = [&](void* dst, const CUtensorMap* m, int c0, int c1, int c2, int c3) {
            if (CG == 2) ptx::tma_load_4d_cg2(dst, m, fb, c0, c1, c2, c3);
            else ptx::tma_load_4d(dst, m, &full[stage], c0, c1, c2, c3);
          };
          // BLEND B tiles complete on this CTA's own barrier: its transform warps wait there
          auto ldb2 = [&](void* dst, const CUtensorMap* m, int x, int y) {
            if (BLEND) ptx::tma_load_2d(dst, m, &full[stage], x, y);
            else ld2(dst, m, x, y);
          };
          auto ldb4 = [&](void* dst, const CUtensorMap* m, int c0, int c1, int c2, int c3) {
            if (BLEND) ptx::tma_load_4d(dst, m, &full[stage], c0, c1, c2, c3);
            else ld4(dst, m, c0, c1, c2, c3);
          };
          auto ldi = [&](void* dst, const CUtensorMap* m, int c, int w, int h, int n, int ow, int oh) {
            if (CG == 2)
              ptx::tma_load_im2col_4d_cg2(dst, m, fb, c, w, h, n, static_cast<uint16_t>(ow), static_cast<uint16_t>(oh));
            else
              ptx::tma_load_im2col_4d(dst, m, &full[stage], c, w, h, n, static_cast<uint16_t>(ow),
                                      static_cast<uint16_t>(oh));
          };
          // ---- A tile(s): 128 rows x 64 K (MH of them: this CTA's rows of each 256-row half)
#pragma unroll
          for (int h = 0; h < MH; ++h) {
          uint8_t* const sA = sA0 + h * A_BYTES;
          const int m0 = mb * MROWS + h * BM * CG + static_cast<int>(rank) * BM;   // this CTA's 128 rows
          if ((CONV == CONV_FWD || CONV == CONV_DGRAD) && args.cv.im2col) {
            // im2col-mode TMA: K block kb = (filter tap, 64-channel block); the 128 output pixels
            // of this M block are 128 consecutive receptive-field origins of the traversal,
            // shifted by the tap (kw, kh); out-of-image taps read zeros (= the padding)
            const ConvGeom& g = args.cv;
            const int cpb = g.C / 64;
            const int tap = kb / cpb, c0 = (kb - tap * cpb) * 64;
            const int kh = tap / g.k, kw = tap - kh * g.k;
            const int PQ = g.Ho * g.Wo;
            const int n_img = m0 / PQ, rem = m0 - n_img * PQ, ho = rem / g.Wo, wo = rem - ho * g.Wo;
            ldi(sA, &tmA, c0, wo * g.s - g.p, ho * g.s - g.p, n_img, kw, kh);
          } else if (CONV == CONV_FWD || CONV == CONV_DGRAD) {
            // implicit im2col: K block kb = (kh, kw, 64-channel block); the 128 output pixels
            // of this M block form one (w, h, n) box of the NHWC input, shifted by (kh-1, kw-1);
            // TMA zero-fills the out-of-image halo (= the padding)
            const int cpb = args.cv.C / 64;
            const int khw = kb / cpb, c0 = (kb - khw * cpb) * 64;
            const int P = args.cv.H * args.cv.W;
            const int n_img = m0 / P, rem = m0 - n_img * P, h0 = rem / args.cv.W, w0 = rem - h0 * args.cv.W;
            ld4(sA, &tmA, c0, w0 + khw % 3 - 1, h0 + khw / 3 - 1, n_img);
          } else if (!A_MN) {
            ld2(sA, &tmA, kb * BKE, m0);
          } else {
#pragma unroll
            for (int i = 0; i < BM / MNC; ++i) ld2(sA + i * CHB, &tmA, m0 + MNC * i, kb * BKE);
          }
          }   // h
          // ---- B tile: BN/CG rows (K-major) or BN/CG columns (MN-major) x 64 K
          // BLEND: stash -> sB (the MMA operand slot), latest -> sB + B_BYTES; the transform
          // warps overwrite sB with the blend in place
          uint8_t* dB = sB;
          if (CONV == CONV_DGRAD) {
            // B[(kh',kw',co), ci] = W[co, 2-kh', 2-kw', ci]: the flipped kernel, read in place
            const int cpb = args.cv.C / 64;
            const int khw = kb / cpb, co0 = (kb - khw * cpb) * 64;
            const int kh = khw / 3, kw = khw % 3;
#pragma unroll
            for (int i = 0; i < BN / CG / 64; ++i) {
              ldb4(dB + i * 8192, &tmB, n0 + 64 * i, 2 - kw, 2 - kh, co0);
              if (BLEND) ldb4(dB + C::B_BYTES + i * 8192, &tmB2, n0 + 64 * i, 2 - kw, 2 - kh, co0);
            }
          } else if (CONV == CONV_WGRAD && args.cv.im2col) {
            // B = im2col(X): K block = 64 consecutive output pixels, column (kh, kw, ci)
            const ConvGeom& g = args.cv;
            const int PQ = g.Ho * g.Wo;
            const int p0 = kb * BK;
            const int n_img = p0 / PQ, rem = p0 - n_img * PQ, ho = rem / g.Wo, wo = rem - ho * g.Wo;
#pragma unroll
            for (int i = 0; i < BN / CG / 64; ++i) {
              const int col = n0 + 64 * i;
              const int tap = col / g.C, ci0 = col - tap * g.C;
              const int kh = tap / g.k, kw = tap - kh * g.k;
              ldi(dB + i * 8192, &tmB, ci0, wo * g.s - g.p, ho * g.s - g.p, n_img, kw, kh);
            }
          } else if (CONV == CONV_WGRAD) {
            // B = im2col(X): K block = 64 pixels (one (w,h,n) box), column (kh, kw, ci)
            const int P = args.cv.H * args.cv.W;
            const int p0 = kb * BK;
            const int n_img = p0 / P, rem = p0 - n_img * P, h0 = rem / args.cv.W, w0 = rem - h0 * args.cv.W;
#pragma unroll
            for (int i = 0; i < BN / CG / 64; ++i) {
              const int col = n0 + 64 * i;
              const int khw = col / args.cv.C, ci0 = col - khw * args.cv.C;
              ld4(dB + i * 8192, &tmB, ci0, w0 + khw % 3 - 1, h0 + khw / 3 - 1, n_img);
            }
          } else if (!B_MN) {
            ldb2(dB, &tmB, kb * BKE, n0);
            if (BLEND) ldb2(dB + C::B_BYTES, &tmB2, kb * BKE, n0);
          } else {
#pragma unroll
            for (int i = 0; i < BN / CG / MNC; ++i) {
              if (i >= nw / CG / MNC) break;      // half item: this CTA's half of the narrower B
              ldb2(dB + i * CHB, &tmB, n0 + MNC * i, kb * BKE);
              if (BLEND) ldb2(dB + C::B_BYTES + i * CHB, &tmB2, n0 + MNC * i, kb * BKE);
            }
          }
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    if (lane == 0 && rank == 0) {
      constexpr uint32_t idesc_full = TF ? ptx::make_idesc_tf32(BM * CG, BN, A_MN, B_MN)
                                         : ptx::make_idesc_bf16(BM * CG, BN, A_MN, B_MN);
      constexpr uint32_t idesc_half = TF ? ptx::make_idesc_tf32(BM * CG, BN / 2, A_MN, B_MN)
                                         : ptx::make_idesc_bf16(BM * CG, BN / 2, A_MN, B_MN);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int wi = cid; wi < n_items; wi += ncl, ++it) {
        int t, noff_, nw;
        item(wi, t, noff_, nw);
        const uint32_t idesc = nw == BN ? idesc_full : idesc_half;
        const int acc = it % C::ACC;
        const uint32_t acc_phase = (it / C::ACC) & 1;
        MBAR_WAIT(2, &tmem_empty[acc], acc_phase ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN * MH;
        int mb_, nb_, kb0, kb1;
        tile_split(t, num_m, num_n, num_k, args.kper, mb_, nb_, kb0, kb1);
        for (int kb = kb0; kb < (TPS_DBG_NOMAIN ? kb0 : kb1); ++kb) {
          MBAR_WAIT(3, &full[stage], phase);
          if (BLEND) MBAR_WAIT(4, &xform[stage], phase);
          ptx::tc_fence_after();
          const uint32_t a_addr = ptx::smem_u32(stages + stage * C::STAGE_BYTES);
          const uint32_t b_addr = a_addr + MH * A_BYTES;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {   // 4 MMAs per stage: K = 16 (bf16) or 8 (tf32) each
            // K-major SW128: +32 B per MMA K step, SBO = 8 rows x 128 B
            // MN-major SW128: +16 (bf16) / 8 (tf32) K-rows x 128 B per step, LBO = one MN chunk box
            // (64 bf16 / 32 tf32 columns: CHB bytes), SBO = 1 KiB
            // (tf32 MN-major: SWIZZLE_128B_BASE32B, SBO = 4 rows x 128 B)
            auto mn_desc = [&](uint32_t addr) {
              return TF ? ptx::make_sdesc_sw128_base32b(addr, CHB, 512) : ptx::make_sdesc_sw128(addr, CHB, 1024);
            };
            const uint64_t bd = B_MN ? mn_desc(b_addr + kk * KSTEP_MN) : ptx::make_sdesc_sw128(b_addr + kk * 32, 16, 1024);
#pragma unroll
            for (int h = 0; h < MH; ++h) {   // MH = 2: both row halves reuse this B tile
              const uint32_t ah = a_addr + h * A_BYTES;
              const uint64_t ad = A_MN ? mn_desc(ah + kk * KSTEP_MN) : ptx::make_sdesc_sw128(ah + kk * 32, 16, 1024);
              const uint32_t acc_on = (kb != kb0) || (kk != 0);
              if (TF) {
                if (CG == 2) ptx::umma_tf32_cg2(d_tmem + h * BN, ad, bd, idesc, acc_on);
                else ptx::umma_tf32(d_tmem + h * BN, ad, bd, idesc, acc_on);
              } else {
                if (CG == 2) ptx::umma_f16_cg2(d_tmem + h * BN, ad, bd, idesc, acc_on);
                else ptx::umma_f16(d_tmem + h * BN, ad, bd, idesc, acc_on);
              }
            }
          }
          if (CG == 2) ptx::umma_commit_cg2_mc(&empty[stage], 0x3);
          else ptx::umma_commit(&empty[stage]);
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
        if (CG == 2) ptx::umma_commit_cg2_mc(&tmem_full[acc], 0x3);
        else ptx::umma_commit(&tmem_full[acc]);
      }
    }
  } else if (SGD && warp < 2 + SGD_WARPS) {
    // ===================== fused SGD/momentum update epilogue (row a10) =====================
    // Each warp owns TMEM lane quarter q (32 rows of the CTA's 128) and walks the tile's 32-column
    // chunks.  w and v of a chunk arrive by TMA (128B-swizzled 32x32 fp32 boxes) SGD_NB-1 chunks
    // ahead; thread = row updates its row in place (g' = g + wd·w; v = μ·v + g'; w = w - lr·v),
    // writes bf16(w) into a 64B-swizzled box, and TMA stores write w, v, bf16(w) back.  No dW
    // round trip and no register-bound load latency.
    const int e = warp - 2;
    const int q = warp & 3;
    uint8_t* ebase = epi_smem + e * (SGD_NB * SGD_BUF);
    uint64_t* ebar = sgd_bar + e * SGD_NB;
    constexpr int CW = SGD_CW, ROWB = CW * 4, NCH = BN / CW;
    constexpr int NW = SGD_WARPS / 4;                 // warps sharing a TMEM lane quarter
    constexpr int NCHW = NCH / NW;                    // column chunks per warp per tile
    static_assert(NCH % NW == 0, "chunks split evenly between the warps of a lane quarter");
    const int half = e / 4;                            // this warp takes chunks c = half + NW·k
    const bool mom = args.mu != 0.0f;
    const uint64_t pol_stream = TPS_SGD_L2HINT ? ptx::policy_evict_first() : 0ull;
    // 16-byte chunk `ch` of row `row` in the swizzled box (128B swizzle for 128-byte rows, 64B
    // swizzle for 64-byte rows)
    auto swz = [](int row, int ch) { return CW == 32 ? (ch ^ (row & 7)) : (ch ^ ((row >> 1) & 3)); };
    // this warp's chunk i (running count: item ti = i / NCHW, chunk i % NCHW of it) -> global
    // (row0, col0); false past the last item or past a half item's chunks
    auto chunk_at = [&](int i, int& row0, int& col0) {
      const int ti = i / NCHW, cl = i - ti * NCHW;
      const int wi = cid + ti * ncl;
      if (wi >= n_items) return false;
      int t, noff, nw;
      item(wi, t, noff, nw);
      if (cl >= nw / CW / NW) return false;
      int mb, nb;
      tile_coords(t, num_m, num_n, mb, nb);
      row0 = mb * BM * CG + static_cast<int>(rank) * BM + q * 32;
      col0 = nb * BN + noff + (half + NW * cl) * CW;
      return true;
    };
    // TPS_SGD_LDGSTS: every lane copies 8 x 16 B of w (and of v) with cp.async into the same
    // 128B-swizzled layout the TMA box has (row r at r·128 B, 16-byte chunk j at (j ^ (r & 7))),
    // 4 whole rows per instruction, then arrives (noinc) on the chunk's barrier (count 32)
    auto issue_lsu = [&](int i) {
      int row0, col0;
      if (!chunk_at(i, row0, col0)) {
        ptx::cp_async_mbar_arrive_noinc(&ebar[i % SGD_NB]);   // keep the barrier's phase count
        return;
      }
      uint8_t* w_s = ebase + (i % SGD_NB) * SGD_BUF;
      const size_t ld = static_cast<size_t>(args.ldo);
      const int j = lane & 7;
      // rows past M (a tile's padding rows) and columns past N are not read (zero-filled, never
      // written back): the TMA boxes clip them the same way
      const bool col_ok = col0 + j * 4 + 4 <= args.N;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int rr = (lane >> 3) + 4 * k;
        const bool ok = col_ok && row0 + rr < args.M;
        const size_t g = ok ? static_cast<size_t>(row0 + rr) * ld + col0 + j * 4 : 0;
        const int off = rr * 128 + ((j ^ (rr & 7)) * 16);
        ptx::cp_async_16(w_s + off, args.w + g, ok ? 16u : 0u);
        if (mom) ptx::cp_async_16(w_s + SGD_WBYTES + off, args.v + g, ok ? 16u : 0u);
      }
      ptx::cp_async_mbar_arrive_noinc(&ebar[i % SGD_NB]);
    };
    auto issue = [&](int i) {            // lane 0: TMA loads of this warp's chunk i into buffer i % SGD_NB
      int row0, col0;
      if (!chunk_at(i, row0, col0)) return;
      const int buf = i % SGD_NB;
      uint8_t* w_s = ebase + buf * SGD_BUF;
      ptx::mbar_expect_tx(&ebar[buf], mom ? 2u * SGD_WBYTES : 1u * SGD_WBYTES);
      if (TPS_SGD_L2HINT) {
        ptx::tma_load_2d_hint(w_s, &tmW, &ebar[buf], col0, row0, pol_stream);
        if (mom) ptx::tma_load_2d_hint(w_s + SGD_WBYTES, &tmV, &ebar[buf], col0, row0, pol_stream);
      } else {
        ptx::tma_load_2d(w_s, &tmW, &ebar[buf], col0, row0);
        if (mom) ptx::tma_load_2d(w_s + SGD_WBYTES, &tmV, &ebar[buf], col0, row0);
      }
    };
    // L2 prefetch of chunk i (TPS_SGD_PF chunks ahead of its shared-memory load), so that load
    // hits L2 instead of waiting a full DRAM round trip; no shared memory or registers held
    auto prefetch = [&](int i) {
      int row0, col0;
      if (!chunk_at(i, row0, col0)) return;
      ptx::tma_prefetch_2d(&tmW, col0, row0);
      if (mom) ptx::tma_prefetch_2d(&tmV, col0, row0);
    };
    if (TPS_SGD_LDGSTS && !TPS_DBG_SGD)
      for (int i = 0; i < SGD_NB; ++i) issue_lsu(i);
    if (lane == 0 && !TPS_DBG_SGD) {
      if (TPS_SGD_PF)
        for (int i = SGD_NB; i < SGD_NB + TPS_SGD_PF; ++i) prefetch(i);
      if (!TPS_SGD_LDGSTS)
        for (int i = 0; i < SGD_NB; ++i) issue(i);
      // HBM idles while the first tile's MMAs run: pull the first tiles' w / v into L2 so
      // their epilogues run at L2 latency
      if (TPS_SGD_PF0)
        for (int i = SGD_NB; i < NCHW * TPS_SGD_PF0; ++i) prefetch(i);
    }
    int i = 0, it = 0;
    for (int wi = cid; wi < n_items; wi += ncl, ++it) {
      int t, noff, nw;
      item(wi, t, noff, nw);
      int mb, nb;
      tile_coords(t, num_m, num_n, mb, nb);
      const int acc = it % C::ACC;
      const uint32_t acc_phase = (it / C::ACC) & 1;
      MBAR_WAIT(5, &tmem_full[acc], acc_phase);
      ptx::tc_fence_after();
      const int row0 = mb * BM * CG + static_cast<int>(rank) * BM + q * 32;
      const int nchw = nw / CW / NW;                  // this item's chunks per warp
#pragma unroll 1
      for (int ci = 0; ci < nchw; ++ci, ++i) {
        const int c = half + NW * ci;
        uint32_t r[CW];
        if constexpr (CW == 32)
          ptx::tmem_ld_32x32b_x32(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN + c * CW,
                                  *reinterpret_cast<uint32_t(*)[32]>(r));
        else
          ptx::tmem_ld_32x32b_x16(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN + c * CW,
                                  *reinterpret_cast<uint32_t(*)[16]>(r));
        ptx::tmem_ld_wait();
        if (ci == nchw - 1) {              // last TMEM read of this warp for this tile
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if (CG == 2) ptx::mbar_arrive_remote(ptx::mapa(ptx::smem_u32(&tmem_empty[acc]), 0));
            else ptx::mbar_arrive(&tmem_empty[acc]);
          }
        }
        if (TPS_DBG_SGD) continue;
        const int buf = i % SGD_NB;
        MBAR_WAIT(6, &ebar[buf], (i / SGD_NB) & 1);
        uint8_t* w_s = ebase + buf * SGD_BUF;
        float4* wrow = reinterpret_cast<float4*>(w_s + lane * ROWB);
        float4* vrow = reinterpret_cast<float4*>(w_s + SGD_WBYTES + lane * ROWB);
        uint8_t* qrow = w_s + 2 * SGD_WBYTES + lane * 64;
#pragma unroll
        for (int j = 0; j < CW / 4; ++j) {
          const int pos = swz(lane, j);                   // 16B chunk j of row `lane`
          float4 wv = wrow[pos];
          float4 vv = mom ? vrow[pos] : make_float4(0.f, 0.f, 0.f, 0.f);
          float* wp = &wv.x;
          float* vp = &vv.x;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const float g = __uint_as_float(r[4 * j + k]);
            const float gp = __fadd_rn(g, __fmul_rn(args.wd, wp[k]));
            float upd = gp;
            if (mom) {
              vp[k] = __fadd_rn(__fmul_rn(args.mu, vp[k]), gp);
              upd = vp[k];
            }
            wp[k] = __fsub_rn(wp[k], __fmul_rn(args.lr, upd));
          }
          wrow[pos] = wv;
          if (mom) vrow[pos] = vv;
          if (!TPS_SGD_STG) {
            const int qpos = (j >> 1) ^ ((lane >> 1) & 3);  // 64B swizzle of the bf16 row
            *reinterpret_cast<uint2*>(qrow + qpos * 16 + (j & 1) * 8) =
                make_uint2(pack_bf16(wv.x, wv.y), pack_bf16(wv.z, wv.w));
          }
        }
        if (TPS_SGD_STG) {
          // coalesced write-back: after the row pass, lanes re-read the (swizzled) buffer by
          // 16-byte column chunks so each store instruction writes whole 128-byte row segments;
          // the buffer can be refilled as soon as its contents sit in registers
          __syncwarp();
          const int col0 = nb * BN + noff + c * CW;
          const size_t ld = static_cast<size_t>(args.ldo);
          constexpr int LPR = CW / 4;                     // lanes per row segment (16 B each)
#pragma unroll
          for (int k = 0; k < 32 / (32 / LPR); ++k) {
            const int rr = (32 / LPR) * k + lane / LPR, ch = lane % LPR;
            const int pos = swz(rr, ch);
            const int grow = row0 + rr, gcol = col0 + ch * 4;
            const float4 wv = *reinterpret_cast<const float4*>(w_s + rr * ROWB + pos * 16);
            float4 vv;
            if (mom) vv = *reinterpret_cast<const float4*>(w_s + SGD_WBYTES + rr * ROWB + pos * 16);
            if (grow < args.M && gcol < args.N) {
              __stcs(reinterpret_cast<float4*>(args.w + grow * ld + gcol), wv);
              if (mom) __stcs(reinterpret_cast<float4*>(args.v + grow * ld + gcol), vv);
              if (TF)   // new tf32 version
                *reinterpret_cast<float4*>(reinterpret_cast<float*>(args.ver) + grow * ld + gcol) =
                    make_float4(ptx::rna_tf32(wv.x), ptx::rna_tf32(wv.y), ptx::rna_tf32(wv.z), ptx::rna_tf32(wv.w));
              else      // new bf16 version
                *reinterpret_cast<uint2*>(args.ver + grow * ld + gcol) =
                    make_uint2(pack_bf16(wv.x, wv.y), pack_bf16(wv.z, wv.w));
            }
          }
          ptx::fence_proxy_async_smem();   // generic reads of the buffer before the async refill
          __syncwarp();
          if (TPS_SGD_LDGSTS) issue_lsu(i + SGD_NB);
          if (lane == 0) {
            if (!TPS_SGD_LDGSTS) issue(i + SGD_NB);
            if (TPS_SGD_PF) prefetch(i + SGD_NB + TPS_SGD_PF);
          }
          __syncwarp();
          continue;
        }
        ptx::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          const int col0 = nb * BN + noff + c * CW;
          if (TPS_SGD_L2HINT) {
            ptx::tma_store_2d_hint(&tmW, w_s, col0, row0, pol_stream);
            if (mom) ptx::tma_store_2d_hint(&tmV, w_s + SGD_WBYTES, col0, row0, pol_stream);
            ptx::tma_store_2d_hint(&tmQ, w_s + 2 * SGD_WBYTES, col0, row0, pol_stream);
          } else {
            ptx::tma_store_2d(&tmW, w_s, col0, row0);
            if (mom) ptx::tma_store_2d(&tmV, w_s + SGD_WBYTES, col0, row0);
            ptx::tma_store_2d(&tmQ, w_s + 2 * SGD_WBYTES, col0, row0);
          }
          ptx::bulk_commit();
          ptx::bulk_wait_read<0>();       // the buffer may be refilled once the stores read it
          issue(i + SGD_NB);
          if (TPS_SGD_PF) prefetch(i + SGD_NB + TPS_SGD_PF);
        }
        __syncwarp();
      }
    }
    if (lane == 0) ptx::bulk_wait_all();
  } else if (!SGD && warp < 2 + EPI_WARPS) {
    // ===================== epilogue =====================
    // 8 warps: warp w reads TMEM lane quarter (w % 4) and handles one half of the tile's
    // 32-column chunks; thread = row, 16-byte vector loads/stores along the row.
    const int e = warp - 2;
    const int q = warp & 3;                 // TMEM lane quarter this warp may access
    const int half = e >> 2;                // which half of the tile's columns this warp owns
    constexpr int CPW = BN / 64;            // 32-column chunks per warp per tile
    int it = 0;
    for (int t = cid; t < num_tiles; t += ncl, ++it) {
      int mb, nb, kb0, kb1;
      tile_split(t, num_m, num_n, num_k, args.kper, mb, nb, kb0, kb1);
      // split-K partials go to slice ks of the fp32 workspace (same ld), reduced afterwards
      void* const outp = args.splits > 1
          ? static_cast<void*>(args.ws + static_cast<size_t>(kb0 / args.kper) * args.M * args.ldo)
          : args.out;
      const int acc = it % C::ACC;
      const uint32_t acc_phase = (it / C::ACC) & 1;
      MBAR_WAIT(7, &tmem_full[acc], acc_phase);
      ptx::tc_fence_after();
#pragma unroll 1
      for (int h = 0; h < MH; ++h) {
      const int row0 = mb * MROWS + h * BM * CG + static_cast<int>(rank) * BM + q * 32;
#pragma unroll 1
      for (int ci = 0; ci < CPW; ++ci) {
        const int c = half * CPW + ci;
        uint32_t r[32];
        ptx::tmem_ld_32x32b_x32(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + (acc * MH + h) * BN + c * 32, r);
        ptx::tmem_ld_wait();
        if (ci == CPW - 1 && h == MH - 1) {   // last TMEM read of this warp for this tile
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if (CG == 2) ptx::mbar_arrive_remote(ptx::mapa(ptx::smem_u32(&tmem_empty[acc]), 0));
            else ptx::mbar_arrive(&tmem_empty[acc]);
          }
        }
        // plain epilogue: thread = row, 16-byte vector loads/stores along the row
        const int grow = row0 + lane;
        const int gcol = nb * BN + c * 32;
        if (gcol >= args.N) continue;                    // warp-uniform
        const bool live = grow < args.M;
        float v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
        if (live) {
        const int nchunk = min(4, (args.N - gcol) >> 3);   // 8-column chunks inside N
        if (args.alpha != 1.0f) {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = __fmul_rn(v[i], args.alpha);
        }
        if (args.bias) {
          const float* bp = args.bias + gcol;
#pragma unroll
          for (int ch = 0; ch < 4; ++ch) {
            if (ch < nchunk) {
              const float4 b0 = __ldg(reinterpret_cast<const float4*>(bp + ch * 8));
              const float4 b1 = __ldg(reinterpret_cast<const float4*>(bp + ch * 8 + 4));
              v[ch * 8 + 0] = __fadd_rn(v[ch * 8 + 0], b0.x);
              v[ch * 8 + 1] = __fadd_rn(v[ch * 8 + 1], b0.y);
              v[ch * 8 + 2] = __fadd_rn(v[ch * 8 + 2], b0.z);
              v[ch * 8 + 3] = __fadd_rn(v[ch * 8 + 3], b0.w);
              v[ch * 8 + 4] = __fadd_rn(v[ch * 8 + 4], b1.x);
              v[ch * 8 + 5] = __fadd_rn(v[ch * 8 + 5], b1.y);
              v[ch * 8 + 6] = __fadd_rn(v[ch * 8 + 6], b1.z);
              v[ch * 8 + 7] = __fadd_rn(v[ch * 8 + 7], b1.w);
            }
          }
        }
        if (args.relu) {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = fmaxf(v[i], 0.0f);
        }
        if (args.mask && TF) {   // fp32 (tf32) mask source: positive = sign clear, nonzero
          const uint4* mp = reinterpret_cast<const uint4*>(reinterpret_cast<const uint32_t*>(args.mask) +
                                                           static_cast<size_t>(grow) * args.ldm + gcol);
#pragma unroll
          for (int ch = 0; ch < 8; ++ch) {
            if ((ch >> 1) < nchunk) {
              const uint4 mv = __ldg(mp + ch);
              const uint32_t w[4] = {mv.x, mv.y, mv.z, mv.w};
#pragma unroll
              for (int e2 = 0; e2 < 4; ++e2)
                if (!(((w[e2] & 0x80000000u) == 0u) && ((w[e2] & 0x7FFFFFFFu) != 0u))) v[ch * 4 + e2] = 0.0f;
            }
          }
        } else if (args.mask) {
          const uint4* mp = reinterpret_cast<const uint4*>(args.mask + static_cast<size_t>(grow) * args.ldm + gcol);
#pragma unroll
          for (int ch = 0; ch < 4; ++ch) {
            if (ch < nchunk) {
              const uint4 mv = __ldg(mp + ch);
              const uint32_t w[4] = {mv.x, mv.y, mv.z, mv.w};
#pragma unroll
              for (int e2 = 0; e2 < 8; ++e2) {
                const uint32_t h = (w[e2 >> 1] >> ((e2 & 1) * 16)) & 0xFFFFu;
                const bool pos = ((h & 0x8000u) == 0u) && ((h & 0x7FFFu) != 0u);
                if (!pos) v[ch * 8 + e2] = 0.0f;
              }
            }
          }
        }
        if (args.addend && !TF) {
          const uint4* ap = reinterpret_cast<const uint4*>(args.addend + static_cast<size_t>(grow) * args.ldo + gcol);
#pragma unroll
          for (int ch = 0; ch < 4; ++ch) {
            if (ch < nchunk) {
              const uint4 av = ap[ch];
              const uint32_t w[4] = {av.x, av.y, av.z, av.w};
#pragma unroll
              for (int e2 = 0; e2 < 8; ++e2)
                v[ch * 8 + e2] = __fadd_rn(v[ch * 8 + e2], __uint_as_float(((w[e2 >> 1] >> ((e2 & 1) * 16)) & 0xFFFFu) << 16));
            }
          }
        }
        if (TF && !args.out_f32) {   // tf32 store (reading Z28)
          float* op = reinterpret_cast<float*>(outp) + static_cast<size_t>(grow) * args.ldo + gcol;
#pragma unroll
          for (int ch = 0; ch < 4; ++ch) {
            if (ch < nchunk) {
              reinterpret_cast<float4*>(op + ch * 8)[0] =
                  make_float4(ptx::rna_tf32(v[ch * 8]), ptx::rna_tf32(v[ch * 8 + 1]), ptx::rna_tf32(v[ch * 8 + 2]),
                              ptx::rna_tf32(v[ch * 8 + 3]));
              reinterpret_cast<float4*>(op + ch * 8)[1] =
                  make_float4(ptx::rna_tf32(v[ch * 8 + 4]), ptx::rna_tf32(v[ch * 8 + 5]), ptx::rna_tf32(v[ch * 8 + 6]),
                              ptx::rna_tf32(v[ch * 8 + 7]));
            }
          }
        } else if (args.out_f32) {
          float* op = reinterpret_cast<float*>(outp) + static_cast<size_t>(grow) * args.ldo + gcol;
#pragma unroll
          for (int ch = 0; ch < 4; ++ch) {
            if (ch < nchunk) {
              reinterpret_cast<float4*>(op + ch * 8)[0] = make_float4(v[ch * 8], v[ch * 8 + 1], v[ch * 8 + 2], v[ch * 8 + 3]);
              reinterpret_cast<float4*>(op + ch * 8)[1] =
                  make_float4(v[ch * 8 + 4], v[ch * 8 + 5], v[ch * 8 + 6], v[ch * 8 + 7]);
            }
          }
        } else {
          __nv_bfloat16* op = reinterpret_cast<__nv_bfloat16*>(outp) + static_cast<size_t>(grow) * args.ldo + gcol;
#pragma unroll
          for (int ch = 0; ch < 4; ++ch) {
            if (ch < nchunk) {
              uint4 o;
              o.x = pack_bf16(v[ch * 8 + 0], v[ch * 8 + 1]);
              o.y = pack_bf16(v[ch * 8 + 2], v[ch * 8 + 3]);
              o.z = pack_bf16(v[ch * 8 + 4], v[ch * 8 + 5]);
              o.w = pack_bf16(v[ch * 8 + 6], v[ch * 8 + 7]);
              reinterpret_cast<uint4*>(op)[ch] = o;
            }
          }
        }
        }   // live
        if (args.colsum && args.splits <= 1 && row0 < args.M) {   // warp-uniform: the group holds rows
          // column sums of the values as STORED (bf16-rounded unless fp32 out) over this warp's 32
          // rows: a fixed butterfly transposes the reduction so lane j ends with column gcol + j;
          // written as one partial row per 32-row group (Σx, and Σx² in a second plane if asked)
          float a[32], q2[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const float x = !live ? 0.0f
                                  : (args.out_f32 ? v[i] : (TF ? ptx::rna_tf32(v[i]) : __bfloat162float(__float2bfloat16_rn(v[i]))));
            a[i] = x;
            q2[i] = x * x;
          }
          warp_transpose_sum(a, lane);
          if (args.colsum_sq) warp_transpose_sum(q2, lane);
          const int64_t grp = row0 >> 5;
          const int64_t groups = (args.M + 31) >> 5;
          if (gcol + lane < args.N) {
            args.colsum[grp * args.N + gcol + lane] = a[0];
            if (args.colsum_sq) args.colsum[(groups + grp) * args.N + gcol + lane] = q2[0];
          }
        }
      }
      }   // h
    }
  } else if (BLEND) {
    // ===================== operand transform: W_res = α·W_stash + β·W_latest =====================
    // identical swizzled layouts: the blend is elementwise on raw 16-byte chunks, written back
    // over the stash tile (each thread reads and writes only its own chunks); packed fp32x2
    // arithmetic: bf16(fma(β, W_latest, fp32(α·W_stash))) (reading Z14)
    const int tt = threadIdx.x - (2 + C::NEPI) * 32;    // 0 .. 32·XF_WARPS-1
    const uint64_t xa2 = ptx::f32x2_splat(args.xa), xb2 = ptx::f32x2_splat(args.xb);
    int stage = 0;
    uint32_t phase = 0;
    for (int t = cid; t < num_tiles; t += ncl) {
      for (int kb = 0; kb < num_k; ++kb) {
        MBAR_WAIT(8, &full[stage], phase);
        uint8_t* sB = stages + stage * C::STAGE_BYTES + MH * A_BYTES;
        uint4* s = reinterpret_cast<uint4*>(sB);
        const uint4* l = reinterpret_cast<const uint4*>(sB + C::B_BYTES);
#pragma unroll
        for (int i = tt; i < (TPS_DBG_XF ? 0 : C::B_BYTES / 16); i += XF_WARPS * 32) {
          if (TF) {   // 4 tf32 values per 16-byte chunk
            const ulonglong2 a = reinterpret_cast<const ulonglong2*>(s)[i];
            const ulonglong2 b = reinterpret_cast<const ulonglong2*>(l)[i];
            reinterpret_cast<ulonglong2*>(s)[i] =
                make_ulonglong2(ptx::blend_tf32x2(a.x, b.x, xa2, xb2), ptx::blend_tf32x2(a.y, b.y, xa2, xb2));
          } else {
            const uint4 a = s[i];
            const uint4 b = l[i];
            s[i] = make_uint4(ptx::blend_bf16x2(a.x, b.x, xa2, xb2), ptx::blend_bf16x2(a.y, b.y, xa2, xb2),
                              ptx::blend_bf16x2(a.z, b.z, xa2, xb2), ptx::blend_bf16x2(a.w, b.w, xa2, xb2));
          }
        }
        ptx::fence_proxy_async_smem();
        __syncwarp();                   // one arrival per warp once all its lanes have fenced
        if (lane == 0) {
          if (CG == 2) ptx::mbar_arrive_remote(ptx::mapa(ptx::smem_u32(&xform[stage]), 0));
          else ptx::mbar_arrive(&xform[stage]);
        }
        if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
      }
    }
  }

  ptx::tc_fence_before();
  if (CG == 2) ptx::cluster_sync();
  else __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    if (CG == 2) {
      ptx::tmem_relinquish_cg2();
      ptx::tmem_dealloc_cg2(tmem_base, C::TMEM_COLS);
    } else {
      ptx::tmem_relinquish();
      ptx::tmem_dealloc(tmem_base, C::TMEM_COLS);
    }
  }
}


// ---------------------------------------------------------------- dual backward launch
// Layer k's weight gradient + fused update (tiles "W": K = batch rows, HBM-heavy epilogue) and
// layer k-1's input gradient (tiles "D": K = layer width, light epilogue) in ONE persistent
// launch.  The split backward used to run them as two kernels that queued for the same SMs, so
// each SM's tensor pipe idled while its update epilogue streamed w / v.  Here every CTA pair
// walks a list mixing both kinds: the MMAs of a D tile run while the epilogue warps stream the
// previous W tile's update.  Each tile is computed exactly as by the separate kernels (same
// operand staging, instruction shapes and K order), so the results are bit-identical.
//
// Work split (closed form, no device memory, graph-safe): D tiles are dealt round-robin over
// the cluster pairs; W tiles are given out in consecutive runs so that every pair's MMA work
// (in K blocks) is within one W tile of the average.  Inside a pair's list the D tiles are
// spread evenly among the W tiles (a W tile first, a D tile last: its epilogue is the short one).
__host__ __device__ inline int64_t dual_dpre(int c, int n_d, int ncl) {
  return static_cast<int64_t>(n_d / ncl) * c + (c < n_d % ncl ? c : n_d % ncl);
}
__host__ __device__ inline int dual_wpre(int c, int n_d, int n_w, int kd, int kw, int ncl) {
  const int64_t U = static_cast<int64_t>(n_d) * kd + static_cast<int64_t>(n_w) * kw;
  const int64_t r = static_cast<int64_t>(c) * U / ncl - static_cast<int64_t>(kd) * dual_dpre(c, n_d, ncl);
  const int64_t w = r <= 0 ? 0 : (r + kw / 2) / kw;
  return static_cast<int>(w < n_w ? w : n_w);
}

template <int BN, int CG>
__global__ void __launch_bounds__(Cfg<BN, 0, 1, CG>::THREADS, 1)
    bwd_dual_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const __grid_constant__ CUtensorMap tmDA, const __grid_constant__ CUtensorMap tmDB,
                    const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmV,
                    const GemmArgs args, const DualArgs dg) {
  using C = Cfg<BN, 0, 1, CG>;
  static_assert(CG == 2 && TPS_SGD_STG, "dual launch: CTA pairs, STG write-back");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* stages = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tmem_full = empty + 2 * C::STAGES;
  uint64_t* tmem_empty = tmem_full + C::ACC;
  uint64_t* sgd_bar = tmem_empty + C::ACC;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sgd_bar + SGD_WARPS * SGD_NB);
  uint8_t* epi_smem = smem + C::STAGES * C::STAGE_BYTES + 1024;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = ptx::cluster_rank();
  const int cid = blockIdx.x / CG, ncl = gridDim.x / CG;
  const int wm = (args.M + BM * CG - 1) / (BM * CG), wn = (args.N + BN - 1) / BN, kw = (args.K + BK - 1) / BK;
  const int dm = (dg.M + BM * CG - 1) / (BM * CG), dn = (dg.N + BN - 1) / BN, kd = (dg.K + BK - 1) / BK;
  const int n_w = wm * wn, n_d = dm * dn;
  const int d_c = cid < n_d ? (n_d - cid - 1) / ncl + 1 : 0;
  const int w0 = dual_wpre(cid, n_d, n_w, kd, kw, ncl);
  const int w_c = dual_wpre(cid + 1, n_d, n_w, kd, kw, ncl) - w0;
  const int len = d_c + w_c;
  // position k of this pair's list -> (kind, tile index within its GEMM)
  auto at = [&](int k, bool& is_d, int& t) {
    const int before = static_cast<int>(static_cast<int64_t>(k) * d_c / len);     // D tiles before k
    is_d = static_cast<int>(static_cast<int64_t>(k + 1) * d_c / len) > before;
    t = is_d ? cid + before * ncl : w0 + (k - before);
  };

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmA);
    ptx::prefetch_tmap(&tmB);
    ptx::prefetch_tmap(&tmDA);
    ptx::prefetch_tmap(&tmDB);
    for (int s = 0; s < C::STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < C::ACC; ++a) {
      ptx::mbar_init(&tmem_full[a], 1);
      ptx::mbar_init(&tmem_empty[a], C::NEPI * CG);
    }
    for (int i = 0; i < SGD_WARPS * SGD_NB; ++i) ptx::mbar_init(&sgd_bar[i], 1);
    ptx::fence_barrier_init();
  }
  ptx::cluster_sync();   // both CTAs resident before the pair's TMEM allocation (see gemm_kernel)
  if (warp == 1) ptx::tmem_alloc_cg2(tmem_slot, C::TMEM_COLS);
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  ptx::grid_dep_wait();

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      const uint64_t pol_keep = TPS_SGD_L2HINT ? ptx::policy_evict_last() : 0ull;
      int stage = 0;
      uint32_t phase = 0;
      for (int k = 0; k < len; ++k) {
        bool is_d;
        int t, mb, nb;
        at(k, is_d, t);
        tile_coords(t, is_d ? dm : wm, is_d ? dn : wn, mb, nb);
        const int m0 = mb * BM * CG + static_cast<int>(rank) * BM;
        const int n0 = nb * BN + static_cast<int>(rank) * (BN / CG);
        const int nk = is_d ? kd : kw;
        const CUtensorMap* mA = is_d ? &tmDA : &tmA;
        const CUtensorMap* mB = is_d ? &tmDB : &tmB;
        for (int kb = 0; kb < nk; ++kb) {
          MBAR_WAIT(1, &empty[stage], phase ^ 1);
          uint8_t* sA = stages + stage * C::STAGE_BYTES;
          uint8_t* sB = sA + A_BYTES;
          if (rank == 0) ptx::mbar_expect_tx(&full[stage], C::TX);
          const uint32_t fb = ptx::mapa(ptx::smem_u32(&full[stage]), 0);
          auto ld2 = [&](void* dst, const CUtensorMap* m, int x, int y) {
            if (TPS_SGD_L2HINT) ptx::tma_load_2d_cg2_hint(dst, m, fb, x, y, pol_keep);
            else ptx::tma_load_2d_cg2(dst, m, fb, x, y);
          };
          if (is_d) {
            ld2(sA, mA, kb * BK, m0);                                   // G [M, K], K-major
          } else {
#pragma unroll
            for (int i = 0; i < BM / 64; ++i) ld2(sA + i * 8192, mA, m0 + 64 * i, kb * BK);   // stored [K, M]
          }
#pragma unroll
          for (int i = 0; i < BN / CG / 64; ++i) ld2(sB + i * 8192, mB, n0 + 64 * i, kb * BK);  // stored [K, N]
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (leader CTA) =====================
    if (lane == 0 && rank == 0) {
      constexpr uint32_t idesc_w = ptx::make_idesc_bf16(BM * CG, BN, 1, 1);
      constexpr uint32_t idesc_d = ptx::make_idesc_bf16(BM * CG, BN, 0, 1);
      int stage = 0;
      uint32_t phase = 0;
      for (int k = 0; k < len; ++k) {
        const int acc = k % C::ACC;
        MBAR_WAIT(2, &tmem_empty[acc], ((k / C::ACC) & 1) ^ 1);
        ptx::tc_fence_after();
        bool is_d;
        int t;
        at(k, is_d, t);
        const uint32_t d_tmem = tmem_base + acc * BN;
        const int nk = is_d ? kd : kw;
        for (int kb = 0; kb < nk; ++kb) {
          MBAR_WAIT(3, &full[stage], phase);
          ptx::tc_fence_after();
          const uint32_t a_addr = ptx::smem_u32(stages + stage * C::STAGE_BYTES);
          const uint32_t b_addr = a_addr + A_BYTES;
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            const uint64_t ad = is_d ? ptx::make_sdesc_sw128(a_addr + kk * 32, 16, 1024)
                                     : ptx::make_sdesc_sw128(a_addr + kk * 2048, 8192, 1024);
            const uint64_t bd = ptx::make_sdesc_sw128(b_addr + kk * 2048, 8192, 1024);
            ptx::umma_f16_cg2(d_tmem, ad, bd, is_d ? idesc_d : idesc_w, (kb != 0) || (kk != 0));
          }
          ptx::umma_commit_cg2_mc(&empty[stage], 0x3);
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
        ptx::umma_commit_cg2_mc(&tmem_full[acc], 0x3);
      }
    }
  } else if (warp < 2 + SGD_WARPS) {
    // ===================== epilogue: fused update (W tiles) / masked bf16 store (D tiles) ==========
    const int e = warp - 2;
    const int q = warp & 3;
    uint8_t* ebase = epi_smem + e * (SGD_NB * SGD_BUF);
    uint64_t* ebar = sgd_bar + e * SGD_NB;
    constexpr int CW = SGD_CW, ROWB = CW * 4, NCH = BN / CW;
    constexpr int NW = SGD_WARPS / 4;
    constexpr int NCHW = NCH / NW;
    constexpr int NCHD = BN / 32 / NW;                 // 32-column D chunks per warp per tile
    const int half = e / 4;
    const bool mom = args.mu != 0.0f;
    const uint64_t pol_stream = TPS_SGD_L2HINT ? ptx::policy_evict_first() : 0ull;
    auto swz = [](int row, int ch) { return CW == 32 ? (ch ^ (row & 7)) : (ch ^ ((row >> 1) & 3)); };
    auto issue = [&](int i) {            // lane 0: TMA loads of this warp's W chunk i (W tiles only)
      const int ti = i / NCHW, c = half + NW * (i - ti * NCHW);
      if (ti >= w_c) return;
      int mb, nb;
      tile_coords(w0 + ti, wm, wn, mb, nb);
      const int row0 = mb * BM * CG + static_cast<int>(rank) * BM + q * 32;
      const int col0 = nb * BN + c * CW;
      const int buf = i % SGD_NB;
      uint8_t* w_s = ebase + buf * SGD_BUF;
      ptx::mbar_expect_tx(&ebar[buf], mom ? 2u * SGD_WBYTES : 1u * SGD_WBYTES);
      if (TPS_SGD_L2HINT) {
        ptx::tma_load_2d_hint(w_s, &tmW, &ebar[buf], col0, row0, pol_stream);
        if (mom) ptx::tma_load_2d_hint(w_s + SGD_WBYTES, &tmV, &ebar[buf], col0, row0, pol_stream);
      } else {
        ptx::tma_load_2d(w_s, &tmW, &ebar[buf], col0, row0);
        if (mom) ptx::tma_load_2d(w_s + SGD_WBYTES, &tmV, &ebar[buf], col0, row0);
      }
    };
    if (lane == 0)
      for (int i = 0; i < SGD_NB; ++i) issue(i);
    int i = 0;
    for (int k = 0; k < len; ++k) {
      bool is_d;
      int t, mb, nb;
      at(k, is_d, t);
      tile_coords(t, is_d ? dm : wm, is_d ? dn : wn, mb, nb);
      const int acc = k % C::ACC;
      MBAR_WAIT(5, &tmem_full[acc], (k / C::ACC) & 1);
      ptx::tc_fence_after();
      const int row0 = mb * BM * CG + static_cast<int>(rank) * BM + q * 32;
      if (is_d) {
        // ---- input gradient: α, ReLU mask, bf16 store (thread = row, as gemm_kernel's epilogue)
#pragma unroll 1
        for (int ci = 0; ci < NCHD; ++ci) {
          const int c = half + NW * ci;
          uint32_t r[32];
          ptx::tmem_ld_32x32b_x32(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN + c * 32, r);
          ptx::tmem_ld_wait();
          if (ci == NCHD - 1) {
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive_remote(ptx::mapa(ptx::smem_u32(&tmem_empty[acc]), 0));
          }
          const int grow = row0 + lane;
          const int gcol = nb * BN + c * 32;
          if (gcol < dg.N && grow < dg.M) {     // (rows past M: lane-divergent, reconverges below)
          const int nchunk = min(4, (dg.N - gcol) >> 3);
          float v[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
          if (dg.alpha != 1.0f) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = __fmul_rn(v[j], dg.alpha);
          }
          if (dg.mask) {
            const uint4* mp = reinterpret_cast<const uint4*>(dg.mask + static_cast<size_t>(grow) * dg.ldm + gcol);
#pragma unroll
            for (int ch = 0; ch < 4; ++ch) {
              if (ch < nchunk) {
                const uint4 mv = __ldg(mp + ch);
                const uint32_t w[4] = {mv.x, mv.y, mv.z, mv.w};
#pragma unroll
                for (int e2 = 0; e2 < 8; ++e2) {
                  const uint32_t h = (w[e2 >> 1] >> ((e2 & 1) * 16)) & 0xFFFFu;
                  const bool pos = ((h & 0x8000u) == 0u) && ((h & 0x7FFFu) != 0u);
                  if (!pos) v[ch * 8 + e2] = 0.0f;
                }
              }
            }
          }
          __nv_bfloat16* op = reinterpret_cast<__nv_bfloat16*>(dg.out) + static_cast<size_t>(grow) * dg.ldo + gcol;
#pragma unroll
          for (int ch = 0; ch < 4; ++ch) {
            if (ch < nchunk) {
              uint4 o;
              o.x = pack_bf16(v[ch * 8 + 0], v[ch * 8 + 1]);
              o.y = pack_bf16(v[ch * 8 + 2], v[ch * 8 + 3]);
              o.z = pack_bf16(v[ch * 8 + 4], v[ch * 8 + 5]);
              o.w = pack_bf16(v[ch * 8 + 6], v[ch * 8 + 7]);
              reinterpret_cast<uint4*>(op)[ch] = o;
            }
          }
          }   // live
          __syncwarp();
        }
        continue;
      }
      // ---- weight gradient: the fused SGD/momentum update (as gemm_kernel's SGD epilogue)
#pragma unroll 1
      for (int ci = 0; ci < NCHW; ++ci, ++i) {
        const int c = half + NW * ci;
        uint32_t r[CW];
        if constexpr (CW == 32)
          ptx::tmem_ld_32x32b_x32(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN + c * CW,
                                  *reinterpret_cast<uint32_t(*)[32]>(r));
        else
          ptx::tmem_ld_32x32b_x16(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN + c * CW,
                                  *reinterpret_cast<uint32_t(*)[16]>(r));
        ptx::tmem_ld_wait();
        if (ci == NCHW - 1) {
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive_remote(ptx::mapa(ptx::smem_u32(&tmem_empty[acc]), 0));
        }
        const int buf = i % SGD_NB;
        MBAR_WAIT(6, &ebar[buf], (i / SGD_NB) & 1);
        uint8_t* w_s = ebase + buf * SGD_BUF;
        float4* wrow = reinterpret_cast<float4*>(w_s + lane * ROWB);
        float4* vrow = reinterpret_cast<float4*>(w_s + SGD_WBYTES + lane * ROWB);
#pragma unroll
        for (int j = 0; j < CW / 4; ++j) {
          const int pos = swz(lane, j);
          float4 wv = wrow[pos];
          float4 vv = mom ? vrow[pos] : make_float4(0.f, 0.f, 0.f, 0.f);
          float* wp = &wv.x;
          float* vp = &vv.x;
#pragma unroll
          for (int k2 = 0; k2 < 4; ++k2) {
            const float g = __uint_as_float(r[4 * j + k2]);
            const float gp = __fadd_rn(g, __fmul_rn(args.wd, wp[k2]));
            float upd = gp;
            if (mom) {
              vp[k2] = __fadd_rn(__fmul_rn(args.mu, vp[k2]), gp);
              upd = vp[k2];
            }
            wp[k2] = __fsub_rn(wp[k2], __fmul_rn(args.lr, upd));
          }
          wrow[pos] = wv;
          if (mom) vrow[pos] = vv;
        }
        __syncwarp();
        const int col0 = nb * BN + c * CW;
        const size_t ld = static_cast<size_t>(args.ldo);
        constexpr int LPR = CW / 4;
#pragma unroll
        for (int k2 = 0; k2 < 32 / (32 / LPR); ++k2) {
          const int rr = (32 / LPR) * k2 + lane / LPR, ch = lane % LPR;
          const int pos = swz(rr, ch);
          const int grow = row0 + rr, gcol = col0 + ch * 4;
          const float4 wv = *reinterpret_cast<const float4*>(w_s + rr * ROWB + pos * 16);
          float4 vv;
          if (mom) vv = *reinterpret_cast<const float4*>(w_s + SGD_WBYTES + rr * ROWB + pos * 16);
          if (grow < args.M && gcol < args.N) {
            __stcs(reinterpret_cast<float4*>(args.w + grow * ld + gcol), wv);
            if (mom) __stcs(reinterpret_cast<float4*>(args.v + grow * ld + gcol), vv);
            *reinterpret_cast<uint2*>(args.ver + grow * ld + gcol) =
                make_uint2(pack_bf16(wv.x, wv.y), pack_bf16(wv.z, wv.w));
          }
        }
        ptx::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) issue(i + SGD_NB);
        __syncwarp();
      }
    }
  }

  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_relinquish_cg2();
    ptx::tmem_dealloc_cg2(tmem_base, C::TMEM_COLS);
  }
}

// ---------------------------------------------------------------- host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// 2-D bf16 tensor [rows, cols] (cols contiguous, ld elements), box {64, box_rows}, 128B swizzle.
bool make_tmap(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint64_t ld, uint32_t box_rows) {
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// 2-D operand tensor [rows, cols] (cols contiguous, ld elements) of bf16 (box {64, box_rows}) or,
// tf = 1, of fp32-held tf32 values (box {32, box_rows}): one 128-byte swizzled row per box row
// (mn = 1: the tile is an MN-major operand; tf32 MN-major operands use the 32-byte-atom 128-byte
// swizzle, the only MN-major smem layout kind::tf32 reads)
bool make_tmap_t(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint64_t ld, uint32_t box_rows,
                 int tf, int mn) {
  if (!tf) return make_tmap(m, base, rows, cols, ld, box_rows);
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * 4};
  cuuint32_t box[2] = {32, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, mn ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// 2-D tensor of any element type with an explicit box and swizzle (fused-update epilogue boxes)
bool make_tmap_box(CUtensorMap* m, const void* base, CUtensorMapDataType dt, uint32_t esize, uint64_t rows,
                   uint64_t cols, uint64_t ld, uint32_t box_cols, uint32_t box_rows, CUtensorMapSwizzle sw) {
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * esize};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, dt, 2, const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// 4-D bf16 NHWC-style tensor: dims {d0 (contiguous), d1, d2, d3}, box {64, b1, b2, b3}, 128B swizzle.
bool make_tmap4(CUtensorMap* m, const void* base, const uint64_t (&d)[4], const uint32_t (&box)[4]) {
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) return false;
  cuuint64_t dims[4] = {d[0], d[1], d[2], d[3]};
  cuuint64_t strides[3] = {d[0] * 2, d[0] * d[1] * 2, d[0] * d[1] * d[2] * 2};
  cuuint32_t bx[4] = {box[0], box[1], box[2], box[3]};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, bx, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

typedef CUresult (*EncodeIm2colFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const int*, const int*, cuuint32_t, cuuint32_t,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// im2col-mode map of an NHWC bf16 tensor [N, H, W, C] for a k x k / stride s / pad p filter:
// each load walks `pixels` receptive-field origins (W fastest, then H, then N) within the box
// [-p, dim - 1 + p - (k - 1)] per spatial dim, stepping by s, 64 channels per pixel, 128B swizzle
bool make_tmap_im2col(CUtensorMap* m, const void* base, const ConvGeom& g, int C, uint32_t pixels) {
  static EncodeIm2colFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeIm2colFn>(p);
    if (!fn) return false;
  }
  cuuint64_t dims[4] = {static_cast<cuuint64_t>(C), static_cast<cuuint64_t>(g.W), static_cast<cuuint64_t>(g.H),
                        static_cast<cuuint64_t>(g.N)};
  cuuint64_t strides[3] = {dims[0] * 2, dims[0] * dims[1] * 2, dims[0] * dims[1] * dims[2] * 2};
  const int lower[2] = {-g.p, -g.p};                              // {W, H}
  const int upper[2] = {g.p - (g.k - 1), g.p - (g.k - 1)};
  cuuint32_t es[4] = {1, static_cast<cuuint32_t>(g.s), static_cast<cuuint32_t>(g.s), 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, lower, upper, 64,
                  pixels, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// (w, h, n) extent of a box holding `pixels` consecutive NHWC pixels (row-major n, h, w)
bool pixel_box(int pixels, int H, int W, uint32_t (&box)[4]) {
  const int P = H * W;
  if (W > 256 || H > 256) return false;
  if (P >= pixels) {
    if (pixels % W || P % pixels) return false;
    box[1] = W; box[2] = pixels / W; box[3] = 1;
  } else {
    if (pixels % P || pixels / P > 256) return false;
    box[1] = W; box[2] = H; box[3] = pixels / P;
  }
  box[0] = 64;
  return true;
}

__global__ void splitk_reduce(const float4* __restrict__ ws, float4* __restrict__ out, int64_t n4, int splits) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float4 a = ws[i];
    for (int k = 1; k < splits; ++k) {
      const float4 b = ws[i + k * n4];
      a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
    }
    out[i] = a;
  }
}

// split-K forward / input gradient: out = epilogue(Σ_ks ws[ks]) — the partials summed in split
// order (deterministic), then the plain epilogue's steps in its order: α scale, + bias, ReLU,
// ReLU mask (bf16 source, positive = sign clear and nonzero), + bf16 addend, bf16 RNE store.
// One thread per 8 columns of a row (N % 8 == 0).
__global__ void splitk_finish(const float* __restrict__ ws, int splits, int M, int N, GemmArgs a) {
  const int n8 = N / 8;
  const int64_t total = static_cast<int64_t>(M) * n8;
  const int64_t slice = static_cast<int64_t>(M) * N;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int row = static_cast<int>(i / n8), col = static_cast<int>(i - static_cast<int64_t>(row) * n8) * 8;
    const float4* p = reinterpret_cast<const float4*>(ws + static_cast<int64_t>(row) * N + col);
    float4 a0 = __ldcs(p), a1 = __ldcs(p + 1);
    for (int k = 1; k < splits; ++k) {
      const float4 b0 = __ldcs(p + k * slice / 4), b1 = __ldcs(p + k * slice / 4 + 1);
      a0.x += b0.x; a0.y += b0.y; a0.z += b0.z; a0.w += b0.w;
      a1.x += b1.x; a1.y += b1.y; a1.z += b1.z; a1.w += b1.w;
    }
    float v[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
    if (a.alpha != 1.0f) {
#pragma unroll
      for (int e = 0; e < 8; ++e) v[e] = __fmul_rn(v[e], a.alpha);
    }
    if (a.bias) {
#pragma unroll
      for (int e = 0; e < 8; ++e) v[e] = __fadd_rn(v[e], __ldg(a.bias + col + e));
    }
    if (a.relu) {
#pragma unroll
      for (int e = 0; e < 8; ++e) v[e] = fmaxf(v[e], 0.0f);
    }
    if (a.mask) {
      const uint4 mv = __ldg(reinterpret_cast<const uint4*>(a.mask + static_cast<size_t>(row) * a.ldm + col));
      const uint32_t w[4] = {mv.x, mv.y, mv.z, mv.w};
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const uint32_t h = (w[e >> 1] >> ((e & 1) * 16)) & 0xFFFFu;
        if (!(((h & 0x8000u) == 0u) && ((h & 0x7FFFu) != 0u))) v[e] = 0.0f;
      }
    }
    if (a.addend) {
      const uint4 av = *reinterpret_cast<const uint4*>(a.addend + static_cast<size_t>(row) * a.ldo + col);
      const uint32_t w[4] = {av.x, av.y, av.z, av.w};
#pragma unroll
      for (int e = 0; e < 8; ++e) v[e] = __fadd_rn(v[e], __uint_as_float(((w[e >> 1] >> ((e & 1) * 16)) & 0xFFFFu) << 16));
    }
    uint4 o;
    o.x = pack_bf16(v[0], v[1]);
    o.y = pack_bf16(v[2], v[3]);
    o.z = pack_bf16(v[4], v[5]);
    o.w = pack_bf16(v[6], v[7]);
    *reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(a.out) + static_cast<size_t>(row) * a.ldo + col) = o;
  }
}

}  // namespace

bool conv_implicit_ok(int H, int W) {
  uint32_t b[4];
  return pixel_box(128, H, W, b) && pixel_box(64, H, W, b);
}

namespace {

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

struct EpiMaps {
  CUtensorMap w, v, q;   // fused update: fp32 master, fp32 momentum, bf16 version (32x32 boxes)
};

template <int BN, int A_MN, int B_MN, int BLEND, int SGD = 0, int CG = 1, int CONV = CONV_NONE, int MH = 1, int TF = 0>
cudaError_t launch(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& b2, const EpiMaps& em,
                   const GemmArgs& args, cudaStream_t st) {
  using C = Cfg<BN, BLEND, SGD, CG, MH>;
  auto kern = gemm_kernel<BN, A_MN, B_MN, BLEND, SGD, CG, CONV, MH, TF>;
  static bool attr_set = false;   // per instantiation
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  const int tiles = ((args.M + BM * CG * MH - 1) / (BM * CG * MH)) * ((args.N + BN - 1) / BN) * std::max(1, args.splits);
  const int sms = args.max_ctas > 0 ? std::min(args.max_ctas, num_sms()) : num_sms();
  const int clusters = std::max(1, std::min(tiles, sms / CG));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(clusters * CG);
  cfg.blockDim = dim3(C::THREADS);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  // TPS_PDL=1 launches the GEMMs as programmatic dependents (prologue overlaps the previous
  // kernel's tail); measured within noise on C5 and ResNet-50, so off by default
  static const int pdl = [] {
    const char* e = std::getenv("TPS_PDL");
    return e ? std::atoi(e) : 0;
  }();
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 2 : 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, a, b, b2, em.w, em.v, em.q, args);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

struct Tiling {
  int cg, bn;
  int splits = 1, kper = 0;
};

// Pick the CTA-pair mode and tile width.  Pairs (256 x BN tiles, cta_group::2) cut operand
// traffic per SM by a third; they are used when M fills at least two 128-row blocks and the
// pair grid still covers the chip.  Env TPS_GEMM_CG=1 forces single-CTA tiles.
Tiling pick_tiling_base(int M, int N, int K, int mode, bool sgd, int max_ctas);

// Forward / input-gradient GEMMs whose single-CTA tiles cannot fill a third of the GPU while
// their K is long (VGG-16 on 32x32 inputs: the 2x2 convolutions and the 4096-wide heads at
// 64-sample micro-batches; 32 CTAs for ~29 us) split K like the weight gradients; the caller
// (gemm_run) reduces the partials and applies the epilogue in splitk_finish.  Same-box A/B:
// C3 VGG-16 S = 1 111.4k vs 102.7k samples/s; TPS_SPLITK_FD=0 disables it.
Tiling pick_tiling(int M, int N, int K, int mode, bool sgd, int max_ctas = 0) {
  Tiling tl = pick_tiling_base(M, N, K, mode, sgd, max_ctas);
  static int no_fd = -1;
  if (no_fd < 0) {
    const char* e = std::getenv("TPS_SPLITK_FD");
    no_fd = (e && e[0] == '0') ? 1 : 0;
  }
  const bool fd = mode == GEMM_FWD || mode == GEMM_DGRAD || mode == GEMM_CONV_FWD || mode == GEMM_CONV_DGRAD;
  if (!fd || no_fd || tl.cg != 1 || tl.splits > 1 || (N & 7)) return tl;
  const int sms = max_ctas > 0 ? std::min(max_ctas, num_sms()) : num_sms();
  const int tiles = ((M + BM - 1) / BM) * ((N + tl.bn - 1) / tl.bn);
  const int num_k = (K + BK - 1) / BK;
  if (tiles * 3 > sms || num_k < 32) return tl;
  int splits = std::min({sms / tiles, num_k / 16, 8});
  if (splits < 2) return tl;
  const int kper = (num_k + splits - 1) / splits;
  splits = (num_k + kper - 1) / kper;
  return {1, tl.bn, splits, kper};
}

Tiling pick_tiling_base(int M, int N, int K, int mode, bool sgd, int max_ctas) {
  if (mode == GEMM_DGRAD_BLEND || mode == GEMM_CONV_DGRAD_BLEND) {
    // three operand tiles per stage: CTA pairs (256 x 256 tiles) halve the L2 -> SM operand
    // bytes per FLOP, which is what bounds the blended dgrad
    static int force_cg_b = -1;
    if (force_cg_b < 0) {
      const char* e = std::getenv("TPS_GEMM_CG");
      force_cg_b = e ? std::atoi(e) : 0;
    }
    if (force_cg_b != 1 && M >= 256 && N > 128 && ((M + 255) / 256) * ((N + 255) / 256) >= num_sms() / 2 * 3 / 4)
      return {2, 256};
    // fewer rows (C2: M = 512): 256 x 128 pair tiles still fill the pairs and, per SM, stage and
    // blend half the B bytes of a 128 x 128 single-CTA tile for the same MMA work
    if (force_cg_b != 1 && M >= 256 && N > 64 && ((M + 255) / 256) * ((N + 127) / 128) >= num_sms() / 2 * 3 / 4)
      return {2, 128};
    return {1, 128};
  }
  const int sms0 = max_ctas > 0 ? std::min(max_ctas, num_sms()) : num_sms();
  static int no_split = -1;
  if (no_split < 0) {
    const char* e = std::getenv("TPS_NO_SPLITK");
    no_split = (e && e[0] == '1') ? 1 : 0;
  }
  if ((mode == GEMM_WGRAD || mode == GEMM_CONV_WGRAD) && !sgd && !no_split) {
    // weight gradients of convolutions: small M x N, K = every pixel of the batch.  When the
    // output tiles cannot fill the GPU, split K across CTAs (fp32 partials + ordered reduce)
    const int bn = N <= 64 ? 64 : (N <= 128 ? 128 : 256);
    const int tiles = ((M + BM - 1) / BM) * ((N + bn - 1) / bn);
    const int num_k = (K + BK - 1) / BK;
    if (tiles < sms0 * 3 / 4 && num_k >= 16) {
      int splits = std::min({(sms0 + tiles - 1) / tiles, num_k / 8, 64});
      if (splits > 1) {
        const int kper = (num_k + splits - 1) / splits;
        splits = (num_k + kper - 1) / kper;          // every split non-empty
        return {1, bn, splits, kper};
      }
    }
  }
  const int sms = sms0;
  static int force_cg = -1;
  if (force_cg < 0) {
    const char* e = std::getenv("TPS_GEMM_CG");
    force_cg = e ? std::atoi(e) : 0;
  }
  static int sgd_bn = -1;
  if (sgd_bn < 0) {
    const char* e = std::getenv("TPS_SGD_BN");
    sgd_bn = e ? std::atoi(e) : 0;
  }
  if (sgd && sgd_bn && force_cg != 1 && M >= 256) return {2, sgd_bn};
  if (force_cg != 1 && M >= 256) {
    const int tm = (M + 255) / 256;
    if (max_ctas > 0 && !sgd) {
      // partitioned grid (split backward): pick the pair tile width with the better last-wave
      // fill, 256 unless 128 fills the partition's waves clearly better
      const int cl = std::max(1, sms / 2);
      double best = -1.0;
      int best_bn = 256;
      for (int bn : {256, 128}) {
        if (N <= bn / 2) continue;
        const int tiles = tm * ((N + bn - 1) / bn);
        const int waves = (tiles + cl - 1) / cl;
        const double fill = static_cast<double>(tiles) / (static_cast<double>(waves) * cl);
        if (fill > best + 0.05) { best = fill; best_bn = bn; }
      }
      if (best > 0) return {2, best_bn};
    }
    for (int bn : {256, 128}) {
      if (N <= bn / 2) continue;
      const int tiles = tm * ((N + bn - 1) / bn);
      if (tiles >= (sms / 2) * 3 / 4) return {2, bn};
    }
  }
  const int tm = (M + BM - 1) / BM;
  const int cand[3] = {256, 128, 64};
  for (int i = 0; i < 3; ++i) {
    const int bn = cand[i];
    if (bn > 64 && N <= bn / 2) continue;          // mostly padding
    const int tiles = tm * ((N + bn - 1) / bn);
    if (tiles >= (sms * 3) / 4 || bn == 64) return {1, bn};
  }
  return {1, 64};
}

template <int A_MN, int B_MN, int SGD, int CONV = CONV_NONE, int TF = 0>
cudaError_t dispatch(const Tiling& tl, const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tb2,
                     const EpiMaps& em, const GemmArgs& args, cudaStream_t st) {
  if (tl.cg == 2) {
    if (tl.bn == 256) return launch<256, A_MN, B_MN, 0, SGD, 2, CONV, 1, TF>(ta, tb, tb2, em, args, st);
    return launch<128, A_MN, B_MN, 0, SGD, 2, CONV, 1, TF>(ta, tb, tb2, em, args, st);
  }
  if (tl.bn == 256) return launch<256, A_MN, B_MN, 0, SGD, 1, CONV, 1, TF>(ta, tb, tb2, em, args, st);
  if (tl.bn == 128) return launch<128, A_MN, B_MN, 0, SGD, 1, CONV, 1, TF>(ta, tb, tb2, em, args, st);
  return launch<64, A_MN, B_MN, 0, SGD, 1, CONV, 1, TF>(ta, tb, tb2, em, args, st);
}

}  // namespace

// Blended input gradient on CTA pairs: 512-row tiles (MH = 2, two accumulators sharing one
// blended B tile) when the K loop is long enough that the single accumulator buffer's exposed
// epilogue is small and two waves of 256-row tiles become (at most) one of 512-row tiles.  TPS_BLEND_MH=1 keeps 256-row tiles.
bool blend_mh2(const GemmArgs& a) {
  static int mh = -1;
  if (mh < 0) {
    const char* e = std::getenv("TPS_BLEND_MH");
    mh = e ? std::atoi(e) : 2;
  }
  if (mh != 2 || (a.K + BK - 1) / BK < 16) return false;
  const int pairs = num_sms() / 2, nn = (a.N + 255) / 256;
  const int w256 = ((a.M + 255) / 256 * nn + pairs - 1) / pairs;       // waves of 256-row tiles
  const int w512 = ((a.M + 511) / 512 * nn + pairs - 1) / pairs;       // waves of 512-row tiles
  return 2 * w512 <= w256;
}

const char* gemm_mode_name(int mode) {
  switch (mode) {
    case GEMM_FWD: return "fwd";
    case GEMM_DGRAD: return "dgrad";
    case GEMM_WGRAD: return "wgrad";
    case GEMM_DGRAD_BLEND: return "dgrad_blend";
    case GEMM_CONV_FWD: return "conv_fwd";
    case GEMM_CONV_DGRAD: return "conv_dgrad";
    case GEMM_CONV_DGRAD_BLEND: return "conv_dgrad_blend";
    case GEMM_CONV_WGRAD: return "conv_wgrad";
  }
  return "?";
}

cudaError_t gemm_run(int mode, const GemmOperands& op, const GemmArgs& args_in, cudaStream_t st, int* bn_out) {
  GemmArgs args = args_in;
  if (args.M <= 0 || args.N <= 0 || args.K <= 0) return cudaSuccess;
  const bool sgd = ((mode == GEMM_WGRAD || mode == GEMM_CONV_WGRAD) && args.epi == EPI_SGD);
  if (args.tf32 && (mode >= GEMM_CONV_FWD || args.addend)) return cudaErrorInvalidValue;
  {
    static int st_env = -1;
    if (st_env < 0) {
      const char* e = std::getenv("TPS_SGD_SPLIT_TAIL");
      st_env = (e && e[0] == '0') ? 0 : 1;
    }
    args.split_tail = sgd && st_env;
  }
  Tiling tl = pick_tiling(args.M, args.N, args.K, mode, sgd, args.max_ctas);
  if (args.tf32) tl.splits = 1;                      // tf32: one pass over K
  const bool fd = mode == GEMM_FWD || mode == GEMM_DGRAD || mode == GEMM_CONV_FWD || mode == GEMM_CONV_DGRAD;
  GemmArgs fin{};                                    // split forward / input gradient: the epilogue
  bool fd_split = false;
  if (tl.splits > 1 && fd) {
    if (!args.ws || args.ws_floats < static_cast<int64_t>(tl.splits) * args.M * args.N || args.colsum ||
        args.out_f32 || (args.ldo & 7) || (args.mask && (args.ldm & 7))) {
      tl.splits = 1;
    } else {
      fd_split = true;
      fin = args;
      args.out_f32 = 1; args.ldo = args.N; args.bias = nullptr; args.relu = 0; args.mask = nullptr;
      args.addend = nullptr; args.alpha = 1.0f;
    }
  } else if (tl.splits > 1 &&
             (!args.ws || args.ws_floats < static_cast<int64_t>(tl.splits) * args.M * args.ldo || !args.out_f32 ||
              args.ldo != args.N)) {
    tl.splits = 1;                                   // no workspace supplied: one pass over K
  }
  args.splits = tl.splits;
  const int bke = args.tf32 ? 32 : BK;             // K elements per pipeline stage
  args.kper = tl.splits > 1 ? tl.kper : (args.K + bke - 1) / bke;
  CUtensorMap ta, tb, tb2;
  bool ok = true;
  if (mode >= GEMM_CONV_FWD) {
    const ConvGeom& g = op.cv;
    args.cv = g;
    if (g.C % 64 || g.N * g.H * g.W <= 0) return cudaErrorInvalidValue;
    const uint64_t act_dims[4] = {static_cast<uint64_t>(g.C), static_cast<uint64_t>(g.W),
                                  static_cast<uint64_t>(g.H), static_cast<uint64_t>(g.N)};
    uint32_t box128[4], box64[4];
    if (g.im2col) {
      if (g.k < 1 || g.s < 1 || g.s > 8 || g.p < 0 || g.Ho < 1 || g.Wo < 1) return cudaErrorInvalidValue;
      if ((mode == GEMM_CONV_DGRAD || mode == GEMM_CONV_DGRAD_BLEND) && (g.k != 3 || g.s != 1 || g.p != 1))
        return cudaErrorInvalidValue;
    } else if (!pixel_box(128, g.H, g.W, box128) || !pixel_box(64, g.H, g.W, box64)) {
      return cudaErrorInvalidValue;
    }
    if (g.im2col) {
      if (mode == GEMM_CONV_FWD) {
        ok &= make_tmap_im2col(&ta, op.A, g, g.C, 128);                             // X (NHWC)
        ok &= make_tmap(&tb, op.B, args.N, args.K, op.ldb, tl.bn / tl.cg);         // W [Co, k·k·Ci]
        tb2 = tb;
      } else if (mode == GEMM_CONV_DGRAD || mode == GEMM_CONV_DGRAD_BLEND) {
        ok &= make_tmap_im2col(&ta, op.A, g, g.C, 128);                             // dY (NHWC, C = Co)
        const uint64_t wd[4] = {static_cast<uint64_t>(op.Cw), 3, 3, static_cast<uint64_t>(g.C)};
        const uint32_t wb[4] = {64, 1, 1, 64};
        ok &= make_tmap4(&tb, op.B, wd, wb);
        if (mode == GEMM_CONV_DGRAD_BLEND) ok &= make_tmap4(&tb2, op.B2, wd, wb);
        else tb2 = tb;
        if (op.Cw % 64) return cudaErrorInvalidValue;
      } else {
        ok &= make_tmap(&ta, op.A, args.K, args.M, op.lda, 64);                     // dY [N·Ho·Wo, Co]
        ok &= make_tmap_im2col(&tb, op.B, g, g.C, 64);                              // X (NHWC)
        tb2 = tb;
      }
    } else if (mode == GEMM_CONV_FWD) {
      ok &= make_tmap4(&ta, op.A, act_dims, box128);                              // X (NHWC)
      ok &= make_tmap(&tb, op.B, args.N, args.K, op.ldb, tl.bn / tl.cg);           // W [Co, 9Ci]
      tb2 = tb;
    } else if (mode == GEMM_CONV_DGRAD || mode == GEMM_CONV_DGRAD_BLEND) {
      ok &= make_tmap4(&ta, op.A, act_dims, box128);                              // dY (NHWC, C = Co)
      const uint64_t wd[4] = {static_cast<uint64_t>(op.Cw), 3, 3, static_cast<uint64_t>(g.C)};
      const uint32_t wb[4] = {64, 1, 1, 64};
      ok &= make_tmap4(&tb, op.B, wd, wb);                                        // W [Co,3,3,Ci]
      if (mode == GEMM_CONV_DGRAD_BLEND) ok &= make_tmap4(&tb2, op.B2, wd, wb);
      else tb2 = tb;
      if (op.Cw % 64) return cudaErrorInvalidValue;
    } else {  // GEMM_CONV_WGRAD
      ok &= make_tmap(&ta, op.A, args.K, args.M, op.lda, 64);                     // dY [NHW, Co], MN-major
      ok &= make_tmap4(&tb, op.B, act_dims, box64);                               // X (NHWC)
      tb2 = tb;
    }
  } else {
    const bool a_mn = (mode == GEMM_WGRAD);
    const bool b_mn = (mode != GEMM_FWD);
    // A: K-major [M,K] -> box {64 K, 128 rows}; MN-major stored [K,M] -> box {64 M, 64 K}
    // B: K-major [N,K] -> box {64 K, BN/CG rows} (each CTA of a pair loads its share)
    // (tf32: box {32, ·}; MN-major boxes 32 x 32)
    const int tf = args.tf32;
    if (!a_mn) ok &= make_tmap_t(&ta, op.A, args.M, args.K, op.lda, BM, tf, 0);
    else ok &= make_tmap_t(&ta, op.A, args.K, args.M, op.lda, bke, tf, 1);
    if (!b_mn) ok &= make_tmap_t(&tb, op.B, args.N, args.K, op.ldb, tl.bn / tl.cg, tf, 0);
    else ok &= make_tmap_t(&tb, op.B, args.K, args.N, op.ldb, bke, tf, 1);
    if (mode == GEMM_DGRAD_BLEND) ok &= make_tmap_t(&tb2, op.B2, args.K, args.N, op.ldb, bke, tf, 1);
    else tb2 = tb;
  }
  EpiMaps em;
  em.w = em.v = em.q = ta;   // unused unless sgd
  if (sgd) {
    const CUtensorMapSwizzle wsw = SGD_CW == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
    ok &= make_tmap_box(&em.w, args.w, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, args.M, args.N, args.ldo, SGD_CW, 32, wsw);
    if (args.mu != 0.0f)
      ok &= make_tmap_box(&em.v, args.v, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, args.M, args.N, args.ldo, SGD_CW, 32, wsw);
    ok &= make_tmap_box(&em.q, args.ver, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, args.M, args.N, args.ldo, 32, 32,
                        CU_TENSOR_MAP_SWIZZLE_64B);
  }
  if (!ok) return cudaErrorInvalidValue;
  if (bn_out) *bn_out = tl.bn * 10 + tl.cg;
  cudaError_t e = cudaErrorInvalidValue;
  if (args.tf32) {
    switch (mode) {
      case GEMM_FWD: return dispatch<0, 0, 0, CONV_NONE, 1>(tl, ta, tb, tb2, em, args, st);
      case GEMM_DGRAD: return dispatch<0, 1, 0, CONV_NONE, 1>(tl, ta, tb, tb2, em, args, st);
      case GEMM_WGRAD:
        return sgd ? dispatch<1, 1, 1, CONV_NONE, 1>(tl, ta, tb, tb2, em, args, st)
                   : dispatch<1, 1, 0, CONV_NONE, 1>(tl, ta, tb, tb2, em, args, st);
      case GEMM_DGRAD_BLEND:
        if (tl.cg == 2)
          return tl.bn == 128 ? launch<128, 0, 1, 1, 0, 2, CONV_NONE, 1, 1>(ta, tb, tb2, em, args, st)
                 : blend_mh2(args) ? launch<256, 0, 1, 1, 0, 2, CONV_NONE, 2, 1>(ta, tb, tb2, em, args, st)
                                   : launch<256, 0, 1, 1, 0, 2, CONV_NONE, 1, 1>(ta, tb, tb2, em, args, st);
        return launch<128, 0, 1, 1, 0, 1, CONV_NONE, 1, 1>(ta, tb, tb2, em, args, st);
      default: return cudaErrorInvalidValue;
    }
  }
  switch (mode) {
    case GEMM_FWD: e = dispatch<0, 0, 0>(tl, ta, tb, tb2, em, args, st); break;
    case GEMM_DGRAD: e = dispatch<0, 1, 0>(tl, ta, tb, tb2, em, args, st); break;
    case GEMM_WGRAD:
      e = sgd ? dispatch<1, 1, 1>(tl, ta, tb, tb2, em, args, st) : dispatch<1, 1, 0>(tl, ta, tb, tb2, em, args, st);
      break;
    case GEMM_DGRAD_BLEND:
      e = tl.cg == 2 ? (tl.bn == 128 ? launch<128, 0, 1, 1, 0, 2>(ta, tb, tb2, em, args, st)
                        : blend_mh2(args) ? launch<256, 0, 1, 1, 0, 2, CONV_NONE, 2>(ta, tb, tb2, em, args, st)
                                          : launch<256, 0, 1, 1, 0, 2>(ta, tb, tb2, em, args, st))
                     : launch<128, 0, 1, 1, 0, 1>(ta, tb, tb2, em, args, st);
      break;
    case GEMM_CONV_FWD: e = dispatch<0, 0, 0, CONV_FWD>(tl, ta, tb, tb2, em, args, st); break;
    case GEMM_CONV_DGRAD: e = dispatch<0, 1, 0, CONV_DGRAD>(tl, ta, tb, tb2, em, args, st); break;
    case GEMM_CONV_DGRAD_BLEND:
      e = tl.cg == 2 ? (tl.bn == 128 ? launch<128, 0, 1, 1, 0, 2, CONV_DGRAD>(ta, tb, tb2, em, args, st)
                        : blend_mh2(args) ? launch<256, 0, 1, 1, 0, 2, CONV_DGRAD, 2>(ta, tb, tb2, em, args, st)
                                          : launch<256, 0, 1, 1, 0, 2, CONV_DGRAD>(ta, tb, tb2, em, args, st))
                     : launch<128, 0, 1, 1, 0, 1, CONV_DGRAD>(ta, tb, tb2, em, args, st);
      break;
    case GEMM_CONV_WGRAD:
      e = sgd ? dispatch<1, 1, 1, CONV_WGRAD>(tl, ta, tb, tb2, em, args, st)
              : dispatch<1, 1, 0, CONV_WGRAD>(tl, ta, tb, tb2, em, args, st);
      break;
  }
  if (e != cudaSuccess || tl.splits <= 1) return e;
  if (fd_split) {
    const int64_t n8 = static_cast<int64_t>(args.M) * args.N / 8;
    const int blocks = static_cast<int>(std::min<int64_t>((n8 + 255) / 256, static_cast<int64_t>(num_sms()) * 8));
    splitk_finish<<<blocks, 256, 0, st>>>(args.ws, tl.splits, args.M, args.N, fin);
    return cudaGetLastError();
  }
  // ordered reduction of the split-K partials: out = Σ_ks ws[ks] (deterministic)
  const int64_t n4 = static_cast<int64_t>(args.M) * args.ldo / 4;
  const int blocks = static_cast<int>(std::min<int64_t>((n4 + 255) / 256, static_cast<int64_t>(num_sms()) * 8));
  splitk_reduce<<<blocks, 256, 0, st>>>(reinterpret_cast<const float4*>(args.ws), reinterpret_cast<float4*>(args.out),
                                        n4, tl.splits);
  return cudaGetLastError();
}

cudaError_t gemm_bwd_dual(const GemmOperands& opw, const GemmArgs& aw_in, const GemmOperands& opd, const DualArgs& dg,
                          cudaStream_t st) {
  constexpr int BN = 256, CG = 2;
  using C = Cfg<BN, 0, 1, CG>;
  GemmArgs aw = aw_in;
  if (aw.tf32 || aw.epi != EPI_SGD || aw.M < BM * CG || dg.M < BM * CG || aw.N <= BN / 2 || dg.N <= BN / 2 || aw.K <= 0 ||
      dg.K <= 0 || (dg.N & 7) || (aw.N & 7))
    return cudaErrorNotSupported;
  const int n_w = ((aw.M + BM * CG - 1) / (BM * CG)) * ((aw.N + BN - 1) / BN);
  const int n_d = ((dg.M + BM * CG - 1) / (BM * CG)) * ((dg.N + BN - 1) / BN);
  const int kw = (aw.K + BK - 1) / BK, kd = (dg.K + BK - 1) / BK;
  const int ncl = std::min(num_sms() / CG, n_w + n_d);
  // the closed-form split must hand every W tile to exactly one pair (monotone prefix)
  for (int c = 0; c < ncl; ++c)
    if (dual_wpre(c + 1, n_d, n_w, kd, kw, ncl) < dual_wpre(c, n_d, n_w, kd, kw, ncl)) return cudaErrorNotSupported;
  if (dual_wpre(ncl, n_d, n_w, kd, kw, ncl) != n_w) return cudaErrorNotSupported;
  aw.splits = 1;
  aw.kper = kw;
  CUtensorMap ta, tb, tda, tdb, tw, tv;
  bool ok = make_tmap(&ta, opw.A, aw.K, aw.M, opw.lda, 64) && make_tmap(&tb, opw.B, aw.K, aw.N, opw.ldb, 64) &&
            make_tmap(&tda, opd.A, dg.M, dg.K, opd.lda, BM) && make_tmap(&tdb, opd.B, dg.K, dg.N, opd.ldb, 64);
  const CUtensorMapSwizzle wsw = SGD_CW == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
  ok = ok && make_tmap_box(&tw, aw.w, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, aw.M, aw.N, aw.ldo, SGD_CW, 32, wsw);
  if (aw.mu != 0.0f)
    ok = ok && make_tmap_box(&tv, aw.v, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, aw.M, aw.N, aw.ldo, SGD_CW, 32, wsw);
  else
    tv = tw;
  if (!ok) return cudaErrorInvalidValue;
  auto kern = bwd_dual_kernel<BN, CG>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(ncl * CG);
  cfg.blockDim = dim3(C::THREADS);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, ta, tb, tda, tdb, tw, tv, aw, dg);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

int64_t gemm_splitk_floats(int mode, int M, int N, int K, int ldo) {
  if (M <= 0 || N <= 0 || K <= 0) return 0;
  const Tiling tl = pick_tiling(M, N, K, mode, false);
  return tl.splits > 1 ? static_cast<int64_t>(tl.splits) * M * std::max(ldo, N) : 0;
}

}  // namespace tps

// TMA-fed tcgen05 3xTF32 implicit-GEMM convolutions (minml/kernels.py:197-239):
// conv2d fprop, stride-1 grad_input (dgrad) and stride-1 grad_weight (wgrad).
//
// gemm_tc.cu feeds the tensor cores from SIMT producer warps that gather, split and swizzle
// every operand element; ncu shows those producers issue-bound at ~20 instructions per
// element with the tensor pipe <10% busy.  Here the split moves out of the GEMM:
//   1. a pre-pass (HBM-bound) writes each operand as two planes, hi = rna_tf32(x) and
//      lo = x - hi (exact in f32): activations NHWC for fprop/dgrad; for wgrad x and g as
//      per-(n, channel) planes on the zero-padded grid of row pitch Wp = roundup(W+2p, 4),
//      flattened, so a filter tap (r, s) is a constant shift r*Wp + s along the plane (x is
//      written once per s, pre-shifted by s, because TMA box starts must be 16-byte aligned);
//      weights K-major [rows][(r,s,c)];
//   2. the GEMM kernel's single producer thread loads every tile with TMA straight into
//      128B-swizzled K-major shared memory: fprop/dgrad activation tiles in im2col mode (the
//      hardware walks output pixels across rows and images, applies stride and padding and
//      zero-fills out-of-range taps), weight tiles in tiled mode; wgrad tiles (K = positions
//      on the padded output grid, 32 per k-block) as 3-D boxes of 32 positions x 128 channels,
//      x shifted by r*Wp (copy s), g unshifted (g is zero on the padding columns);
//   3. one thread issues 3 tcgen05.mma.kind::tf32 per 8-deep k step (lo*hi, hi*lo, hi*hi)
//      into TMEM; the drain warps fold 2-k-block chunks into f32 registers with IEEE
//      round-to-nearest (the same accumulation scheme as gemm_tc.cu, so results agree with it
//      to rounding) and store through the output functor.
// The split is gemm_tc.cu's (hi = rna_tf32(x), lo = rna_tf32(x - hi)), so both kernel
// families produce the same products.
//
// Shapes the kernel declines (PB_ERR_UNSUPPORTED, no side effects) fall through to
// gemm_tc.cu: channel counts not a multiple of 32 (the RGB stem), strided dgrad, and
// anything whose coordinates do not fit the TMA limits.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include "common.cuh"
#include "tc_common.cuh"

namespace pb {
namespace tma {

using namespace pb::tc;

constexpr int BM = 128;  // D rows per CTA = TMEM lanes
constexpr int BK = 32;   // k per stage: one 128-byte swizzled row of f32
constexpr int CK = 2;    // k-blocks accumulated in TMEM per register drain (4 fails a golden wgrad case at 1e-5)

// ---- driver entry points (no libcuda link: resolved through the runtime) -------------------
typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
typedef CUresult (*EncodeIm2col)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const int*, const int*, cuuint32_t, cuuint32_t,
                                 const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                 CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiled g_tiled = nullptr;
static EncodeIm2col g_im2col = nullptr;

static bool driver_ok() {
  static int state = -1;
  if (state < 0) {
    cudaDriverEntryPointQueryResult q1, q2;
    void* f1 = nullptr;
    void* f2 = nullptr;
    state = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f1, cudaEnableDefault, &q1) == cudaSuccess &&
            cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &f2, cudaEnableDefault, &q2) == cudaSuccess &&
            q1 == cudaDriverEntryPointSuccess && q2 == cudaDriverEntryPointSuccess && f1 && f2;
    g_tiled = (EncodeTiled)f1;
    g_im2col = (EncodeIm2col)f2;
  }
  return state == 1;
}

// 2-D K-major (or MN-major) plane [rows][cols] f32, box {32 cols, box_rows}
static bool map_2d(CUtensorMap* m, const float* p, int64_t cols, int64_t rows, int box_rows) {
  cuuint64_t dim[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t str[1] = {(cuuint64_t)cols * 4};
  cuuint32_t box[2] = {32, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  return g_tiled(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)p, dim, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                 CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// flattened planes [copies][N][C][L] (L % 4 == 0), box {32 positions, bc channels, 1, 1}
static bool map_planes(CUtensorMap* m, const float* p, int copies, int N, int C, int64_t L, int bc) {
  cuuint64_t dim[4] = {(cuuint64_t)L, (cuuint64_t)C, (cuuint64_t)N, (cuuint64_t)copies};
  cuuint64_t str[3] = {(cuuint64_t)L * 4, (cuuint64_t)C * L * 4, (cuuint64_t)N * C * L * 4};
  cuuint32_t box[4] = {32, (cuuint32_t)bc, 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return g_tiled(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, (void*)p, dim, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                 CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// NHWC plane [N][H][W][C] in im2col mode: 32 channels x `pixels` output pixels per load
static bool map_im2col(CUtensorMap* m, const float* p, int N, int H, int W, int C, int KH, int KW, int SH, int SW,
                       int PH, int PW, int pixels) {
  cuuint64_t dim[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
  cuuint64_t str[3] = {(cuuint64_t)C * 4, (cuuint64_t)W * C * 4, (cuuint64_t)H * W * C * 4};
  int lower[2] = {-PW, -PH};
  int upper[2] = {PW - (KW - 1), PH - (KH - 1)};
  cuuint32_t es[4] = {1, (cuuint32_t)SW, (cuuint32_t)SH, 1};
  return g_im2col(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, (void*)p, dim, str, lower, upper, 32, (cuuint32_t)pixels,
                  es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// the same with explicit corners (a stride-1 walk whose first and last base positions are
// `lower` and W - 1 + `upper`: the sub-pixel dgrad classes have asymmetric halos)
static bool map_im2col_lu(CUtensorMap* m, const float* p, int N, int H, int W, int C, int lw, int lh, int uw, int uh,
                          int pixels) {
  cuuint64_t dim[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
  cuuint64_t str[3] = {(cuuint64_t)C * 4, (cuuint64_t)W * C * 4, (cuuint64_t)H * W * C * 4};
  int lower[2] = {lw, lh};
  int upper[2] = {uw, uh};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return g_im2col(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, (void*)p, dim, str, lower, upper, 32, (cuuint32_t)pixels,
                  es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// ---- PTX: TMA loads, expect-tx --------------------------------------------------------------
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_2d(uint32_t dst, const CUtensorMap* m, uint64_t* bar, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::
          "r"(dst),
      "l"((uint64_t)m), "r"(smem_u32(bar)), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void tma_im2col(uint32_t dst, const CUtensorMap* m, uint64_t* bar, int c, int w, int h,
                                           int n, uint16_t ow, uint16_t oh) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, "
      "%6}], [%2], {%7, %8};" ::"r"(dst),
      "l"((uint64_t)m), "r"(smem_u32(bar)), "r"(c), "r"(w), "r"(h), "r"(n), "h"(ow), "h"(oh)
      : "memory");
}
__device__ __forceinline__ void tma_3d(uint32_t dst, const CUtensorMap* m, uint64_t* bar, int x, int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
      "[%2];" ::"r"(dst),
      "l"((uint64_t)m), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(z)
      : "memory");
}
__device__ __forceinline__ void tma_4d(uint32_t dst, const CUtensorMap* m, uint64_t* bar, int x, int y, int z,
                                       int w) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], "
      "[%2];" ::"r"(dst),
      "l"((uint64_t)m), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(z), "r"(w)
      : "memory");
}
__device__ __forceinline__ void prefetch_map(const CUtensorMap* m) {
  asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)m) : "memory");
}

// UMMA smem descriptor, SWIZZLE_128B, K-major: SBO = 1024 B between 8-row groups
__device__ __forceinline__ uint64_t desc_kmajor(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// instruction descriptor: D f32, A/B tf32, K-major unless transposed (bit 15 A, bit 16 B)
__host__ __device__ constexpr uint32_t idesc(int M, int N, bool mn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (mn ? (1u << 15) | (1u << 16) : 0u) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}

// ---- problem descriptions --------------------------------------------------------------------
// CONV (fprop, and stride-1 dgrad as an fprop over the gradient with flipped weights):
//   D[i = (n,ho,wo)][j = f] = sum_{k = (r,s,c)} X[n, ho*sh-ph+r, wo*sw-pw+s, c] * Wt[f][k]
// WGRAD (stride 1), q = ho * Wp + wo on the padded grid (Wp = roundup(W + 2pw, 4)):
//   D[i = c][j = f] (tap z % RS, split z / RS) = sum_{n, q} Xs[s][n, c, q + r*Wp] * Gpad[n, f, q]
//   with Xs[s][n, c, q] = Xpad[n, c, q + s]
struct Prob {
  int N, H, W, C;      // activation plane X (NHWC)
  int KH, KW, SH, SW, PH, PW, HO, WO;
  int F;               // output channels (fprop / wgrad), or input channels (dgrad)
  int Mi, Nj, K;       // GEMM extents
  int kper;            // wgrad: k per split (multiple of BK)
  int Wp;              // wgrad: padded row pitch roundup(W + 2pw, 4)
  FastDiv fKB;         // wgrad: k-blocks per image
  int ti, tj, ntiles, zdim;
  FastDiv fP, fWO;     // output pixel decode (ho*wo, wo)
  int plain;           // 1x1, stride 1, no padding: A is a plain [pixels][C] plane (tiled TMA)
  int noload;          // diagnostics (PB_TMA_NOLOAD=1): stages are released without loading -- the
                       // MMA/drain pipeline alone, timed by tools/conv_table.py (results are garbage)
};

template <int BN, bool WG>
struct Cfg {
  static constexpr int A_BYTES = BM * 128;
  static constexpr int B_BYTES = BN * 128;
  static constexpr int STAGE = 2 * A_BYTES + 2 * B_BYTES;
  static constexpr int STAGES = (200 * 1024) / STAGE;
  static constexpr int SMEM = 1024 + STAGES * STAGE + 256;
  // drain warps: one per (TMEM lane quadrant, 32 accumulator columns) -- each thread folds 32
  // columns of a chunk, so a chunk drains in about the time the MMA needs for the next one
  static constexpr int NDRAIN = BN / 8;
  static constexpr int THREADS = 64 + NDRAIN * 32;
  // TMEM chunk buffers ({big, small} x BN columns each) in the 512 columns: the MMA may run up to
  // NBUF - 1 chunks ahead of the drain
  static constexpr int NBUF = 512 / (2 * BN) < 4 ? 512 / (2 * BN) : 4;
  static constexpr int TMEM_COLS = NBUF * 2 * BN;
  static constexpr uint32_t IDESC = idesc(BM, BN, false);
};

// Output functor for wgrad: tap-major columns into dw[f][c][r][s] (split 0) or the split-K
// workspace ws[split][f][c][r][s]; folded afterwards by fold_partials with OutMat.
// Output functor for strided 1x1 dgrad: row i = (n, ho, wo) of the gradient grid writes
// dx[n][j][ho*s][wo*s]; the other pixels receive no contribution and are zero-filled first
struct OutScatter {
  float* p;
  int Mi, Nj;
  FastDiv fP, fWO;
  int sh, sw, W, HW;
  struct Row {
    float* p;
  };
  __device__ __forceinline__ Row row(int, int i) const {
    Row o;
    o.p = nullptr;
    if (i < Mi) {
      uint32_t n, pix, ho, wo;
      fP.divmod(i, n, pix);
      fWO.divmod(pix, ho, wo);
      o.p = p + (int64_t)n * Nj * HW + (int64_t)ho * sh * W + (int64_t)wo * sw;
    }
    return o;
  }
  __device__ __forceinline__ void put(const Row& rw, int j, float v) const {
    if (rw.p && j < Nj) rw.p[(int64_t)j * HW] = v;
  }
};

struct OutWgrad {
  float* p;
  int C, F, RS;
  struct Row {
    float* p;
  };
  __device__ __forceinline__ Row row(int z, int i) const {
    Row o;
    const int split = z / RS, tap = z - split * RS;
    o.p = i < C ? p + (int64_t)split * F * C * RS + (int64_t)i * RS + tap : nullptr;
    return o;
  }
  __device__ __forceinline__ void put(const Row& rw, int j, float v) const {
    if (rw.p && j < F) rw.p[(int64_t)j * C * RS] = v;
  }
};

template <int BN, bool WG, class OUT>
__global__ void __launch_bounds__(Cfg<BN, WG>::THREADS, 1)
    tma_conv_kernel(const __grid_constant__ CUtensorMap xa_hi, const __grid_constant__ CUtensorMap xa_lo,
                    const __grid_constant__ CUtensorMap b_hi, const __grid_constant__ CUtensorMap b_lo, Prob pr,
                    OUT out) {
  typedef Cfg<BN, WG> C;
  extern __shared__ uint8_t smem_raw[];
  char* smem = (char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE);
  uint64_t* empty = full + C::STAGES;
  uint64_t* accf = empty + C::STAGES;
  uint64_t* acce = accf + C::NBUF;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acce + C::NBUF);

  const int tid = threadIdx.x, warp = tid >> 5;
  const int per_z = pr.ti * pr.tj;
  const int cblocks = pr.C / BK;

  if (tid == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < C::NBUF; ++s) {
      mbar_init(&accf[s], 1);
      mbar_init(&acce[s], C::NDRAIN * 32);
    }
    fence_barrier_init();
    prefetch_map(&xa_hi);
    prefetch_map(&xa_lo);
    prefetch_map(&b_hi);
    prefetch_map(&b_lo);
  }
  if (warp == 1) tmem_alloc<C::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // k range of tile t: CONV covers all of K; WGRAD's z = split * RS + tap takes one split
  auto krange = [&](int t, int& kbeg, int& kend) {
    if (WG) {
      const int z = t / per_z, split = z / (pr.KH * pr.KW);
      kbeg = split * pr.kper;
      kend = min(pr.K, kbeg + pr.kper);
    } else if (pr.zdim > 1) {  // plain GEMM with split K: z = split
      kbeg = (t / per_z) * pr.kper;
      kend = min(pr.K, kbeg + pr.kper);
    } else {
      kbeg = 0;
      kend = pr.K;
    }
  };

  if (warp == 0) {
    // ===== TMA producer (one thread) =====
    if (tid == 0) {
      uint32_t it = 0;
      for (int t = blockIdx.x; t < pr.ntiles; t += gridDim.x) {
        const int z = t / per_z, rem = t - z * per_z;
        const int i0 = (rem / pr.tj) * BM, j0 = (rem % pr.tj) * BN;
        int kbeg, kend;
        krange(t, kbeg, kend);
        const int nkb = kend > kbeg ? (kend - kbeg + BK - 1) / BK : 0;
        int n = 0, ho = 0, wo = 0, tr = 0, ts = 0;
        if (!WG) {  // first output pixel of the tile
          uint32_t nn, pix, h, w;
          pr.fP.divmod((uint32_t)i0, nn, pix);
          pr.fWO.divmod(pix, h, w);
          n = (int)nn, ho = (int)h, wo = (int)w;
        } else {
          const int tap = z % (pr.KH * pr.KW);
          tr = tap / pr.KW;
          ts = tap - tr * pr.KW;
        }
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % C::STAGES;
          if (it >= (uint32_t)C::STAGES) mbar_wait(&empty[s], ((it / C::STAGES) - 1) & 1);
          const uint32_t base = smem_u32(smem + s * C::STAGE);
          if (pr.noload) {
            mbar_arrive(&full[s]);
            continue;
          }
          mbar_expect_tx(&full[s], C::STAGE);
          const int k0 = kbeg + kb * BK;
          if (!WG) {
            const int kg = k0 / BK;  // global k-block (split K starts mid-way through the taps)
            const int tap = kg / cblocks, c0 = (kg - tap * cblocks) * BK;
            const int r = tap / pr.KW, sx = tap - r * pr.KW;
            const int wc = wo * pr.SW - pr.PW, hc = ho * pr.SH - pr.PH;
            if (pr.plain) {  // [rows][K] planes: the k-block is simply k0
              tma_2d(base, &xa_hi, &full[s], k0, i0);
              tma_2d(base + C::A_BYTES, &xa_lo, &full[s], k0, i0);
            } else {
              tma_im2col(base, &xa_hi, &full[s], c0, wc, hc, n, (uint16_t)sx, (uint16_t)r);
              tma_im2col(base + C::A_BYTES, &xa_lo, &full[s], c0, wc, hc, n, (uint16_t)sx, (uint16_t)r);
            }
            tma_2d(base + 2 * C::A_BYTES, &b_hi, &full[s], k0, j0);
            tma_2d(base + 2 * C::A_BYTES + C::B_BYTES, &b_lo, &full[s], k0, j0);
          } else {
            // k-block k0 / BK -> (image, 32 positions of its padded output grid)
            uint32_t nn, qb;
            pr.fKB.divmod((uint32_t)(k0 / BK), nn, qb);
            const int q0 = (int)qb * BK, sh = tr * pr.Wp;
            tma_4d(base, &xa_hi, &full[s], q0 + sh, i0, (int)nn, ts);
            tma_4d(base + C::A_BYTES, &xa_lo, &full[s], q0 + sh, i0, (int)nn, ts);
            tma_4d(base + 2 * C::A_BYTES, &b_hi, &full[s], q0, j0, (int)nn, 0);
            tma_4d(base + 2 * C::A_BYTES + C::B_BYTES, &b_lo, &full[s], q0, j0, (int)nn, 0);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ===== MMA issuer: the whole warp walks the pipeline (warp-uniform values stay in uniform
    // registers), one elected lane issues.  Stage descriptors are precomputed: within the 128B
    // swizzle atom a k step of 8 tf32 (32 bytes) is +2 in the descriptor's address field. =====
    const uint64_t d0 = desc_kmajor(smem_u32(smem));
    const uint64_t dstage = (uint64_t)(C::STAGE >> 4);
    const uint64_t dalo = (uint64_t)(C::A_BYTES >> 4), dbhi = (uint64_t)((2 * C::A_BYTES) >> 4);
    const uint64_t dblo = (uint64_t)((2 * C::A_BYTES + C::B_BYTES) >> 4);
    uint32_t it = 0, cc = 0;
    for (int t = blockIdx.x; t < pr.ntiles; t += gridDim.x) {
      int kbeg, kend;
      krange(t, kbeg, kend);
      const int nkb = kend > kbeg ? (kend - kbeg + BK - 1) / BK : 0;
      uint32_t dbig = 0, dsmall = 0;
      for (int kb = 0; kb < nkb; ++kb, ++it) {
        const int s = it % C::STAGES;
        const bool first = (kb % CK) == 0;
        if (first) {
          const uint32_t buf = cc % C::NBUF;
          if (cc >= (uint32_t)C::NBUF && pr.noload < 4) {
            mbar_wait(&acce[buf], ((cc / C::NBUF) - 1) & 1);
            tc_fence_after();
          }
          dbig = tmem + buf * 2 * BN;
          dsmall = dbig + BN;
        }
        mbar_wait(&full[s], (it / C::STAGES) & 1);
        tc_fence_after();
        if (elect_one()) {
          const uint64_t ds = d0 + (uint64_t)s * dstage;
          if (pr.noload < 3) {  // (diagnostics: PB_TMA_NOLOAD=3 skips the MMAs)
#pragma unroll
            for (int kk = 0; kk < BK / 8; ++kk) {
              const uint64_t ahi = ds + 2 * kk, alo = ahi + dalo, bhi = ahi + dbhi, blo = ahi + dblo;
              const uint32_t acc = !(first && kk == 0);
              mma_tf32(dsmall, alo, bhi, C::IDESC, acc);
              mma_tf32(dsmall, ahi, blo, C::IDESC, 1);
              mma_tf32(dbig, ahi, bhi, C::IDESC, acc);
            }
          }
          mma_commit(&empty[s]);
          if (((kb % CK) == CK - 1 || kb == nkb - 1) && pr.noload < 4) mma_commit(&accf[cc % C::NBUF]);
        }
        __syncwarp();
        if ((kb % CK) == CK - 1 || kb == nkb - 1) ++cc;
      }
    }
  } else {
    // ===== drain + epilogue: TMEM lane quadrant is fixed by warp % 4, 32 columns per warp =====
    const int q = warp & 3, cg = (warp - 2) >> 2;
    const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(cg * 32);
    uint32_t cc = 0;
    for (int t = blockIdx.x; t < pr.ntiles; t += gridDim.x) {
      const int z = t / per_z, rem = t - z * per_z;
      const int i0 = (rem / pr.tj) * BM, j0 = (rem % pr.tj) * BN;
      int kbeg, kend;
      krange(t, kbeg, kend);
      const int nkb = kend > kbeg ? (kend - kbeg + BK - 1) / BK : 0;
      float acc[32];
#pragma unroll
      for (int e = 0; e < 32; ++e) acc[e] = 0.f;
      const int nch = pr.noload >= 4 ? 0 : (nkb + CK - 1) / CK;  // (diagnostics: 4 = no drain)
      for (int c = 0; c < nch; ++c, ++cc) {
        const uint32_t buf = cc % C::NBUF;
        mbar_wait(&accf[buf], (cc / C::NBUF) & 1);
        tc_fence_after();
        uint32_t rb[32], rs[32];
        if (pr.noload >= 2) {  // diagnostics: release the chunk unread
          tc_fence_before();
          mbar_arrive(&acce[buf]);
          continue;
        }
        tmem_ld16(lane_base + buf * 2 * BN, rb);
        tmem_ld16(lane_base + buf * 2 * BN + 16, rb + 16);
        tmem_ld16(lane_base + buf * 2 * BN + BN, rs);
        tmem_ld16(lane_base + buf * 2 * BN + BN + 16, rs + 16);
        tmem_wait_ld();
        tc_fence_before();
        mbar_arrive(&acce[buf]);  // the registers hold the chunk: the MMA may refill the buffer
#pragma unroll
        for (int e = 0; e < 32; ++e)
          acc[e] = __fadd_rn(acc[e], __fadd_rn(__uint_as_float(rb[e]), __uint_as_float(rs[e])));
      }
      if (pr.noload >= 5) continue;  // (diagnostics: 5 = no epilogue stores)
      const int i = i0 + q * 32 + (tid & 31);
      typename OUT::Row orow = out.row(z, i);
#pragma unroll
      for (int e = 0; e < 32; ++e) out.put(orow, j0 + cg * 32 + e, acc[e]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<C::TMEM_COLS>(tmem);
  }
}

// ---- pre-pass kernels -----------------------------------------------------------------------
// hi = rna_tf32(x), lo = rna_tf32(x - hi): the same split as gemm_tc.cu's producers (free
// here: the pre-pass is HBM-bound), |lo| <= 2^-11 |x|, per-product error <= ~2^-22
__device__ __forceinline__ void split_hl(float x, float& h, float& l) {
  split1(x, h, l);
}

// x[n][c][p] (NCHW, C % 32 == 0) -> hi/lo[n][p][c] (NHWC), a 32x32 tile per block through smem
__global__ void __launch_bounds__(256) nchw_split_nhwc(const float* __restrict__ x, float* __restrict__ hi,
                                                       float* __restrict__ lo, int C, int P) {
  // a 32-channel x 128-pixel tile per block: 16 loads in flight per thread before the barrier
  // (a 64-pixel tile left the pass latency-bound at ~2 TB/s: one round trip per 8 KB block)
  __shared__ float t[32][129];
  const int n = blockIdx.z, c0 = blockIdx.y * 32, p0 = blockIdx.x * 128;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const float* src = x + ((int64_t)n * C + c0) * P + p0;
  float v[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const int c = ty + 8 * (k & 3), px = tx + 32 * (k >> 2);
    v[k] = p0 + px < P ? __ldg(src + (int64_t)c * P + px) : 0.f;
  }
#pragma unroll
  for (int k = 0; k < 16; ++k) t[ty + 8 * (k & 3)][tx + 32 * (k >> 2)] = v[k];
  __syncthreads();
  const int64_t ob = ((int64_t)n * P + p0) * C + c0;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const int p = ty + 8 * k;
    if (p0 + p < P) {
      float h, l;
      split_hl(t[tx][p], h, l);
      hi[ob + (int64_t)p * C + tx] = h;
      lo[ob + (int64_t)p * C + tx] = l;
    }
  }
}

// x[plane][H][W] -> hi/lo[copy][plane][L] for copy = 0..copies-1: position q of copy j holds
// x[hq - off][wq - off] with hq * Wp + wq = q + j (zero outside the image), L % 4 == 0
__global__ void __launch_bounds__(256) split_planes(const float* __restrict__ x, float* __restrict__ hi,
                                                    float* __restrict__ lo, int64_t n, int copies, FastDiv fL,
                                                    FastDiv fWp, int H, int W, int off) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t plane, q;
    fL.divmod((uint32_t)i, plane, q);
    for (int j = 0; j < copies; ++j) {
      uint32_t hq, wq;
      fWp.divmod(q + j, hq, wq);
      const int hh = (int)hq - off, ww = (int)wq - off;
      float h = 0.f, l = 0.f;
      if ((unsigned)hh < (unsigned)H && (unsigned)ww < (unsigned)W)
        split_hl(__ldg(x + ((int64_t)plane * H + hh) * W + ww), h, l);
      hi[i + j * n] = h;
      lo[i + j * n] = l;
    }
  }
}

// weights w[f][c][r][s] -> hi/lo[a][(r,s,b)]: fprop (a,b) = (f,c); dgrad (a,b) = (c,f) with the
// taps flipped (r,s) -> (KH-1-r, KW-1-s)
__global__ void weight_split(const float* __restrict__ w, float* __restrict__ hi, float* __restrict__ lo, int F,
                             int Cc, int KH, int KW, int dgrad, FastDiv fRS, FastDiv fC) {
  // walks the OUTPUT index so the two planes are written coalesced; the (small, L2-resident)
  // weights are gathered.  fC divides by the plane's innermost extent: Cc (fprop) or F (dgrad)
  const int RS = KH * KW;
  const uint32_t n = (uint32_t)F * Cc * RS;  // < 2^31 (the callers' fits() checks)
  for (uint32_t o = blockIdx.x * blockDim.x + threadIdx.x; o < n; o += gridDim.x * blockDim.x) {
    uint32_t t, inner, outer, rsu;
    fC.divmod(o, t, inner);
    fRS.divmod(t, outer, rsu);
    int f, c, rs = (int)rsu;
    if (!dgrad) {  // o = (f*RS + rs)*Cc + c
      f = (int)outer;
      c = (int)inner;
    } else {       // o = (c*RS + rs')*F + f; dgrad == 1 stores the taps flipped: rs' = RS-1-rs
      f = (int)inner;
      c = (int)outer;
      if (dgrad == 1) rs = RS - 1 - rs;
    }
    float h, l;
    split_hl(__ldg(w + ((int64_t)f * Cc + c) * RS + rs), h, l);
    hi[o] = h;
    lo[o] = l;
  }
}

// strided view v(r, k) = src[r * sr + k * sk] -> hi/lo[r][k] with row pitch kp (k >= K: 0),
// a 32x32 tile per block through shared memory; loads run along whichever axis is unit stride
__global__ void __launch_bounds__(256) kmajor_split(const float* __restrict__ src, float* __restrict__ hi,
                                                    float* __restrict__ lo, int R, int K, int kp, int64_t sr,
                                                    int64_t sk) {
  __shared__ float t[32][33];
  const int r0 = blockIdx.y * 32, k0 = blockIdx.x * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const bool along_r = sk != 1 && sr == 1;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int a = ty + 8 * q;  // the slow index of this load
    const int r = along_r ? r0 + tx : r0 + a, k = along_r ? k0 + a : k0 + tx;
    const float v = r < R && k < K ? __ldg(src + (int64_t)r * sr + (int64_t)k * sk) : 0.f;
    if (along_r) t[tx][a] = v;
    else t[a][tx] = v;
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int rr = ty + 8 * q, r = r0 + rr, k = k0 + tx;
    if (r < R && k < kp) {
      float h, l;
      split_hl(t[rr][tx], h, l);
      hi[(int64_t)r * kp + k] = h;
      lo[(int64_t)r * kp + k] = l;
    }
  }
}

// the operand planes of a 1x1 wgrad: v(r, k) = src[r * sr + n * sn + ho * sh + wo * sw] with
// k = (n, ho, wo) over an N x HO x WO grid -> hi/lo[r][k], row pitch kp (k >= K: 0).  Lanes run
// along k (consecutive wo), so loads are unit-stride (stride 1) or every other float (stride 2).
__global__ void __launch_bounds__(256) kmajor_split_grid(const float* __restrict__ src, float* __restrict__ hi,
                                                         float* __restrict__ lo, int R, int K, int kp, int64_t sr,
                                                         int64_t sn, int64_t sh, int64_t sw, FastDiv fP, FastDiv fWO) {
  const int r0 = blockIdx.y * 8, k = blockIdx.x * 32 + (threadIdx.x & 31);
  const int r = r0 + (threadIdx.x >> 5);
  if (r >= R || k >= kp) return;
  float h = 0.f, l = 0.f;
  if (k < K) {
    uint32_t n, q, ho, wo;
    fP.divmod((uint32_t)k, n, q);
    fWO.divmod(q, ho, wo);
    split_hl(__ldg(src + (int64_t)r * sr + (int64_t)n * sn + (int64_t)ho * sh + (int64_t)wo * sw), h, l);
  }
  hi[(int64_t)r * kp + k] = h;
  lo[(int64_t)r * kp + k] = l;
}

// kmajor_split_grid for stride-1 rows whose plane length HO*WO is a multiple of 4: each
// thread converts 4 consecutive k (one image, contiguous in the source) with 16-byte accesses
__global__ void __launch_bounds__(256) kmajor_split_grid4(const float* __restrict__ src, float* __restrict__ hi,
                                                          float* __restrict__ lo, int R, int K, int kp, int64_t sr,
                                                          int64_t sn, FastDiv fP) {
  const int r = blockIdx.y * 8 + (threadIdx.x >> 5);
  const int k = (blockIdx.x * 32 + (threadIdx.x & 31)) * 4;
  if (r >= R || k >= kp) return;
  float4 h = make_float4(0.f, 0.f, 0.f, 0.f), l = h;
  if (k < K) {  // K % 4 == 0 here, so the vector is all in range
    uint32_t n, q;
    fP.divmod((uint32_t)k, n, q);
    const float4 v = __ldg(reinterpret_cast<const float4*>(src + (int64_t)r * sr + (int64_t)n * sn + q));
    split_hl(v.x, h.x, l.x);
    split_hl(v.y, h.y, l.y);
    split_hl(v.z, h.z, l.z);
    split_hl(v.w, h.w, l.w);
  }
  *reinterpret_cast<float4*>(hi + (int64_t)r * kp + k) = h;
  *reinterpret_cast<float4*>(lo + (int64_t)r * kp + k) = l;
}

// out[i * ld + j] (a row-major matrix whose row index runs along the TMEM lanes)
struct OutRows {
  float* p;
  int Mi, Nj;
  int64_t ld;
  struct Row {
    float* p;
  };
  __device__ __forceinline__ Row row(int, int i) const {
    Row o;
    o.p = i < Mi ? p + (int64_t)i * ld : nullptr;
    return o;
  }
  __device__ __forceinline__ void put(const Row& rw, int j, float v) const {
    if (rw.p && j < Nj) rw.p[j] = v;
  }
};

// sub-pixel dgrad weights: class (ah, aw) of a stride-s dgrad keeps the taps r = ah + p - s*d
// (d = dh0 + tr, tr < th) and s' = aw + p - s*d' (d' = dw0 + ts, ts < tw); plane
// [C][(tr, ts, f)] (K-major over the gradient's channels f), taps in increasing displacement
__global__ void weight_split_class(const float* __restrict__ w, float* __restrict__ hi, float* __restrict__ lo, int F,
                                   int Cc, int KH, int KW, int rh0, int th, int rw0, int tw, int s) {
  const int64_t n = (int64_t)Cc * th * tw * F;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n; idx += (int64_t)gridDim.x * blockDim.x) {
    const int f = (int)(idx % F);
    int64_t t = idx / F;
    const int ts = (int)(t % tw);
    t /= tw;
    const int tr = (int)(t % th);
    const int c = (int)(t / th);
    const int r = rh0 - s * tr, q = rw0 - s * ts;  // tap for displacement dh0 + tr, dw0 + ts
    float h, l;
    split_hl(w[(((int64_t)f * Cc + c) * KH + r) * KW + q], h, l);
    hi[idx] = h;
    lo[idx] = l;
  }
}

// strided dgrad, second half: dx[n][c][h][w] = sum over the taps (r, s) that land on the
// stride grid of Y[(c, r, s)][(n, ho, wo)], ho = (h + ph - r) / sh; taps in (r, s) order, f64
__global__ void __launch_bounds__(256) col2im_dgrad(const float* __restrict__ Y, float* __restrict__ dx, int N, int C,
                                                    int H, int W, int KH, int KW, int SH, int SW, int PH, int PW,
                                                    int HO, int WO) {
  const int64_t total = (int64_t)N * C * H * W;
  const int64_t P = (int64_t)N * HO * WO;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int w = (int)(i % W);
    int64_t t = i / W;
    const int h = (int)(t % H);
    t /= H;
    const int c = (int)(t % C);
    const int n = (int)(t / C);
    double acc = 0.0;
    for (int r = 0; r < KH; ++r) {
      const int hh = h + PH - r;
      if (hh < 0 || hh % SH) continue;
      const int ho = hh / SH;
      if (ho >= HO) continue;
      for (int s = 0; s < KW; ++s) {
        const int ww = w + PW - s;
        if (ww < 0 || ww % SW) continue;
        const int wo = ww / SW;
        if (wo >= WO) continue;
        acc += (double)__ldg(Y + ((int64_t)(c * KH + r) * KW + s) * P + ((int64_t)n * HO + ho) * WO + wo);
      }
    }
    dx[i] = (float)acc;
  }
}

// ---- host ----------------------------------------------------------------------------------
template <int BN, bool WG, class OUT>
static int launch(const CUtensorMap& ah, const CUtensorMap& al, const CUtensorMap& bh, const CUtensorMap& bl,
                  Prob& pr, const OUT& out) {
  typedef Cfg<BN, WG> C;
  static bool attr = false;
  if (!attr) {
    PB_CUDA(cudaFuncSetAttribute(tma_conv_kernel<BN, WG, OUT>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
    attr = true;
  }
  pr.ti = (pr.Mi + BM - 1) / BM;
  pr.tj = (pr.Nj + BN - 1) / BN;
  const int64_t nt = (int64_t)pr.ti * pr.tj * pr.zdim;
  if (nt >= ((int64_t)1 << 31)) return PB_ERR_UNSUPPORTED;
  pr.ntiles = (int)nt;
  static const int noload = getenv("PB_TMA_NOLOAD") ? atoi(getenv("PB_TMA_NOLOAD")) : 0;
  pr.noload = noload;
  const int grid = (int)(nt < num_sms() ? nt : num_sms());
  tma_conv_kernel<BN, WG, OUT><<<grid, C::THREADS, C::SMEM, compute_stream()>>>(ah, al, bh, bl, pr, out);
  PB_LAUNCHED();
  return PB_OK;
}

static int split_act(const float* x, float* hi, float* lo, int N, int C, int P) {
  dim3 grid((P + 127) / 128, C / 32, N);
  nchw_split_nhwc<<<grid, 256, 0, compute_stream()>>>(x, hi, lo, C, P);
  PB_LAUNCHED();
  return PB_OK;
}

static bool fits(int64_t v) { return v < ((int64_t)1 << 31) - 1024; }

static Prob make_prob(int N, int H, int W, int C, int KH, int KW, int SH, int SW, int PH, int PW) {
  Prob pr{};
  pr.N = N, pr.H = H, pr.W = W, pr.C = C, pr.KH = KH, pr.KW = KW, pr.SH = SH, pr.SW = SW, pr.PH = PH, pr.PW = PW;
  pr.HO = (H + 2 * PH - KH) / SH + 1;
  pr.WO = (W + 2 * PW - KW) / SW + 1;
  pr.fP = FastDiv((uint32_t)(pr.HO * pr.WO));
  pr.fWO = FastDiv((uint32_t)pr.WO);
  return pr;
}

static int conv_bn(const Prob& pr) { return pr.Nj <= 64 ? 64 : 128; }  // (128 wins even with a ragged wave)

// split K over z when the tile grid leaves SMs idle (the 14x14 and 7x7 stages at b32: 98 and
// 52 tiles on 148 SMs): minimise waves x k-blocks per tile plus the partials' round trip
// (folded in f64, in split order, by fold_partials -- deterministic)
static int conv_splits(const Prob& pr) {
  const int64_t tiles = (int64_t)((pr.Mi + BM - 1) / BM) * ((pr.Nj + conv_bn(pr) - 1) / conv_bn(pr));
  const int64_t nkb = (pr.K + BK - 1) / BK, sms = num_sms();
  if (tiles >= sms || nkb < 8) return 1;
  int best = 1;
  double best_cost = (double)((tiles + sms - 1) / sms) * nkb;
  static const double per_kb = getenv("PB_SPLIT_BYTES_PER_KB") ? atof(getenv("PB_SPLIT_BYTES_PER_KB")) : 637500.0;
  for (int sp = 2; sp <= 16 && nkb / sp >= 4; ++sp) {
    const double cost = (double)((tiles * sp + sms - 1) / sms) * ((nkb + sp - 1) / sp) +
                        (double)pr.Mi * pr.Nj * sp / per_kb;  // ~one k-block per 2.5 MB of partials
    if (cost < best_cost * 0.95) {
      best = sp;
      best_cost = cost;
    }
  }
  return best;
}

static size_t conv_partial_bytes(const Prob& pr) {
  const int sp = conv_splits(pr);
  return sp > 1 ? ((size_t)sp * pr.Mi * pr.Nj * 4 + 1023) / 1024 * 1024 : 0;
}

// D = implicit GEMM over the NHWC planes (xh, xl) and K-major weight planes (wh, wl) [Nj][K];
// pw: conv_partial_bytes(pr) of scratch for split K (or null: no split)
template <class OUT>
static int run_conv(Prob& pr, const float* xh, const float* xl, const float* wh, const float* wl, const OUT& o,
                    float* pw = nullptr) {
  CUtensorMap ah, al, bh, bl;
  const int BN = conv_bn(pr);
  static int plain_ok = -1;  // experiment hook: PB_TMA_PLAIN=0 keeps 1x1 convs on im2col boxes
  if (plain_ok < 0) {
    const char* e = getenv("PB_TMA_PLAIN");
    plain_ok = !(e && e[0] == '0');
  }
  pr.plain = plain_ok && pr.KH == 1 && pr.KW == 1 && pr.SH == 1 && pr.SW == 1 && pr.PH == 0 && pr.PW == 0;
  const int64_t pix = (int64_t)pr.N * pr.H * pr.W;
  bool ok = pr.plain ? map_2d(&ah, xh, pr.C, pix, BM) && map_2d(&al, xl, pr.C, pix, BM)
                     : map_im2col(&ah, xh, pr.N, pr.H, pr.W, pr.C, pr.KH, pr.KW, pr.SH, pr.SW, pr.PH, pr.PW, BM) &&
                           map_im2col(&al, xl, pr.N, pr.H, pr.W, pr.C, pr.KH, pr.KW, pr.SH, pr.SW, pr.PH, pr.PW, BM);
  if (!ok || !map_2d(&bh, wh, pr.K, pr.Nj, BN) || !map_2d(&bl, wl, pr.K, pr.Nj, BN))
    return fail(PB_ERR_CUDA, "tma conv: tensor map encoding failed");
  pr.zdim = 1;
  const int sp = pw ? conv_splits(pr) : 1;
  if (sp > 1) {
    const int nkb = (pr.K + BK - 1) / BK;
    pr.kper = (nkb + sp - 1) / sp * BK;
    pr.zdim = (pr.K + pr.kper - 1) / pr.kper;
    OutPartial op{pw, pr.Mi, pr.Nj};
    int rc = BN == 64 ? launch<64, false>(ah, al, bh, bl, pr, op) : launch<128, false>(ah, al, bh, bl, pr, op);
    if (rc) return rc;
    launch_fold<OUT>(pw, pr.zdim, pr.Mi, pr.Nj, o, compute_stream());
    PB_LAUNCHED();
    return PB_OK;
  }
  if (BN == 64) return launch<64, false>(ah, al, bh, bl, pr, o);
  return launch<128, false>(ah, al, bh, bl, pr, o);
}

static bool geometry_ok(const Prob& pr) {
  // im2col corners and 16-bit tap offsets; the C % 32 channel blocks; i32 indexing
  return pr.C % 32 == 0 && pr.KH <= 32 && pr.KW <= 32 && pr.PH <= 64 && pr.PW <= 64 && pr.HO > 0 && pr.WO > 0 &&
         pr.SH <= 8 && pr.SW <= 8;
}

}  // namespace tma
}  // namespace pb

using namespace pb;
using namespace pb::tma;

static int g_tma = 1;

// 1x1 convs over more pixels than this stay on gemm_tc.cu.  Round 1 measured 56x56 planes (b32)
// losing to the hi/lo pre-pass; with round 2's MMA issue loop and drains the TMA kernel wins
// there too (ResNet-50 step 23.52 -> 23.48 ms, profiles/r2/experiments/conv_route_sweep.txt),
// so there is no limit by default; PB_TMA_1X1_MAXPIX sets one (experiment hook)
static int64_t max_1x1_pixels() {
  static const int64_t v = getenv("PB_TMA_1X1_MAXPIX") ? atoll(getenv("PB_TMA_1X1_MAXPIX")) : ((int64_t)1 << 40);
  return v;
}

// strided k x k dgrad by sub-pixel decomposition: output pixel (s*a + ah, s*b + aw) only meets
// taps r = ah + p (mod s), at gradient row a + (ah + p - r) / s.  Each of the s*s classes is a
// stride-1 correlation of g (NHWC planes, shared) with its own sub-kernel and asymmetric halo,
// run through the TMA implicit GEMM and scattered into dx by OutScatter; the classes partition
// dx, so there is no memset and no zero work (the useful FLOPs exactly).
static int dgrad_subpixel(const pb_tensor* gr, const pb_tensor* w, const pb_conv* p, const pb_tensor* out) {
  static int off = -1;  // experiment hook: PB_DG_SUB=0 keeps the col2im / gemm_tc paths
  if (off < 0) {
    const char* e = getenv("PB_DG_SUB");
    off = e && e[0] == '0';
  }
  if (off) return PB_ERR_UNSUPPORTED;
  const int N = (int)out->shape[0], Cx = (int)out->shape[1], H = (int)out->shape[2], W = (int)out->shape[3];
  const int F = (int)w->shape[0], KH = (int)w->shape[2], KW = (int)w->shape[3];
  const int HO = (int)gr->shape[2], WO = (int)gr->shape[3];
  const int sh = p->stride_h, sw = p->stride_w, ph = p->pad_h, pw = p->pad_w;
  if (F % 32 || Cx % 4 || Cx < 32 || N == 0 || sh > 4 || sw > 4 || ph >= KH || pw >= KW) return PB_ERR_UNSUPPORTED;
  const int64_t act = (int64_t)N * F * HO * WO;
  if (!fits(act) || !fits((int64_t)N * Cx * H * W) || !fits((int64_t)Cx * F * KH * KW)) return PB_ERR_UNSUPPORTED;
  // per class: taps, first displacement, first tap, outputs
  struct Axis {
    int d0, t, r0, n;
  };
  auto axis = [](int a, int k, int pad, int s, int in, int extent) {
    Axis x{0, 0, 0, 0};
    x.n = a < extent ? (extent - a + s - 1) / s : 0;
    int dmin = 1 << 20, dmax = -(1 << 20);
    for (int r = 0; r < k; ++r) {
      const int num = a + pad - r;
      if (((num % s) + s) % s) continue;
      const int d = num >= 0 ? num / s : -((-num) / s);
      dmin = d < dmin ? d : dmin;
      dmax = d > dmax ? d : dmax;
    }
    if (dmax < dmin) return x;
    x.d0 = dmin;
    x.t = dmax - dmin + 1;  // displacements are consecutive
    x.r0 = a + pad - s * dmin;
    (void)in;
    return x;
  };
  for (int ah = 0; ah < sh; ++ah)  // every class needs a tap (kernel >= stride), else decline
    for (int aw = 0; aw < sw; ++aw)
      if ((axis(ah, KH, ph, sh, HO, H).n && !axis(ah, KH, ph, sh, HO, H).t) ||
          (axis(aw, KW, pw, sw, WO, W).n && !axis(aw, KW, pw, sw, WO, W).t))
        return PB_ERR_UNSUPPORTED;
  const size_t ab = ((size_t)act * 4 + 1023) / 1024 * 1024;
  const size_t wb = ((size_t)Cx * F * KH * KW * 4 + 1023) / 1024 * 1024;  // >= any class's taps
  char* ws = (char*)workspace(2 * ab + 2 * wb * sh * sw);
  if (!ws) return fail(PB_ERR_OOM, "conv2d_grad_input (sub-pixel): no workspace");
  float *gh = (float*)ws, *gl = (float*)(ws + ab);
  int rc = split_act((const float*)(uintptr_t)gr->ptr, gh, gl, N, F, HO * WO);
  if (rc) return rc;
  float* dx = (float*)(uintptr_t)out->ptr;
  for (int ah = 0; ah < sh; ++ah) {
    const Axis xh = axis(ah, KH, ph, sh, HO, H);
    for (int aw = 0; aw < sw; ++aw) {
      const Axis xw = axis(aw, KW, pw, sw, WO, W);
      if (xh.n == 0 || xw.n == 0) continue;
      float* whi = (float*)(ws + 2 * ab + (size_t)(2 * (ah * sw + aw)) * wb);
      float* wlo = (float*)(ws + 2 * ab + (size_t)(2 * (ah * sw + aw) + 1) * wb);
      weight_split_class<<<grid_for((int64_t)Cx * xh.t * xw.t * F, 256), 256, 0, compute_stream()>>>(
          (const float*)(uintptr_t)w->ptr, whi, wlo, F, Cx, KH, KW, xh.r0, xh.t, xw.r0, xw.t, sh);
      PB_LAUNCHED();
      Prob pr{};
      pr.N = N, pr.H = HO, pr.W = WO, pr.C = F;
      pr.KH = xh.t, pr.KW = xw.t, pr.SH = 1, pr.SW = 1, pr.PH = -xh.d0, pr.PW = -xw.d0;
      pr.HO = xh.n, pr.WO = xw.n;
      pr.fP = FastDiv((uint32_t)(xh.n * xw.n));
      pr.fWO = FastDiv((uint32_t)xw.n);
      pr.F = Cx;
      pr.Mi = N * xh.n * xw.n;
      pr.Nj = Cx;
      pr.K = F * xh.t * xw.t;
      pr.zdim = 1;
      if (!fits((int64_t)pr.Mi * Cx)) return PB_ERR_UNSUPPORTED;
      const int BN = Cx <= 64 ? 64 : 128;
      CUtensorMap am, al, bm, bl;
      const int uw = xw.n + xw.d0 - WO, uh = xh.n + xh.d0 - HO;
      if (!map_im2col_lu(&am, gh, N, HO, WO, F, xw.d0, xh.d0, uw, uh, BM) ||
          !map_im2col_lu(&al, gl, N, HO, WO, F, xw.d0, xh.d0, uw, uh, BM) ||
          !map_2d(&bm, whi, pr.K, Cx, BN) || !map_2d(&bl, wlo, pr.K, Cx, BN))
        return fail(PB_ERR_CUDA, "dgrad (sub-pixel): tensor map encoding failed");
      OutScatter o{dx + (int64_t)ah * W + aw, pr.Mi, Cx, pr.fP, pr.fWO, sh, sw, W, H * W};
      rc = BN == 64 ? launch<64, false>(am, al, bm, bl, pr, o) : launch<128, false>(am, al, bm, bl, pr, o);
      if (rc) return rc;
    }
  }
  return PB_OK;
}

extern "C" {

int pb_tma_enable(int on) {
  g_tma = on ? 1 : 0;
  return PB_OK;
}
int pb_tma_enabled(void) { return g_tma && driver_ok(); }

int pb_conv2d_tma(const pb_tensor* x, const pb_tensor* w, const pb_tensor* bias, const pb_conv* p,
                  const pb_tensor* out) {
  if (!g_tma || !driver_ok()) return PB_ERR_UNSUPPORTED;
  if (x->dtype != PB_F32 || w->dtype != PB_F32 || out->dtype != PB_F32 || (bias && bias->dtype != PB_F32))
    return PB_ERR_UNSUPPORTED;
  if (!is_contiguous(*x) || !is_contiguous(*w) || !is_contiguous(*out)) return PB_ERR_UNSUPPORTED;
  const int N = (int)x->shape[0], C = (int)x->shape[1], H = (int)x->shape[2], W = (int)x->shape[3];
  const int F = (int)w->shape[0], KH = (int)w->shape[2], KW = (int)w->shape[3];
  Prob pr = make_prob(N, H, W, C, KH, KW, p->stride_h, p->stride_w, p->pad_h, p->pad_w);
  if (!geometry_ok(pr) || F == 0 || N == 0) return PB_ERR_UNSUPPORTED;
  // 1x1 convs over large planes are bound by the hi/lo pre-pass (measured: 56x56 at b32
  // runs faster on gemm_tc.cu, which reads x once); 3x3 and the smaller planes win here
  if (KH * KW == 1 && (int64_t)N * H * W > max_1x1_pixels()) return PB_ERR_UNSUPPORTED;
  const int64_t act = (int64_t)N * C * H * W, K = (int64_t)C * KH * KW, rows = (int64_t)N * pr.HO * pr.WO;
  if (!fits(act) || !fits(rows * F) || !fits(K * F) || F % 4 != 0) return PB_ERR_UNSUPPORTED;
  pr.F = F;
  pr.Mi = (int)rows;
  pr.Nj = F;
  pr.K = (int)K;
  const size_t wb = ((size_t)F * K * 4 + 1023) / 1024 * 1024, ab = ((size_t)act * 4 + 1023) / 1024 * 1024;
  const size_t pb = conv_partial_bytes(pr);
  char* ws = (char*)workspace(2 * wb + 2 * ab + pb);
  if (!ws) return fail(PB_ERR_OOM, "conv2d (tma): no workspace");
  float *wh = (float*)ws, *wl = (float*)(ws + wb), *xh = (float*)(ws + 2 * wb), *xl = (float*)(ws + 2 * wb + ab);
  float* pw = pb ? (float*)(ws + 2 * wb + 2 * ab) : nullptr;
  weight_split<<<grid_for((int64_t)F * K, 256), 256, 0, compute_stream()>>>((const float*)(uintptr_t)w->ptr, wh, wl, F, C, KH, KW, 0, FastDiv((uint32_t)((KH) * (KW))), FastDiv((uint32_t)(C)));
  PB_LAUNCHED();
  int rc = split_act((const float*)(uintptr_t)x->ptr, xh, xl, N, C, H * W);
  if (rc) return rc;
  OutConv o{(float*)(uintptr_t)out->ptr, bias ? (const float*)(uintptr_t)bias->ptr : nullptr, (int)rows, F,
            FastDiv((uint32_t)(pr.HO * pr.WO))};
  return run_conv(pr, xh, xl, wh, wl, o, pw);
}

// stride-1 dgrad: dx = conv(g, flip(w)^T) with padding KH-1-ph
int pb_conv2d_grad_input_tma(const pb_tensor* gr, const pb_tensor* w, const pb_conv* p, const pb_tensor* out) {
  if (!g_tma || !driver_ok()) return PB_ERR_UNSUPPORTED;
  if (gr->dtype != PB_F32 || w->dtype != PB_F32 || out->dtype != PB_F32) return PB_ERR_UNSUPPORTED;
  if (!is_contiguous(*gr) || !is_contiguous(*w) || !is_contiguous(*out)) return PB_ERR_UNSUPPORTED;
  const int N = (int)out->shape[0], Cx = (int)out->shape[1], H = (int)out->shape[2], W = (int)out->shape[3];
  const int F = (int)w->shape[0], KH = (int)w->shape[2], KW = (int)w->shape[3];
  const int HO = (int)gr->shape[2], WO = (int)gr->shape[3];
  if ((p->stride_h != 1 || p->stride_w != 1) && KH == 1 && KW == 1 && p->pad_h == 0 && p->pad_w == 0) {
    // strided 1x1: dx[n, :, ho*s, wo*s] = W^T g[n, :, ho, wo], zero elsewhere
    Prob pr = make_prob(N, HO, WO, F, 1, 1, 1, 1, 0, 0);
    const int64_t act = (int64_t)N * F * HO * WO, rows = (int64_t)N * HO * WO;
    if (!geometry_ok(pr) || Cx == 0 || N == 0 || !fits(act) || !fits((int64_t)N * Cx * H * W) || !fits((int64_t)F * Cx))
      return PB_ERR_UNSUPPORTED;
    pr.F = Cx;
    pr.Mi = (int)rows;
    pr.Nj = Cx;
    pr.K = F;
    const size_t wb = ((size_t)Cx * F * 4 + 1023) / 1024 * 1024, ab = ((size_t)act * 4 + 1023) / 1024 * 1024;
    char* ws = (char*)workspace(2 * wb + 2 * ab);
    if (!ws) return fail(PB_ERR_OOM, "conv2d_grad_input (tma): no workspace");
    float *wh = (float*)ws, *wl = (float*)(ws + wb), *gh = (float*)(ws + 2 * wb), *gl = (float*)(ws + 2 * wb + ab);
    PB_CUDA(cudaMemsetAsync((void*)(uintptr_t)out->ptr, 0, (size_t)N * Cx * H * W * 4, compute_stream()));
    weight_split<<<grid_for((int64_t)Cx * F, 256), 256, 0, compute_stream()>>>((const float*)(uintptr_t)w->ptr, wh, wl, F, Cx, 1, 1, 1, FastDiv((uint32_t)((1) * (1))), FastDiv((uint32_t)(F)));
    PB_LAUNCHED();
    int rc = split_act((const float*)(uintptr_t)gr->ptr, gh, gl, N, F, HO * WO);
    if (rc) return rc;
    OutScatter o{(float*)(uintptr_t)out->ptr, (int)rows, Cx, FastDiv((uint32_t)(HO * WO)), FastDiv((uint32_t)WO),
                 p->stride_h, p->stride_w, W, H * W};
    return run_conv(pr, gh, gl, wh, wl, o);
  }
  if ((p->stride_h > 1 || p->stride_w > 1) && KH > 1) {
    int rc = dgrad_subpixel(gr, w, p, out);
    if (rc != PB_ERR_UNSUPPORTED) return rc;
  }
  if ((p->stride_h != 1 || p->stride_w != 1) && ((int64_t)N * HO * WO <= 8192 || Cx < 16)) {
    // strided k x k: Y = W^T g as a GEMM over the gradient pixels (rows) and the (c, r, s)
    // columns, then col2im gathers each dx pixel's on-grid taps.  Measured: wins up to
    // N*HO*WO = 6272 (b32 at 14x14) and for few input channels (the RGB stem: 0.67 vs 8 ms);
    // at 28x28 the 9x-wide Y round trip loses to gemm_tc.cu.
    Prob pr = make_prob(N, HO, WO, F, 1, 1, 1, 1, 0, 0);
    const int RS = KH * KW;
    const int64_t act = (int64_t)N * F * HO * WO, rows = (int64_t)N * HO * WO, cols = (int64_t)Cx * RS;
    if (!geometry_ok(pr) || Cx == 0 || N == 0 || !fits(act) || !fits(rows * cols) || !fits((int64_t)N * Cx * H * W) ||
        !fits(cols * F) || ((int64_t)H + 2 * p->pad_h - KH) / p->stride_h + 1 != HO ||
        ((int64_t)W + 2 * p->pad_w - KW) / p->stride_w + 1 != WO)
      return PB_ERR_UNSUPPORTED;
    pr.F = (int)cols;
    pr.Mi = (int)rows;
    pr.Nj = (int)cols;
    pr.K = F;
    const size_t wb = ((size_t)cols * F * 4 + 1023) / 1024 * 1024, ab = ((size_t)act * 4 + 1023) / 1024 * 1024;
    const size_t yb = (size_t)rows * cols * 4;
    char* ws = (char*)workspace(2 * wb + 2 * ab + yb);
    if (!ws) return fail(PB_ERR_OOM, "conv2d_grad_input (tma): no workspace");
    float *wh = (float*)ws, *wl = (float*)(ws + wb), *gh = (float*)(ws + 2 * wb), *gl = (float*)(ws + 2 * wb + ab);
    float* Y = (float*)(ws + 2 * wb + 2 * ab);
    weight_split<<<grid_for(cols * F, 256), 256, 0, compute_stream()>>>((const float*)(uintptr_t)w->ptr, wh, wl, F, Cx, KH, KW, 2, FastDiv((uint32_t)((KH) * (KW))), FastDiv((uint32_t)(F)));
    PB_LAUNCHED();
    int rc = split_act((const float*)(uintptr_t)gr->ptr, gh, gl, N, F, HO * WO);
    if (rc) return rc;
    OutMat o{Y, (int)rows, (int)cols, rows, 0};  // Y[(c, r, s)][(n, ho, wo)]
    rc = run_conv(pr, gh, gl, wh, wl, o);
    if (rc) return rc;
    col2im_dgrad<<<grid_for((int64_t)N * Cx * H * W, 256), 256, 0, compute_stream()>>>(
        Y, (float*)(uintptr_t)out->ptr, N, Cx, H, W, KH, KW, p->stride_h, p->stride_w, p->pad_h, p->pad_w, HO, WO);
    PB_LAUNCHED();
    return PB_OK;
  }
  const int ph = KH - 1 - p->pad_h, pw = KW - 1 - p->pad_w;
  if (ph < 0 || pw < 0) return PB_ERR_UNSUPPORTED;
  // the "conv" runs over g [N, F, HO, WO] and produces [N, Cx, H, W]
  Prob pr = make_prob(N, HO, WO, F, KH, KW, 1, 1, ph, pw);
  if (!geometry_ok(pr) || pr.HO != H || pr.WO != W || Cx == 0 || N == 0 || Cx % 4 != 0) return PB_ERR_UNSUPPORTED;
  if (KH * KW == 1 && (int64_t)N * H * W > max_1x1_pixels()) return PB_ERR_UNSUPPORTED;  // as in fprop
  const int64_t act = (int64_t)N * F * HO * WO, K = (int64_t)F * KH * KW, rows = (int64_t)N * H * W;
  if (!fits(act) || !fits(rows * Cx) || !fits(K * Cx)) return PB_ERR_UNSUPPORTED;
  pr.F = Cx;
  pr.Mi = (int)rows;
  pr.Nj = Cx;
  pr.K = (int)K;
  const size_t wb = ((size_t)Cx * K * 4 + 1023) / 1024 * 1024, ab = ((size_t)act * 4 + 1023) / 1024 * 1024;
  const size_t pb = conv_partial_bytes(pr);
  char* ws = (char*)workspace(2 * wb + 2 * ab + pb);
  if (!ws) return fail(PB_ERR_OOM, "conv2d_grad_input (tma): no workspace");
  float *wh = (float*)ws, *wl = (float*)(ws + wb), *gh = (float*)(ws + 2 * wb), *gl = (float*)(ws + 2 * wb + ab);
  float* part = pb ? (float*)(ws + 2 * wb + 2 * ab) : nullptr;
  weight_split<<<grid_for((int64_t)Cx * K, 256), 256, 0, compute_stream()>>>((const float*)(uintptr_t)w->ptr, wh, wl, F, Cx, KH, KW, 1, FastDiv((uint32_t)((KH) * (KW))), FastDiv((uint32_t)(F)));
  PB_LAUNCHED();
  int rc = split_act((const float*)(uintptr_t)gr->ptr, gh, gl, N, F, HO * WO);
  if (rc) return rc;
  OutConv o{(float*)(uintptr_t)out->ptr, nullptr, (int)rows, Cx, FastDiv((uint32_t)(H * W))};
  return run_conv(pr, gh, gl, wh, wl, o, part);
}

// stride-1 wgrad over the padded output grid (see the header): K = N * ceil(HO*Wp / 32) * 32
int pb_conv2d_grad_weight_tma(const pb_tensor* x, const pb_tensor* gr, const pb_conv* p, const pb_tensor* out) {
  static int off = -1;  // experiment hook: PB_TMA_WGRAD=0 sends wgrad to gemm_tc.cu
  if (off < 0) {
    const char* e = getenv("PB_TMA_WGRAD");
    off = e && e[0] == '0';
  }
  if (!g_tma || off || !driver_ok()) return PB_ERR_UNSUPPORTED;
  if (x->dtype != PB_F32 || gr->dtype != PB_F32 || out->dtype != PB_F32) return PB_ERR_UNSUPPORTED;
  if (!is_contiguous(*x) || !is_contiguous(*gr) || !is_contiguous(*out)) return PB_ERR_UNSUPPORTED;
  if (p->stride_h != 1 || p->stride_w != 1 || p->pad_h != p->pad_w) return PB_ERR_UNSUPPORTED;
  const int N = (int)x->shape[0], C = (int)x->shape[1], H = (int)x->shape[2], W = (int)x->shape[3];
  const int F = (int)out->shape[0], KH = (int)out->shape[2], KW = (int)out->shape[3];
  Prob pr = make_prob(N, H, W, C, KH, KW, 1, 1, p->pad_h, p->pad_w);
  if (pr.HO <= 0 || pr.WO <= 0 || N == 0 || C == 0 || F == 0) return PB_ERR_UNSUPPORTED;
  const int HO = pr.HO, RS = KH * KW, pad = p->pad_h;
  {
    // Measured on B200 (tools/conv_table.py): the plane pre-pass and the hi/lo operand stream
    // cost more than they save on large pixel counts, where gemm_tc.cu's SIMT-fed wgrad wins;
    // take the TMA kernel for small planes, 3x3 taps up to 28x28 at b32, and wide 1x1 convs.
    static int force = -1;  // experiment hook: PB_TMA_WGRAD=2 takes every eligible shape
    if (force < 0) {
      const char* e = getenv("PB_TMA_WGRAD");
      force = e && e[0] == '2';
    }
    const int64_t P = (int64_t)N * HO * pr.WO;
    static const int64_t p2 = getenv("PB_TMA_WG_P2") ? atoll(getenv("PB_TMA_WG_P2")) : 25088;  // experiment hook
    const bool win = P <= 6272 || (P <= p2 && (RS > 1 || (int64_t)C * F >= 131072));
    if (!force && !win) return PB_ERR_UNSUPPORTED;
  }
  pr.Wp = (W + 2 * pad + 3) / 4 * 4;
  const int64_t Hp = H + 2 * pad;
  const int64_t Lx = (Hp * pr.Wp + 3) / 4 * 4, Lg = ((int64_t)HO * pr.Wp + 3) / 4 * 4;
  const int64_t kb_img = ((int64_t)HO * pr.Wp + BK - 1) / BK, KB = (int64_t)N * kb_img;
  const int64_t xs = (int64_t)N * C * Lx, gs = (int64_t)N * F * Lg;
  if (!fits(xs * KW) || !fits(gs) || !fits(KB * BK) || !fits((int64_t)F * C * RS) || (int64_t)(KH - 1) * pr.Wp + KW > 65535)
    return PB_ERR_UNSUPPORTED;
  pr.fKB = FastDiv((uint32_t)kb_img);
  pr.F = F;
  pr.Mi = C;
  pr.Nj = F;
  pr.K = (int)(KB * BK);
  const int BN = F <= 64 ? 64 : 128;
  // split K so that tiles x splits fill the machine; k per split a multiple of BK
  const int64_t tiles = (int64_t)((C + BM - 1) / BM) * ((F + BN - 1) / BN) * RS;
  int splits = 1;
  if (tiles < num_sms()) {
    splits = (int)(num_sms() / tiles);  // whole waves: one more tile than the SM count costs a wave
    const int maxs = (int)(KB / 4);
    if (splits > maxs) splits = maxs;
    if (splits < 1) splits = 1;
  }
  {
    const char* e = getenv("PB_TMA_WG_SPLITS");  // experiment hook
    if (e && atoi(e) > 0) splits = atoi(e);
  }
  int per = (int)((pr.K + splits - 1) / splits);
  per = (per + BK - 1) / BK * BK;
  splits = (pr.K + per - 1) / per;
  pr.kper = per;
  pr.zdim = splits * RS;
  const size_t ab = ((size_t)xs * KW * 4 + 1023) / 1024 * 1024, gb = ((size_t)gs * 4 + 1023) / 1024 * 1024;
  const size_t pb = splits > 1 ? (size_t)splits * F * C * RS * 4 : 0;
  char* ws = (char*)workspace(2 * ab + 2 * gb + pb);
  if (!ws) return fail(PB_ERR_OOM, "conv2d_grad_weight (tma): no workspace");
  float *xh = (float*)ws, *xl = (float*)(ws + ab), *gh = (float*)(ws + 2 * ab), *gl = (float*)(ws + 2 * ab + gb);
  float* part = (float*)(ws + 2 * ab + 2 * gb);
  split_planes<<<grid_for(xs, 256), 256, 0, compute_stream()>>>((const float*)(uintptr_t)x->ptr, xh, xl, xs, KW,
                                                                 FastDiv((uint32_t)Lx), FastDiv((uint32_t)pr.Wp), H,
                                                                 W, pad);
  PB_LAUNCHED();
  split_planes<<<grid_for(gs, 256), 256, 0, compute_stream()>>>((const float*)(uintptr_t)gr->ptr, gh, gl, gs, 1,
                                                                 FastDiv((uint32_t)Lg), FastDiv((uint32_t)pr.Wp), HO,
                                                                 pr.WO, 0);
  PB_LAUNCHED();
  CUtensorMap ah, al, bh, bl;
  if (!map_planes(&ah, xh, KW, N, C, Lx, BM) || !map_planes(&al, xl, KW, N, C, Lx, BM) ||
      !map_planes(&bh, gh, 1, N, F, Lg, BN) || !map_planes(&bl, gl, 1, N, F, Lg, BN))
    return fail(PB_ERR_CUDA, "wgrad (tma): tensor map encoding failed");
  float* dw = (float*)(uintptr_t)out->ptr;
  OutWgrad o{splits > 1 ? part : dw, C, F, RS};
  int rc = BN == 64 ? launch<64, true>(ah, al, bh, bl, pr, o) : launch<128, true>(ah, al, bh, bl, pr, o);
  if (rc || splits == 1) return rc;
  OutMat fin{dw, C * RS, F, (int64_t)C * RS, 0};
  launch_fold<OutMat>(part, splits, C * RS, F, fin, compute_stream());
  PB_LAUNCHED();
  return PB_OK;
}

// 1x1 grad_weight (no padding, any stride; minml/kernels.py:231-239) as a plain TMA GEMM over
// K = N x HO x WO: dw[f][c] = sum_k g[n, f, ho, wo] x[n, c, ho*s, wo*s].  Both operands are
// split into K-major planes by kmajor_split_grid; the larger of C and F runs along the TMEM
// lanes (a 64-row side would leave half of each 128-lane tile idle); split K fills the SMs and
// the partials fold in f64 in split order.
int pb_conv2d_grad_weight_mm(const pb_tensor* x, const pb_tensor* gr, const pb_conv* p, const pb_tensor* out) {
  static int off = -1;  // experiment hook: PB_WG_MM=0 sends 1x1 wgrad to the other kernels
  if (off < 0) {
    const char* e = getenv("PB_WG_MM");
    off = e && e[0] == '0';
  }
  if (!g_tma || off || !driver_ok()) return PB_ERR_UNSUPPORTED;
  if (x->dtype != PB_F32 || gr->dtype != PB_F32 || out->dtype != PB_F32) return PB_ERR_UNSUPPORTED;
  if (!is_contiguous(*x) || !is_contiguous(*gr) || !is_contiguous(*out)) return PB_ERR_UNSUPPORTED;
  if (out->shape[2] != 1 || out->shape[3] != 1 || p->pad_h || p->pad_w) return PB_ERR_UNSUPPORTED;
  const int64_t N = x->shape[0], C = x->shape[1], H = x->shape[2], W = x->shape[3], F = out->shape[0];
  const int64_t HO = gr->shape[2], WO = gr->shape[3];
  const int64_t K = N * HO * WO;
  if (C < 64 || F < 64 || K < 256 || !fits(K * (C > F ? C : F)) || !fits(N * C * H * W) || !fits(N * F * HO * WO))
    return PB_ERR_UNSUPPORTED;
  // measured per shape (tools/conv_table.py, ResNet-50 b32, vectorised pre-pass): this path
  // wins for strided projections (0.246 -> 0.132 ms at 56->28), 14x14 / 7x7 planes, and
  // stride-1 planes with C*F >= 32768 or F > C (64->256 @56: 0.162 -> 0.123 ms); the
  // SIMT-fed kernel keeps 64->64 and 256->64 @56x56
  static int force = -1;  // experiment hook: PB_WG_MM=2 takes every eligible shape
  if (force < 0) {
    const char* e = getenv("PB_WG_MM");
    force = e && e[0] == '2';
  }
  if (!force && p->stride_h == 1 && p->stride_w == 1 && HO * WO > 196 && C * F < 32768 && F <= C)
    return PB_ERR_UNSUPPORTED;
  const bool swap = C < F;  // rows i of D: the larger channel count
  const int64_t Mi = swap ? F : C, Nj = swap ? C : F;
  const int BN = Nj <= 64 ? 64 : 128;
  const int64_t kp = (K + 3) / 4 * 4;
  Prob pr{};
  pr.plain = 1;
  pr.Mi = (int)Mi;
  pr.Nj = (int)Nj;
  pr.K = (int)kp;
  pr.C = (int)kp;
  pr.KH = pr.KW = pr.SH = pr.SW = 1;
  const int64_t tiles = ((Mi + BM - 1) / BM) * ((Nj + BN - 1) / BN);
  const int64_t kblocks = (kp + BK - 1) / BK;
  int splits = (int)(num_sms() / tiles);
  if (splits > kblocks / 4) splits = (int)(kblocks / 4);
  if (splits < 1) splits = 1;
  const int per = (int)((kblocks + splits - 1) / splits) * BK;
  splits = (int)((kp + per - 1) / per);
  pr.kper = per;
  pr.zdim = splits;
  const size_t ib = ((size_t)Mi * kp * 4 + 1023) / 1024 * 1024, jb = ((size_t)Nj * kp * 4 + 1023) / 1024 * 1024;
  const size_t part = splits > 1 ? (size_t)splits * Mi * Nj * 4 : 0;
  char* ws = (char*)workspace(2 * ib + 2 * jb + part);
  if (!ws) return fail(PB_ERR_OOM, "conv2d_grad_weight (mm): no workspace");
  float *ih = (float*)ws, *il = (float*)(ws + ib), *jh = (float*)(ws + 2 * ib), *jl = (float*)(ws + 2 * ib + jb);
  float* pw = (float*)(ws + 2 * ib + 2 * jb);
  cudaStream_t s = compute_stream();
  const FastDiv fP((uint32_t)(HO * WO)), fWO((uint32_t)WO);
  const float* px = (const float*)(uintptr_t)x->ptr;
  const float* pg = (const float*)(uintptr_t)gr->ptr;
  // x operand: rows c, k -> x[n, c, ho*sh, wo*sw]; g operand: rows f, k -> g[n, f, ho, wo]
  const float* src_i = swap ? pg : px;
  const float* src_j = swap ? px : pg;
  const int64_t xs[4] = {H * W, C * H * W, (int64_t)p->stride_h * W, (int64_t)p->stride_w};
  const int64_t gs[4] = {HO * WO, F * HO * WO, WO, 1};
  const int64_t* si = swap ? gs : xs;
  const int64_t* sj = swap ? xs : gs;
  const bool vec = p->stride_h == 1 && p->stride_w == 1 && (HO * WO) % 4 == 0 && x->ptr % 16 == 0 && gr->ptr % 16 == 0;
  if (vec) {  // K = N*HO*WO is then a multiple of 4 too (kp == K)
    kmajor_split_grid4<<<dim3((unsigned)((kp / 4 + 31) / 32), (unsigned)((Mi + 7) / 8)), 256, 0, s>>>(
        src_i, ih, il, (int)Mi, (int)K, (int)kp, si[0], si[1], fP);
    PB_LAUNCHED();
    kmajor_split_grid4<<<dim3((unsigned)((kp / 4 + 31) / 32), (unsigned)((Nj + 7) / 8)), 256, 0, s>>>(
        src_j, jh, jl, (int)Nj, (int)K, (int)kp, sj[0], sj[1], fP);
    PB_LAUNCHED();
  } else {
    kmajor_split_grid<<<dim3((unsigned)((kp + 31) / 32), (unsigned)((Mi + 7) / 8)), 256, 0, s>>>(
        src_i, ih, il, (int)Mi, (int)K, (int)kp, si[0], si[1], si[2], si[3], fP, fWO);
    PB_LAUNCHED();
    kmajor_split_grid<<<dim3((unsigned)((kp + 31) / 32), (unsigned)((Nj + 7) / 8)), 256, 0, s>>>(
        src_j, jh, jl, (int)Nj, (int)K, (int)kp, sj[0], sj[1], sj[2], sj[3], fP, fWO);
    PB_LAUNCHED();
  }
  CUtensorMap ah, al, bh, bl;
  if (!map_2d(&ah, ih, kp, Mi, BM) || !map_2d(&al, il, kp, Mi, BM) || !map_2d(&bh, jh, kp, Nj, BN) ||
      !map_2d(&bl, jl, kp, Nj, BN))
    return fail(PB_ERR_CUDA, "wgrad (mm): tensor map encoding failed");
  float* dw = (float*)(uintptr_t)out->ptr;
  // dw[f][c]: rows i = c (ld 1 along i, F... ) -- OutMat puts (i, j) at i + j * ld; OutRows at i * ld + j
  if (splits == 1) {
    if (swap) {
      OutRows o{dw, (int)Mi, (int)Nj, C};
      return BN == 64 ? launch<64, false>(ah, al, bh, bl, pr, o) : launch<128, false>(ah, al, bh, bl, pr, o);
    }
    OutMat o{dw, (int)Mi, (int)Nj, C, 0};
    return BN == 64 ? launch<64, false>(ah, al, bh, bl, pr, o) : launch<128, false>(ah, al, bh, bl, pr, o);
  }
  OutPartial op{pw, (int)Mi, (int)Nj};
  int rc = BN == 64 ? launch<64, false>(ah, al, bh, bl, pr, op) : launch<128, false>(ah, al, bh, bl, pr, op);
  if (rc) return rc;
  if (swap) {
    OutRows fin{dw, (int)Mi, (int)Nj, C};
    launch_fold<OutRows>(pw, splits, (int)Mi, (int)Nj, fin, s);
  } else {
    OutMat fin{dw, (int)Mi, (int)Nj, C, 0};
    launch_fold<OutMat>(pw, splits, (int)Mi, (int)Nj, fin, s);
  }
  PB_LAUNCHED();
  return PB_OK;
}

// rank-2 matmul C[m][n] = sum_k A[m][k] B[k][n] (minml/kernels.py:166-173) as the plain
// TMA GEMM D[i = n][j = m]: both operands go through kmajor_split (any strides, so the
// autograd's transposed views need no copy) into [rows][kp] planes; split K over z when the
// tile grid is short of the SM count, partials folded in f64 in split order
int pb_matmul_tma(const pb_tensor* a, const pb_tensor* b, const pb_tensor* out) {
  if (!g_tma || !driver_ok()) return PB_ERR_UNSUPPORTED;
  if (a->ndim != 2 || b->ndim != 2 || a->dtype != PB_F32 || b->dtype != PB_F32 || out->dtype != PB_F32 ||
      !is_contiguous(*out))
    return PB_ERR_UNSUPPORTED;
  const int64_t M = a->shape[0], K = a->shape[1], N = b->shape[1];
  // measured in CUDA graphs (tools/mm_table.py): the operand pre-pass pays off once M >= 256;
  // for the b128 classifier GEMMs (M = 128, multi-MB weights) gemm_tc.cu's in-GEMM split wins
  static const int64_t min_m = getenv("PB_TMA_MM_MIN_M") ? atoll(getenv("PB_TMA_MM_MIN_M")) : 256;  // experiment hook
  if (M < min_m || N < 64 || K < 64 || !fits(M * N) || !fits(M * K) || !fits(N * K)) return PB_ERR_UNSUPPORTED;
  const int64_t kp = (K + 3) / 4 * 4;
  const int BN = M <= 64 ? 64 : 128;
  Prob pr{};
  pr.plain = 1;
  pr.Mi = (int)N;
  pr.Nj = (int)M;
  pr.K = (int)kp;
  pr.C = (int)kp;
  pr.KH = pr.KW = pr.SH = pr.SW = 1;
  const int64_t tiles = ((N + BM - 1) / BM) * ((M + BN - 1) / BN);
  const int64_t kblocks = (kp + BK - 1) / BK;
  int splits = 1;
  if (tiles < num_sms()) {
    splits = (int)(num_sms() / tiles);
    if (splits > kblocks / 4) splits = (int)(kblocks / 4);
    if (splits < 1) splits = 1;
  }
  int per = (int)((kblocks + splits - 1) / splits) * BK;
  splits = (int)((kp + per - 1) / per);
  pr.kper = per;
  pr.zdim = splits;
  const size_t nb = ((size_t)N * kp * 4 + 1023) / 1024 * 1024, mb = ((size_t)M * kp * 4 + 1023) / 1024 * 1024;
  const size_t part = splits > 1 ? (size_t)splits * M * N * 4 : 0;
  char* ws = (char*)workspace(2 * nb + 2 * mb + part);
  if (!ws) return fail(PB_ERR_OOM, "matmul (tma): no workspace");
  float *nh = (float*)ws, *nl = (float*)(ws + nb), *mh = (float*)(ws + 2 * nb), *ml = (float*)(ws + 2 * nb + mb);
  float* pw = (float*)(ws + 2 * nb + 2 * mb);
  cudaStream_t s = compute_stream();
  // rows n of D: B^T, v(n, k) = B[k][n]; rows m: v(m, k) = A[m][k]
  kmajor_split<<<dim3((unsigned)((kp + 31) / 32), (unsigned)((N + 31) / 32)), 256, 0, s>>>(
      (const float*)(uintptr_t)b->ptr, nh, nl, (int)N, (int)K, (int)kp, b->strides[1], b->strides[0]);
  PB_LAUNCHED();
  kmajor_split<<<dim3((unsigned)((kp + 31) / 32), (unsigned)((M + 31) / 32)), 256, 0, s>>>(
      (const float*)(uintptr_t)a->ptr, mh, ml, (int)M, (int)K, (int)kp, a->strides[0], a->strides[1]);
  PB_LAUNCHED();
  CUtensorMap ah, al, bh, bl;
  if (!map_2d(&ah, nh, kp, N, BM) || !map_2d(&al, nl, kp, N, BM) || !map_2d(&bh, mh, kp, M, BN) ||
      !map_2d(&bl, ml, kp, M, BN))
    return fail(PB_ERR_CUDA, "matmul (tma): tensor map encoding failed");
  float* c = (float*)(uintptr_t)out->ptr;
  if (splits == 1) {
    OutMat o{c, (int)N, (int)M, N, 0};
    return BN == 64 ? launch<64, false>(ah, al, bh, bl, pr, o) : launch<128, false>(ah, al, bh, bl, pr, o);
  }
  OutPartial op{pw, (int)N, (int)M};
  int rc = BN == 64 ? launch<64, false>(ah, al, bh, bl, pr, op) : launch<128, false>(ah, al, bh, bl, pr, op);
  if (rc) return rc;
  OutMat fin{c, (int)N, (int)M, N, 0};
  launch_fold<OutMat>(pw, splits, (int)N, (int)M, fin, s);
  PB_LAUNCHED();
  return PB_OK;
}

}  // extern "C"

// tcgen05 / TMEM 3xTF32 contraction kernels for sm_100a: matmul (rank-2 and batched
// rank-3) and conv2d fprop / dgrad / wgrad as implicit GEMMs (minml/kernels.py:166-239).
//
// Why 3xTF32: the reference contracts f32 operands in f64 and rounds once
// (kernels.py:168-169, :176-179); one TF32 pass is ~1e-3 off, which breaks the 1e-5
// parity bar.  Each f32 operand x is split on the fly into
// hi = rna_tf32(x) and lo = rna_tf32(x - hi) (x - hi is exact in f32, |lo| <= 2^-11 |x|),
// and D += Alo*Bhi + Ahi*Blo + Ahi*Bhi: per-product error <= ~2^-22, unbiased.
//
// Accumulation: the tensor core aligns each MMA's products to its f32 accumulator and
// truncates, so (a) the tiny lo-products lose bits against a large accumulator and (b) a
// long K chain (wgrad: K = N*Ho*Wo = 100352 at ResNet-50 b32) drifts with the chain length.
// Hence the lo-products accumulate in their own TMEM accumulator ("small", ~2^-11 of the
// "big" hi*hi one), and the MMA accumulates only `ck` k-blocks (64 k by default) into one
// of two TMEM buffer pairs; dedicated drain warps tcgen05.ld each finished chunk and add
// big + small into f32 registers with IEEE round-to-nearest while the MMA fills the other
// pair.
//
// One CTA computes a 128 x BN tile of D[i][j] = sum_k A(i,k) B(j,k):
//   * warps 0..7 (producers): gather A/B elements through an operand "loader" (the
//     implicit im2col of the conv, or a strided matmul operand), split hi/lo and store
//     them K-major into 128B-swizzled shared memory (the UMMA canonical SW128 layout), a
//     STAGES-deep ring guarded by mbarriers (full: producers -> MMA, empty: tcgen05.commit
//     -> producers);
//   * warp 8 (MMA): allocates 2*BN TMEM columns, one thread issues 3 x tcgen05.mma.kind::tf32
//     (M=128, N=BN, K=8) per 8-wide K step, and commits each stage back to the producers
//     and each chunk to the drain warps;
//   * warps 9.. (BN/16 drain warps): tcgen05.ld 32x32b rows of each finished chunk, sum in
//     registers, and finally store through the output functor.  Rows (TMEM lanes) are
//     always the unit-stride dimension of the output, so a warp's per-column stores are
//     coalesced.
// Small-tile / long-K problems (wgrad, matmul-backward) split K over blockIdx.z into a
// workspace of f32 partials folded in split order (deterministic).
#include <cuda_runtime.h>
#include <stdint.h>
#include "common.cuh"
#include "tc_common.cuh"

namespace pb {
namespace tc {

constexpr int BM = 128;        // D rows per CTA = TMEM lanes = MMA M
constexpr int BK = 32;         // f32 per 128-byte swizzled row
static int g_ck = 2;           // k-blocks accumulated in TMEM before a register drain
constexpr int SMEM_BUDGET = 200 * 1024;

__device__ __forceinline__ float ldg(const float* p) { return __ldg(p); }

// =========================================================================================
// Operand loaders.  A loader describes a logical [rows x K] f32 operand and one of two
// thread mappings (fixed per thread for the whole kernel):
//   row mode (KMODE = false): a thread owns ONE row of the 128/BN-row tile and several
//     4-wide k chunks; lanes of a warp walk consecutive rows (rows are unit-stride in HBM).
//       Row row(b, r);  KB kb(const Row&, k0, kend);  float4 get4(const KB&, chunk)
//   k mode (KMODE = true): a thread owns ONE chunk (k0 + 4*(tid&7) .. +3) of several rows;
//     8 lanes cover a 128-byte row (k is unit-stride in HBM).
//       Row row(b, r);  KB kb(chunk, k0, kend);      float4 get4(const Row&, const KB&)
// KB is the per-(thread, k-block) context, so the index arithmetic that depends only on k
// (im2col decomposition, bounds) is done once per k-block, not once per element.
// Elements at or beyond kend, or outside the operand, read as 0.
// =========================================================================================

// strided rank-3 matrix view X[b][r][k] (matmul operands, any strides)
template <bool KM, bool VEC>
struct MatLoader {
  static constexpr bool KMODE = KM;
  const float* p;
  int64_t sb, sr, sk;
  int R;
  struct Row {
    const float* p;
  };
  __device__ __forceinline__ Row row(int b, int r) const {
    Row o;
    o.p = r < R ? p + (int64_t)b * sb + (int64_t)r * sr : nullptr;
    return o;
  }
  // row mode
  struct KBR {
    const float* q;
    int n;  // valid k in this k-block
  };
  __device__ __forceinline__ KBR kb(const Row& rw, int k0, int kend) const {
    KBR o;
    o.q = rw.p ? rw.p + (int64_t)k0 * sk : nullptr;
    o.n = kend - k0;
    return o;
  }
  __device__ __forceinline__ float4 get4(const KBR& c, int chunk) const {
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (!c.q) return v;
    const int k = chunk * 4;
    const float* q = c.q + (int64_t)k * sk;
    if (k < c.n) v.x = ldg(q);
    if (k + 1 < c.n) v.y = ldg(q + sk);
    if (k + 2 < c.n) v.z = ldg(q + 2 * sk);
    if (k + 3 < c.n) v.w = ldg(q + 3 * sk);
    return v;
  }
  // k mode
  struct KBK {
    int k, n;  // first k of the chunk, valid count (<= 4)
  };
  __device__ __forceinline__ KBK kb(int chunk, int k0, int kend) const {
    KBK o;
    o.k = k0 + chunk * 4;
    o.n = kend - o.k;
    return o;
  }
  __device__ __forceinline__ float4 get4(const Row& rw, const KBK& c) const {
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (!rw.p || c.n <= 0) return v;
    if (VEC && c.n >= 4) return __ldg(reinterpret_cast<const float4*>(rw.p + c.k));
    const float* q = rw.p + (int64_t)c.k * sk;
    v.x = ldg(q);
    if (c.n > 1) v.y = ldg(q + sk);
    if (c.n > 2) v.z = ldg(q + 2 * sk);
    if (c.n > 3) v.w = ldg(q + 3 * sk);
    return v;
  }
};

struct Geo {
  int N, C, H, W, F, KH, KW, SH, SW, PH, PW, HO, WO;
};

// fprop A(i = (n,ho,wo), k = (r,s,c)) = x[n, c, ho*sh-ph+r, wo*sw-pw+s]   (row mode)
// FAST: C % 32 == 0, so a k-block has one (r, s) and 32 consecutive channels
template <bool FAST>
struct FpropX {
  static constexpr bool KMODE = false;
  const float* x;
  Geo g;
  FastDiv fC, fKW, fP, fWO;
  int rows;  // N*HO*WO
  struct Row {
    const float* p;  // x + n*C*H*W, nullptr when out of range
    int ih0, iw0;
  };
  __device__ __forceinline__ Row row(int, int i) const {
    Row o;
    o.p = nullptr;
    o.ih0 = o.iw0 = 0;
    if (i < rows) {
      uint32_t n, pix, ho, wo;
      fP.divmod(i, n, pix);
      fWO.divmod(pix, ho, wo);
      o.p = x + (int64_t)n * g.C * g.H * g.W;
      o.ih0 = (int)ho * g.SH - g.PH;
      o.iw0 = (int)wo * g.SW - g.PW;
    }
    return o;
  }
  struct KBR {
    const float* q;  // FAST: &x[n, c0, ih, iw] or nullptr (padding / out of range)
    Row rw;          // generic path
    int k0, kend;
  };
  __device__ __forceinline__ KBR kb(const Row& rw, int k0, int kend) const {
    KBR o;
    o.rw = rw;
    o.k0 = k0;
    o.kend = kend;
    o.q = nullptr;
    if (FAST && rw.p) {
      uint32_t rs, c0, r, s;
      fC.divmod(k0, rs, c0);
      fKW.divmod(rs, r, s);
      int ih = rw.ih0 + (int)r, iw = rw.iw0 + (int)s;
      if ((unsigned)ih < (unsigned)g.H && (unsigned)iw < (unsigned)g.W)
        o.q = rw.p + ((int64_t)c0 * g.H + ih) * g.W + iw;
    }
    return o;
  }
  __device__ __forceinline__ float one(const Row& rw, int k) const {
    uint32_t rs, c, r, s;
    fC.divmod(k, rs, c);
    fKW.divmod(rs, r, s);
    int ih = rw.ih0 + (int)r, iw = rw.iw0 + (int)s;
    if ((unsigned)ih >= (unsigned)g.H || (unsigned)iw >= (unsigned)g.W) return 0.f;
    return ldg(rw.p + ((int64_t)c * g.H + ih) * g.W + iw);
  }
  __device__ __forceinline__ float4 get4(const KBR& c, int chunk) const {
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (FAST) {
      if (!c.q) return v;
      const int64_t hw = (int64_t)g.H * g.W;
      const float* q = c.q + (int64_t)(chunk * 4) * hw;
      v.x = ldg(q);
      v.y = ldg(q + hw);
      v.z = ldg(q + 2 * hw);
      v.w = ldg(q + 3 * hw);
      return v;
    }
    if (!c.rw.p) return v;
    const int k = c.k0 + chunk * 4;
    if (k < c.kend) v.x = one(c.rw, k);
    if (k + 1 < c.kend) v.y = one(c.rw, k + 1);
    if (k + 2 < c.kend) v.z = one(c.rw, k + 2);
    if (k + 3 < c.kend) v.w = one(c.rw, k + 3);
    return v;
  }
};

// dgrad A(i = (n,h,w), k = (r,s,f)) = g[n, f, (h+ph-r)/sh, (w+pw-s)/sw] when on the stride
// grid and in range, else 0.                                              (row mode)
// FAST: F % 32 == 0, so a k-block has one (r, s) and 32 consecutive filters
template <bool FAST>
struct DgradG {
  static constexpr bool KMODE = false;
  const float* gr;
  Geo g;
  FastDiv fF, fKW, fHW, fW, fSH, fSW;
  int rows;  // N*H*W
  struct Row {
    const float* p;  // g + n*F*HO*WO
    int hp, wp;      // h + ph, w + pw
  };
  __device__ __forceinline__ Row row(int, int i) const {
    Row o;
    o.p = nullptr;
    o.hp = o.wp = 0;
    if (i < rows) {
      uint32_t n, pix, h, w;
      fHW.divmod(i, n, pix);
      fW.divmod(pix, h, w);
      o.p = gr + (int64_t)n * g.F * g.HO * g.WO;
      o.hp = (int)h + g.PH;
      o.wp = (int)w + g.PW;
    }
    return o;
  }
  // &g[n, f, ho, wo] for k = (r,s,f), or nullptr off the stride grid / out of range
  __device__ __forceinline__ const float* at(const Row& rw, int k, uint32_t* f_out) const {
    uint32_t rs, f, r, s;
    fF.divmod(k, rs, f);
    fKW.divmod(rs, r, s);
    *f_out = f;
    int hh = rw.hp - (int)r, ww = rw.wp - (int)s;
    if (hh < 0 || ww < 0) return nullptr;
    uint32_t ho, wo, rh, rw_;
    fSH.divmod(hh, ho, rh);
    fSW.divmod(ww, wo, rw_);
    if (rh | rw_ || ho >= (uint32_t)g.HO || wo >= (uint32_t)g.WO) return nullptr;
    return rw.p + ((int64_t)f * g.HO + ho) * g.WO + wo;
  }
  struct KBR {
    const float* q;  // FAST: &g[n, f0, ho, wo] or nullptr
    Row rw;
    int k0, kend;
  };
  __device__ __forceinline__ KBR kb(const Row& rw, int k0, int kend) const {
    KBR o;
    o.rw = rw;
    o.k0 = k0;
    o.kend = kend;
    o.q = nullptr;
    if (FAST && rw.p) {
      uint32_t f;
      o.q = at(rw, k0, &f);
    }
    return o;
  }
  __device__ __forceinline__ float4 get4(const KBR& c, int chunk) const {
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    const int64_t P = (int64_t)g.HO * g.WO;
    if (FAST) {
      if (!c.q) return v;
      const float* q = c.q + (int64_t)(chunk * 4) * P;
      v.x = ldg(q);
      v.y = ldg(q + P);
      v.z = ldg(q + 2 * P);
      v.w = ldg(q + 3 * P);
      return v;
    }
    if (!c.rw.p) return v;
    float e[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int k = c.k0 + chunk * 4 + t;
      uint32_t f;
      const float* q = k < c.kend ? at(c.rw, k, &f) : nullptr;
      if (q) e[t] = ldg(q);
    }
    return make_float4(e[0], e[1], e[2], e[3]);
  }
};

// wgrad A(i = (c,r,s), k = (n,ho,wo)) = x[n, c, ho*sh-ph+r, wo*sw-pw+s]       (k mode)
struct WgradX {
  static constexpr bool KMODE = true;
  const float* x;
  Geo g;
  FastDiv fP, fWO, fRS, fKW;
  int rows;  // C*KH*KW
  struct Row {
    const float* p;  // x + c*H*W + (r-ph)*W + (s-pw)  (may point before the row: only used when in range)
    int dr, ds;      // r - ph, s - pw; p == nullptr when out of range
  };
  __device__ __forceinline__ Row row(int, int i) const {
    Row o;
    o.p = nullptr;
    o.dr = o.ds = 0;
    if (i < rows) {
      uint32_t c, rs, r, s;
      fRS.divmod(i, c, rs);
      fKW.divmod(rs, r, s);
      o.dr = (int)r - g.PH;
      o.ds = (int)s - g.PW;
      o.p = x + (int64_t)c * g.H * g.W + (int64_t)o.dr * g.W + o.ds;
    }
    return o;
  }
  struct KBK {
    int off[4];     // n*C*H*W + (ho*sh)*W + wo*sw, per element
    int hs[4], ws[4];  // ho*sh, wo*sw; hs = -2^30 marks k >= kend
  };
  __device__ __forceinline__ KBK kb(int chunk, int k0, int kend) const {
    KBK o;
    const int k = k0 + chunk * 4;
    uint32_t n, pix, ho, wo;
    fP.divmod(k < kend ? k : 0, n, pix);
    fWO.divmod(pix, ho, wo);
    const int chw = g.C * g.H * g.W;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const bool ok = k + t < kend;
      o.hs[t] = ok ? (int)ho * g.SH : -(1 << 30);
      o.ws[t] = (int)wo * g.SW;
      o.off[t] = ok ? (int)n * chw + o.hs[t] * g.W + o.ws[t] : 0;
      if (++wo == (uint32_t)g.WO) {
        wo = 0;
        if (++ho == (uint32_t)g.HO) {
          ho = 0;
          ++n;
        }
      }
    }
    return o;
  }
  __device__ __forceinline__ float4 get4(const Row& rw, const KBK& c) const {
    float e[4] = {0.f, 0.f, 0.f, 0.f};
    if (!rw.p) return make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      if ((unsigned)(c.hs[t] + rw.dr) < (unsigned)g.H && (unsigned)(c.ws[t] + rw.ds) < (unsigned)g.W)
        e[t] = ldg(rw.p + c.off[t]);
    }
    return make_float4(e[0], e[1], e[2], e[3]);
  }
};

// wgrad B(j = f, k = (n,p)) = g[n, f, p]                                        (k mode)
struct WgradG {
  static constexpr bool KMODE = true;
  const float* gr;
  Geo g;
  FastDiv fP;
  int rows;  // F
  bool vec;  // P % 4 == 0: a chunk never straddles images, 16B aligned
  struct Row {
    const float* p;  // g + f*P
  };
  __device__ __forceinline__ Row row(int, int f) const {
    Row o;
    o.p = f < rows ? gr + (int64_t)f * g.HO * g.WO : nullptr;
    return o;
  }
  struct KBK {
    int off[4];  // n*F*P + pix per element, -1 when k >= kend
  };
  __device__ __forceinline__ KBK kb(int chunk, int k0, int kend) const {
    KBK o;
    const int k = k0 + chunk * 4;
    uint32_t n, pix;
    fP.divmod(k < kend ? k : 0, n, pix);
    const int fp = g.F * (int)fP.d;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      o.off[t] = k + t < kend ? (int)n * fp + (int)pix : -1;
      if (++pix == fP.d) {
        pix = 0;
        ++n;
      }
    }
    return o;
  }
  __device__ __forceinline__ float4 get4(const Row& rw, const KBK& c) const {
    if (!rw.p) return make_float4(0.f, 0.f, 0.f, 0.f);
    if (vec && c.off[3] >= 0) return __ldg(reinterpret_cast<const float4*>(rw.p + c.off[0]));
    float e[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) e[t] = c.off[t] >= 0 ? ldg(rw.p + c.off[t]) : 0.f;
    return make_float4(e[0], e[1], e[2], e[3]);
  }
};

template <int BN>
struct Cfg {
  static constexpr int A_BYTES = BM * 128;
  static constexpr int B_BYTES = BN * 128;
  static constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
  static constexpr int STAGES = (SMEM_BUDGET - 1024 - 256) / STAGE_BYTES > 6 ? 6 : (SMEM_BUDGET - 1024 - 256) / STAGE_BYTES;
  static constexpr int SMEM = 1024 + STAGES * STAGE_BYTES + 256;  // + 1024 alignment slack + barriers
  // 13 warps either way (416 threads, <= 152 registers each): BN=64 has 8 producer and 4
  // drain warps, BN=128 4 producer and 8 drain warps; every drain thread holds 64 columns
  static constexpr int NDRAIN = BN / 16;
  static constexpr int NPROD = (12 - NDRAIN) * 32;
  static constexpr int MMA_WARP = NPROD / 32;
  static constexpr int A_TASKS = BM * 8 / NPROD;
  static constexpr int B_TASKS = BN * 8 / NPROD;
  static constexpr uint32_t IDESC = idesc_tf32(BM, BN);
  static constexpr int THREADS = NPROD + 32 + NDRAIN * 32;
  static constexpr int TMEM_COLS = 4 * BN;  // 2 buffers x {big, small}
};

// rows/chunk of task t for a tile with `rows` rows
template <bool KMODE, int ROWS>
__device__ __forceinline__ void task_pos(int t, int& row, int& chunk) {
  if (KMODE) {
    row = t >> 3;
    chunk = t & 7;
  } else {
    row = t % ROWS;
    chunk = t / ROWS;
  }
}

// D[i][j] over k in [kbeg, kend) for i in the 128-row tile blockIdx.x, j in tile blockIdx.y,
// batch/split blockIdx.z
template <int BN, class LA, class LB, class OUT>
__global__ void __launch_bounds__(Cfg<BN>::THREADS, 1)
    tc_gemm_kernel(LA la, LB lb, OUT out, int K, int kper, int batched, int CK, int tiles_i, int tiles_j,
                   int ntiles) {
  // Persistent: CTA b walks tiles b, b + gridDim.x, ... of the (z, i-tile, j-tile) space
  // (j fastest, so concurrently running CTAs share their A rows through L2).  Stage and
  // TMEM-chunk counters run on across tiles, so the producers and the MMA start the next
  // tile while the drain warps are still storing the previous one.
  typedef Cfg<BN> C;
  extern __shared__ uint8_t smem_raw[];
  char* smem = (char*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* empty = full + C::STAGES;
  uint64_t* accf = empty + C::STAGES;  // chunk accumulated (MMA -> drain), per TMEM buffer
  uint64_t* acce = accf + 2;           // chunk drained (drain -> MMA)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acce + 2);

  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int per_z = tiles_i * tiles_j;

  if (tid == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], C::NPROD);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&accf[s], 1);
      mbar_init(&acce[s], C::NDRAIN * 32);
    }
    fence_barrier_init();
  }
  if (warp == C::MMA_WARP) tmem_alloc<C::TMEM_COLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == C::MMA_WARP) {
    // ===== MMA issuer =====
    if ((tid & 31) == 0) {
      uint32_t it = 0, cc = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int z = t / per_z;
        const int kbeg = batched ? 0 : z * kper;
        const int kend = min(K, kbeg + kper);
        const int nkb = kend > kbeg ? (kend - kbeg + BK - 1) / BK : 0;
        uint32_t dbig = 0, dsmall = 0;
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % C::STAGES;
          const bool first = (kb % CK) == 0;
          if (first) {
            const uint32_t buf = cc & 1;
            if (cc >= 2) {
              mbar_wait(&acce[buf], ((cc >> 1) - 1) & 1);
              tc_fence_after();
            }
            dbig = tmem + buf * 2 * BN;
            dsmall = dbig + BN;
          }
          mbar_wait(&full[s], (it / C::STAGES) & 1);
          tc_fence_after();
          uint32_t base = smem_u32(smem + s * C::STAGE_BYTES);
          uint64_t ahi = sw128_desc(base), alo = sw128_desc(base + C::A_BYTES);
          uint64_t bhi = sw128_desc(base + 2 * C::A_BYTES), blo = sw128_desc(base + 2 * C::A_BYTES + C::B_BYTES);
#pragma unroll
          for (int kk = 0; kk < BK / 8; ++kk) {
            uint64_t adv = (uint64_t)(kk * 32) >> 4;  // 8 tf32 = 32 bytes along the swizzled row
            const uint32_t acc = !(first && kk == 0);
            mma_tf32(dsmall, alo + adv, bhi + adv, C::IDESC, acc);
            mma_tf32(dsmall, ahi + adv, blo + adv, C::IDESC, 1);
            mma_tf32(dbig, ahi + adv, bhi + adv, C::IDESC, acc);
          }
          mma_commit(&empty[s]);
          if ((kb % CK) == CK - 1 || kb == nkb - 1) {
            mma_commit(&accf[cc & 1]);
            ++cc;
          }
        }
      }
    }
    __syncwarp();
  } else if (warp < C::MMA_WARP) {
    // ===== producers =====
    // row-mode operands: this thread owns one row (NPROD is a multiple of the tile rows)
    // and chunks t*NPROD/ROWS + ...; k-mode operands: one chunk (tid & 7) of rows tid/8 + ...
    int ach[C::A_TASKS], aro[C::A_TASKS], bch[C::B_TASKS], bro[C::B_TASKS];
    uint32_t aoff[C::A_TASKS], boff[C::B_TASKS];
#pragma unroll
    for (int t = 0; t < C::A_TASKS; ++t) {
      task_pos<LA::KMODE, BM>(tid + t * C::NPROD, aro[t], ach[t]);
      aoff[t] = swz(aro[t], ach[t]);
    }
#pragma unroll
    for (int t = 0; t < C::B_TASKS; ++t) {
      task_pos<LB::KMODE, BN>(tid + t * C::NPROD, bro[t], bch[t]);
      boff[t] = swz(bro[t], bch[t]);
    }
    uint32_t it = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const int z = tile / per_z, rem = tile - z * per_z;
      const int i0 = (rem / tiles_j) * BM, j0 = (rem % tiles_j) * BN;
      const int b = batched ? z : 0;
      const int kbeg = batched ? 0 : z * kper;
      const int kend = min(K, kbeg + kper);
      const int nkb = kend > kbeg ? (kend - kbeg + BK - 1) / BK : 0;
      constexpr int NAR = LA::KMODE ? C::A_TASKS : 1, NBR = LB::KMODE ? C::B_TASKS : 1;
      typename LA::Row ar[NAR];
      typename LB::Row br[NBR];
#pragma unroll
      for (int t = 0; t < NAR; ++t) ar[t] = la.row(b, i0 + aro[t]);
#pragma unroll
      for (int t = 0; t < NBR; ++t) br[t] = lb.row(b, j0 + bro[t]);
      float4 av[C::A_TASKS], bv[C::B_TASKS];
      auto gather = [&](int k0) {
        if constexpr (LA::KMODE) {
          const auto ctx = la.kb(ach[0], k0, kend);
#pragma unroll
          for (int t = 0; t < C::A_TASKS; ++t) av[t] = la.get4(ar[t], ctx);
        } else {
          const auto ctx = la.kb(ar[0], k0, kend);
#pragma unroll
          for (int t = 0; t < C::A_TASKS; ++t) av[t] = la.get4(ctx, ach[t]);
        }
        if constexpr (LB::KMODE) {
          const auto ctx = lb.kb(bch[0], k0, kend);
#pragma unroll
          for (int t = 0; t < C::B_TASKS; ++t) bv[t] = lb.get4(br[t], ctx);
        } else {
          const auto ctx = lb.kb(br[0], k0, kend);
#pragma unroll
          for (int t = 0; t < C::B_TASKS; ++t) bv[t] = lb.get4(ctx, bch[t]);
        }
      };
      // software-pipelined: the gathers for k-block kb+1 are in flight while this thread
      // waits for a free stage and stores k-block kb
      if (nkb > 0) gather(kbeg);
      for (int kb = 0; kb < nkb; ++kb, ++it) {
        const int s = it % C::STAGES;
        if (it >= (uint32_t)C::STAGES) mbar_wait(&empty[s], ((it / C::STAGES) - 1) & 1);
        char* st = smem + s * C::STAGE_BYTES;
#pragma unroll
        for (int t = 0; t < C::A_TASKS; ++t) split_store(st, st + C::A_BYTES, aoff[t], av[t]);
#pragma unroll
        for (int t = 0; t < C::B_TASKS; ++t)
          split_store(st + 2 * C::A_BYTES, st + 2 * C::A_BYTES + C::B_BYTES, boff[t], bv[t]);
        fence_proxy_async();
        mbar_arrive(&full[s]);
        if (kb + 1 < nkb) gather(kbeg + (kb + 1) * BK);
      }
    }
  } else {
    // ===== drain + epilogue: TMEM lane quadrant is fixed by warp % 4 =====
    const int q = warp & 3, cg = (warp - C::MMA_WARP - 1) >> 2;
    const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(cg * 64);
    uint32_t cc = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const int z = tile / per_z, rem = tile - z * per_z;
      const int i0 = (rem / tiles_j) * BM, j0 = (rem % tiles_j) * BN;
      const int kbeg = batched ? 0 : z * kper;
      const int kend = min(K, kbeg + kper);
      const int nkb = kend > kbeg ? (kend - kbeg + BK - 1) / BK : 0;
      float acc[64];
#pragma unroll
      for (int e = 0; e < 64; ++e) acc[e] = 0.f;
      const int nch = (nkb + CK - 1) / CK;
      for (int c = 0; c < nch; ++c, ++cc) {
        const uint32_t buf = cc & 1;
        mbar_wait(&accf[buf], (cc >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          uint32_t rb[16], rs[16];
          tmem_ld16(lane_base + buf * 2 * BN + (uint32_t)(p * 16), rb);
          tmem_ld16(lane_base + buf * 2 * BN + BN + (uint32_t)(p * 16), rs);
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < 16; ++e)
            acc[p * 16 + e] = __fadd_rn(acc[p * 16 + e], __fadd_rn(__uint_as_float(rb[e]), __uint_as_float(rs[e])));
        }
        tc_fence_before();
        mbar_arrive(&acce[buf]);
      }
      const int i = i0 + q * 32 + (tid & 31);
      typename OUT::Row orow = out.row(z, i);
#pragma unroll
      for (int e = 0; e < 64; ++e) out.put(orow, j0 + cg * 64 + e, acc[e]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == C::MMA_WARP) {
    tc_fence_after();
    tmem_dealloc<C::TMEM_COLS>(tmem);
  }
}

// weight re-layout: dst[a][(r*KW+s)*Bn + bb] = w[f][c][r][s] with (a,bb) = (f,c) (fprop,
// k = (r,s,c)) or (c,f) (dgrad, k = (r,s,f))
__global__ void weight_rsk(const float* w, float* dst, int F, int Cc, int RS, int dgrad) {
  const uint32_t n = (uint32_t)F * Cc * RS;  // weights: far below 2^31 elements (checked on the host)
  for (uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x; idx < n; idx += gridDim.x * blockDim.x) {
    int rs = (int)(idx % (uint32_t)RS);
    uint32_t t = idx / (uint32_t)RS;
    int c = (int)(t % (uint32_t)Cc);
    int f = (int)(t / (uint32_t)Cc);
    float v = w[idx];
    if (!dgrad)
      dst[((int64_t)f * RS + rs) * Cc + c] = v;
    else
      dst[((int64_t)c * RS + rs) * F + f] = v;
  }
}

// ---- host side --------------------------------------------------------------------------
template <int BN, class LA, class LB, class OUT>
static int launch(const LA& la, const LB& lb, const OUT& out, int Mi, int Nj, int K, int zdim, int kper,
                  int batched) {
  typedef Cfg<BN> C;
  static bool attr = false;
  if (!attr) {
    PB_CUDA(cudaFuncSetAttribute(tc_gemm_kernel<BN, LA, LB, OUT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 C::SMEM));
    attr = true;
  }
  const int ti = (Mi + BM - 1) / BM, tj = (Nj + BN - 1) / BN;
  const int64_t ntiles = (int64_t)ti * tj * zdim;
  if (ntiles >= ((int64_t)1 << 31)) return fail(PB_ERR_UNSUPPORTED, "tc_gemm: too many tiles");
  const int grid = (int)(ntiles < num_sms() ? ntiles : num_sms());
  tc_gemm_kernel<BN, LA, LB, OUT><<<grid, C::THREADS, C::SMEM, compute_stream()>>>(la, lb, out, K, kper, batched,
                                                                                  g_ck, ti, tj, (int)ntiles);
  PB_LAUNCHED();
  return PB_OK;
}

static int g_bn_max = 128;  // widest N tile the dispatcher may pick (experiment hook)
static int pick_bn(int Nj) { return Nj <= 64 || g_bn_max <= 64 ? 64 : 128; }

// number of K splits so that tiles * splits covers the machine; kper a multiple of BK
static int pick_splits(int64_t tiles, int K, int* kper) {
  int splits = 1;
  int64_t want = num_sms();
  if (tiles < want && K >= 8 * BK) {
    splits = (int)(want / tiles);  // whole waves
    int maxs = K / (4 * BK);
    if (splits > maxs) splits = maxs;
    if (splits < 1) splits = 1;
  }
  int per = (K + splits - 1) / splits;
  per = (per + BK - 1) / BK * BK;
  splits = (K + per - 1) / per;
  *kper = per;
  return splits;
}

// run D = A B^T (Mi x Nj over K) into OUT, split-K through the workspace when it helps
template <int BN, class LA, class LB, class OUT>
static int run(const LA& la, const LB& lb, const OUT& out, int Mi, int Nj, int K, int batch, float* ws_after) {
  if (batch > 1) return launch<BN>(la, lb, out, Mi, Nj, K, batch, K, 1);
  int64_t tiles = (int64_t)((Mi + BM - 1) / BM) * ((Nj + BN - 1) / BN);
  int kper;
  int splits = pick_splits(tiles, K, &kper);
  if (splits == 1) return launch<BN>(la, lb, out, Mi, Nj, K, 1, K, 0);
  OutPartial part{ws_after, Mi, Nj};
  int rc = launch<BN>(la, lb, part, Mi, Nj, K, splits, kper, 0);
  if (rc) return rc;
  launch_fold<OUT>(ws_after, splits, Mi, Nj, out, compute_stream());
  PB_LAUNCHED();
  return PB_OK;
}

template <class LA, class LB, class OUT>
static int run_bn(const LA& la, const LB& lb, const OUT& out, int Mi, int Nj, int K, int batch, float* ws) {
  if (pick_bn(Nj) == 64) return run<64>(la, lb, out, Mi, Nj, K, batch, ws);
  return run<128>(la, lb, out, Mi, Nj, K, batch, ws);
}

static size_t split_ws_bytes(int Mi, int Nj) {
  // worst case splits <= num_sms
  return (size_t)num_sms() * Mi * Nj * sizeof(float);
}

static Geo geo(const int64_t* xs, const int64_t* ws, const pb_conv* p) {
  Geo g;
  g.N = (int)xs[0];
  g.C = (int)xs[1];
  g.H = (int)xs[2];
  g.W = (int)xs[3];
  g.F = (int)ws[0];
  g.KH = (int)ws[2];
  g.KW = (int)ws[3];
  g.SH = p->stride_h;
  g.SW = p->stride_w;
  g.PH = p->pad_h;
  g.PW = p->pad_w;
  g.HO = (g.H + 2 * g.PH - g.KH) / g.SH + 1;
  g.WO = (g.W + 2 * g.PW - g.KW) / g.SW + 1;
  return g;
}

static bool f32_all(const pb_tensor* a, const pb_tensor* b, const pb_tensor* o) {
  return a->dtype == PB_F32 && b->dtype == PB_F32 && o->dtype == PB_F32;
}
static bool fits_i32(int64_t v) { return v < ((int64_t)1 << 31) - 64; }

}  // namespace tc
}  // namespace pb

using namespace pb;
using namespace pb::tc;

extern "C" {

// experiment hook (not part of the public ABI): k-blocks per TMEM accumulation chunk
int pb_tc_set_chunk(int ck) {
  if (ck < 1) return PB_ERR_ARG;
  g_ck = ck;
  return PB_OK;
}
int pb_tc_set_bn_max(int bn) {
  g_bn_max = bn;
  return PB_OK;
}

int pb_matmul_tc(const pb_tensor* a, const pb_tensor* b, const pb_tensor* out) {
  if (!f32_all(a, b, out)) return PB_ERR_UNSUPPORTED;
  int r3 = a->ndim == 3;
  int batch = r3 ? (int)a->shape[0] : 1;
  int64_t M = a->shape[r3], K = a->shape[r3 + 1], N = b->shape[r3 + 1];
  if (M * N * batch == 0 || K == 0) return PB_ERR_UNSUPPORTED;  // SIMT handles the trivial cases
  if (!fits_i32(M * N) || !fits_i32(K) || !fits_i32(M) || !fits_i32(N)) return PB_ERR_UNSUPPORTED;
  // D[i = n][j = m] = sum_k B[k][n] A[m][k]: rows of D are output columns (unit stride)
  int64_t bsb = r3 ? b->strides[0] : 0, bsk = b->strides[r3], bsn = b->strides[r3 + 1];
  int64_t asb = r3 ? a->strides[0] : 0, asm_ = a->strides[r3], ask = a->strides[r3 + 1];
  const float* pa = (const float*)(uintptr_t)a->ptr;
  const float* pbp = (const float*)(uintptr_t)b->ptr;
  OutMat o{(float*)(uintptr_t)out->ptr, (int)N, (int)M, N, M * N};
  float* ws = nullptr;
  if (batch == 1) {
    ws = (float*)workspace(split_ws_bytes((int)N, (int)M));
    if (!ws) return fail(PB_ERR_OOM, "matmul: no workspace");
  }
  // A-operand (rows n): n-stride 1 -> row-mode; else k-mode over B's k-stride
  // B-operand (rows m): k-stride 1 -> k-mode vectorised when 16B aligned
  bool avec = ask == 1 && (K % 4 == 0) && (asm_ % 4 == 0) && (asb % 4 == 0) && (a->ptr % 16 == 0);
  if (bsn == 1) {
    MatLoader<false, false> la{pbp, bsb, bsn, bsk, (int)N};
    if (ask == 1) {
      if (avec) return run_bn(la, MatLoader<true, true>{pa, asb, asm_, ask, (int)M}, o, (int)N, (int)M, (int)K, batch, ws);
      return run_bn(la, MatLoader<true, false>{pa, asb, asm_, ask, (int)M}, o, (int)N, (int)M, (int)K, batch, ws);
    }
    return run_bn(la, MatLoader<false, false>{pa, asb, asm_, ask, (int)M}, o, (int)N, (int)M, (int)K, batch, ws);
  }
  MatLoader<true, false> la{pbp, bsb, bsn, bsk, (int)N};
  if (ask == 1) {
    if (avec) return run_bn(la, MatLoader<true, true>{pa, asb, asm_, ask, (int)M}, o, (int)N, (int)M, (int)K, batch, ws);
    return run_bn(la, MatLoader<true, false>{pa, asb, asm_, ask, (int)M}, o, (int)N, (int)M, (int)K, batch, ws);
  }
  return run_bn(la, MatLoader<false, false>{pa, asb, asm_, ask, (int)M}, o, (int)N, (int)M, (int)K, batch, ws);
}

int pb_conv2d_tc(const pb_tensor* x, const pb_tensor* w, const pb_tensor* bias, const pb_conv* p,
                 const pb_tensor* out) {
  if (!f32_all(x, w, out) || (bias && bias->dtype != PB_F32)) return PB_ERR_UNSUPPORTED;
  if (!is_contiguous(*x) || !is_contiguous(*w)) return PB_ERR_UNSUPPORTED;
  Geo g = geo(x->shape, w->shape, p);
  int64_t rows = (int64_t)g.N * g.HO * g.WO, K = (int64_t)g.C * g.KH * g.KW;
  if (rows == 0 || g.F == 0 || K == 0) return PB_ERR_UNSUPPORTED;
  if (!fits_i32(rows * g.F) || !fits_i32((int64_t)g.N * g.C * g.H * g.W)) return PB_ERR_UNSUPPORTED;
  if (!fits_i32((int64_t)g.F * K)) return PB_ERR_UNSUPPORTED;  // weight_rsk indexes in 32 bits
  size_t wbytes = ((size_t)g.F * K * 4 + 255) / 256 * 256;
  char* ws = (char*)workspace(wbytes + split_ws_bytes((int)rows, g.F));
  if (!ws) return fail(PB_ERR_OOM, "conv2d: no workspace");
  float* wt = (float*)ws;
  weight_rsk<<<grid_for((int64_t)g.F * K, 256), 256, 0, compute_stream()>>>((const float*)(uintptr_t)w->ptr, wt, g.F,
                                                                           g.C, g.KH * g.KW, 0);
  PB_LAUNCHED();
  OutConv o{(float*)(uintptr_t)out->ptr, bias ? (const float*)(uintptr_t)bias->ptr : nullptr, (int)rows, g.F,
            FastDiv((uint32_t)(g.HO * g.WO))};
  FastDiv fC(g.C), fKW(g.KW), fP(g.HO * g.WO), fWO(g.WO);
  float* part = (float*)(ws + wbytes);
  if (g.C % 32 == 0) {
    FpropX<true> la{(const float*)(uintptr_t)x->ptr, g, fC, fKW, fP, fWO, (int)rows};
    MatLoader<true, true> lb{wt, 0, K, 1, g.F};
    return run_bn(la, lb, o, (int)rows, g.F, (int)K, 1, part);
  }
  if (g.C % 4 == 0) {
    FpropX<false> la{(const float*)(uintptr_t)x->ptr, g, fC, fKW, fP, fWO, (int)rows};
    MatLoader<true, true> lb{wt, 0, K, 1, g.F};
    return run_bn(la, lb, o, (int)rows, g.F, (int)K, 1, part);
  }
  FpropX<false> la{(const float*)(uintptr_t)x->ptr, g, fC, fKW, fP, fWO, (int)rows};
  MatLoader<true, false> lb{wt, 0, K, 1, g.F};
  return run_bn(la, lb, o, (int)rows, g.F, (int)K, 1, part);
}

int pb_conv2d_grad_input_tc(const pb_tensor* gr, const pb_tensor* w, const pb_conv* p, const pb_tensor* out) {
  if (!f32_all(gr, w, out)) return PB_ERR_UNSUPPORTED;
  if (!is_contiguous(*gr) || !is_contiguous(*w)) return PB_ERR_UNSUPPORTED;
  Geo g = geo(out->shape, w->shape, p);
  int64_t rows = (int64_t)g.N * g.H * g.W, K = (int64_t)g.F * g.KH * g.KW;
  if (rows == 0 || g.C == 0 || K == 0 || g.F % 4 != 0) return PB_ERR_UNSUPPORTED;  // wt rows 16B-aligned
  if (!fits_i32(rows * g.C) || !fits_i32((int64_t)g.N * g.F * g.HO * g.WO)) return PB_ERR_UNSUPPORTED;
  if (!fits_i32((int64_t)g.C * K)) return PB_ERR_UNSUPPORTED;  // weight_rsk indexes in 32 bits
  size_t wbytes = ((size_t)g.C * K * 4 + 255) / 256 * 256;
  char* ws = (char*)workspace(wbytes + split_ws_bytes((int)rows, g.C));
  if (!ws) return fail(PB_ERR_OOM, "conv2d_grad_input: no workspace");
  float* wt = (float*)ws;
  weight_rsk<<<grid_for((int64_t)g.C * K, 256), 256, 0, compute_stream()>>>((const float*)(uintptr_t)w->ptr, wt, g.F,
                                                                           g.C, g.KH * g.KW, 1);
  PB_LAUNCHED();
  OutConv o{(float*)(uintptr_t)out->ptr, nullptr, (int)rows, g.C, FastDiv((uint32_t)(g.H * g.W))};
  MatLoader<true, true> lb{wt, 0, K, 1, g.C};
  if (g.F % 32 == 0) {
    DgradG<true> la{(const float*)(uintptr_t)gr->ptr, g, FastDiv(g.F), FastDiv(g.KW), FastDiv(g.H * g.W),
                    FastDiv(g.W), FastDiv(g.SH), FastDiv(g.SW), (int)rows};
    return run_bn(la, lb, o, (int)rows, g.C, (int)K, 1, (float*)(ws + wbytes));
  }
  DgradG<false> la{(const float*)(uintptr_t)gr->ptr, g, FastDiv(g.F), FastDiv(g.KW), FastDiv(g.H * g.W),
                   FastDiv(g.W), FastDiv(g.SH), FastDiv(g.SW), (int)rows};
  return run_bn(la, lb, o, (int)rows, g.C, (int)K, 1, (float*)(ws + wbytes));
}

int pb_conv2d_grad_weight_tc(const pb_tensor* x, const pb_tensor* gr, const pb_conv* p, const pb_tensor* out) {
  if (!f32_all(x, gr, out)) return PB_ERR_UNSUPPORTED;
  if (!is_contiguous(*x) || !is_contiguous(*gr)) return PB_ERR_UNSUPPORTED;
  Geo g = geo(x->shape, out->shape, p);
  int64_t crs = (int64_t)g.C * g.KH * g.KW, K = (int64_t)g.N * g.HO * g.WO;
  if (crs == 0 || g.F == 0 || K == 0) return PB_ERR_UNSUPPORTED;
  if (!fits_i32(K) || !fits_i32((int64_t)g.N * g.C * g.H * g.W) || !fits_i32((int64_t)g.N * g.F * g.HO * g.WO))
    return PB_ERR_UNSUPPORTED;
  float* ws = (float*)workspace(split_ws_bytes((int)crs, g.F));
  if (!ws) return fail(PB_ERR_OOM, "conv2d_grad_weight: no workspace");
  int P = g.HO * g.WO;
  // D[i = (c,r,s)][j = f] -> dw[f][c][r][s] = out[j * crs + i]
  OutMat o{(float*)(uintptr_t)out->ptr, (int)crs, g.F, crs, 0};
  WgradX la{(const float*)(uintptr_t)x->ptr, g, FastDiv(P), FastDiv(g.WO), FastDiv(g.KH * g.KW), FastDiv(g.KW),
            (int)crs};
  WgradG lb{(const float*)(uintptr_t)gr->ptr, g, FastDiv(P), g.F, (P % 4) == 0};
  return run_bn(la, lb, o, (int)crs, g.F, (int)K, 1, ws);
}

}  // extern "C"

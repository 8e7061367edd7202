// tcgen05 / TMEM / mbarrier PTX wrappers, the 3xTF32 operand split and the output functors
// shared by the contraction kernels (gemm_tc.cu: SIMT-fed; gemm_tma.cu: TMA-fed).  sm_100a only.
#pragma once
#include <stdint.h>
#include "common.cuh"

namespace pb {
namespace tc {

// ---- PTX wrappers ---------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(a),
      "r"(parity)
      : "memory");
}
// one lane of the (converged) warp returns true (elect.sync)
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "elect.sync _|p, 0xffffffff;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(pred));
  return pred != 0;
}
__device__ __forceinline__ void fence_barrier_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

template <int COLS>
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "n"(COLS));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
template <int COLS>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(COLS));
}

// D[tmem] (+)= A[smem] * B[smem]^T, kind::tf32, f32 accumulate
__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// 16 consecutive f32 columns of this thread's TMEM lane (complete after tmem_wait_ld)
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// UMMA shared-memory descriptor: K-major, SWIZZLE_128B, 8-row groups 1024 B apart
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// instruction descriptor: D f32, A/B tf32, both K-major, M x N
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// byte offset of the 16-byte chunk `chunk` (k/4) of row `row` in a 128B-swizzled tile
__device__ __forceinline__ uint32_t swz(int row, int chunk) {
  return (uint32_t)(row * 128 + ((chunk ^ (row & 7)) << 4));
}

// Split x into hi = rna_tf32(x) (integer pipe: add half an ulp, clear 13 bits) and
// lo = rna_tf32(x - hi); x - hi is exact in f32 and |lo| <= 2^-11 |x|.  +-inf keeps
// hi = x, lo = 0 (inf * w then gives the reference's inf, not NaN).
__device__ __forceinline__ void split1(float x, float& h, float& l) {
  uint32_t hb = (__float_as_uint(x) + 0x1000u) & 0xFFFFE000u;
  h = __uint_as_float(hb);
  float d = fabsf(x) == __int_as_float(0x7F800000) ? 0.f : __fsub_rn(x, h);
  l = __uint_as_float((__float_as_uint(d) + 0x1000u) & 0xFFFFE000u);
}
__device__ __forceinline__ void split_store(char* hi_tile, char* lo_tile, uint32_t off, float4 v) {
  float4 h, l;
  split1(v.x, h.x, l.x);
  split1(v.y, h.y, l.y);
  split1(v.z, h.z, l.z);
  split1(v.w, h.w, l.w);
  *reinterpret_cast<float4*>(hi_tile + off) = h;
  *reinterpret_cast<float4*>(lo_tile + off) = l;
}



// =========================================================================================
// Output functors: put(i, j, v) for one D element; rows i are the unit-stride dimension.
// =========================================================================================
struct OutMat {  // C[b][j][i], ld = row pitch (elements)
  float* p;
  int Mi, Nj;
  int64_t ld, sb;
  struct Row {
    float* p;
  };
  __device__ __forceinline__ Row row(int b, int i) const {
    Row o;
    o.p = i < Mi ? p + (int64_t)b * sb + i : nullptr;
    return o;
  }
  __device__ __forceinline__ void put(const Row& rw, int j, float v) const {
    if (rw.p && j < Nj) rw.p[(int64_t)j * ld] = v;
  }
};

struct OutConv {  // out[n][j][pix] for i = (n, pix); optional bias[j]
  float* p;
  const float* bias;
  int Mi, Nj;
  FastDiv fP;
  struct Row {
    float* p;
  };
  __device__ __forceinline__ Row row(int, int i) const {
    Row o;
    o.p = nullptr;
    if (i < Mi) {
      uint32_t n, pix;
      fP.divmod(i, n, pix);
      o.p = p + (int64_t)n * Nj * fP.d + pix;
    }
    return o;
  }
  __device__ __forceinline__ void put(const Row& rw, int j, float v) const {
    if (rw.p && j < Nj) {
      if (bias) v = __fadd_rn(v, __ldg(bias + j));
      rw.p[(int64_t)j * fP.d] = v;
    }
  }
};

struct OutPartial {  // ws[split][j][i] (fold_partials finishes through the real functor)
  float* p;
  int Mi, Nj;
  struct Row {
    float* p;
  };
  __device__ __forceinline__ Row row(int split, int i) const {
    Row o;
    o.p = i < Mi ? p + (int64_t)split * Mi * Nj + i : nullptr;
    return o;
  }
  __device__ __forceinline__ void put(const Row& rw, int j, float v) const {
    if (rw.p && j < Nj) rw.p[(int64_t)j * Mi] = v;
  }
};

// fold split-K partials ws[split][j][i] in split order (f64) and store through OUT.  A thread
// owns V consecutive i of one j (float4 loads when Mi % 4 == 0); all splits' loads are issued
// before the f64 adds, and the (i, j) decode is one 32-bit FastDiv.
template <class OUT, int V>
__global__ void __launch_bounds__(256) fold_partials(const float* __restrict__ ws, int splits, int Mi, int Nj,
                                                     FastDiv fMv, OUT out) {
  const uint32_t MN = (uint32_t)Mi * (uint32_t)Nj, units = MN / V;
  for (uint32_t u = blockIdx.x * blockDim.x + threadIdx.x; u < units; u += gridDim.x * blockDim.x) {
    uint32_t j, iv;
    fMv.divmod(u, j, iv);  // fMv divides by Mi / V
    const uint32_t idx = u * V;
    double a[V];
#pragma unroll
    for (int e = 0; e < V; ++e) a[e] = 0.0;
    int s = 0;
    for (; s + 4 <= splits; s += 4) {
      float v[4][V];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float* src = ws + (size_t)(s + k) * MN + idx;
        if (V == 4) {
          const float4 t = __ldg(reinterpret_cast<const float4*>(src));
          v[k][0] = t.x;
          v[k][V > 1 ? 1 : 0] = t.y;
          v[k][V > 2 ? 2 : 0] = t.z;
          v[k][V > 3 ? 3 : 0] = t.w;
        } else {
          v[k][0] = __ldg(src);
        }
      }
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int e = 0; e < V; ++e) a[e] += (double)v[k][e];
    }
    for (; s < splits; ++s) {
      const float* src = ws + (size_t)s * MN + idx;
#pragma unroll
      for (int e = 0; e < V; ++e) a[e] += (double)__ldg(src + e);
    }
#pragma unroll
    for (int e = 0; e < V; ++e) out.put(out.row(0, (int)(iv * V + e)), (int)j, (float)a[e]);
  }
}

// launch the fold (the partials of split 0 start the sum: v = ws[0] + ws[1] + ... in split order)
template <class OUT>
inline void launch_fold(const float* ws, int splits, int Mi, int Nj, const OUT& out, cudaStream_t st) {
  const int64_t MN = (int64_t)Mi * Nj;
  if (Mi % 4 == 0 && ((uintptr_t)ws & 15) == 0) {
    fold_partials<OUT, 4><<<grid_for(MN / 4, 256), 256, 0, st>>>(ws, splits, Mi, Nj, FastDiv((uint32_t)(Mi / 4)), out);
  } else {
    fold_partials<OUT, 1><<<grid_for(MN, 256), 256, 0, st>>>(ws, splits, Mi, Nj, FastDiv((uint32_t)Mi), out);
  }
}

}  // namespace tc
}  // namespace pb

// Reductions over one axis or all elements: sum / max_reduce / min_reduce / argmax
// (minml/kernels.py:135-160).
//   * f32 sums accumulate in f64 and round once (kernels.py:141-143); integer sums wrap
//     in their own width; f64 sums accumulate in f64.
//   * max/min propagate NaN; argmax returns the first maximum, a NaN beats every number
//     and the first NaN wins (numpy's rule).
// Work decomposition: the reduced axis (extent R, stride sR) is cut into chunks so that
// even a handful of outputs fills all 148 SMs; each (output, chunk) unit is reduced by a
// warp (contiguous reduced axis: lanes read consecutive elements) or by one thread
// (strided reduced axis: consecutive threads own consecutive outputs, so every load
// instruction is coalesced).  Partials land in scratch and a second kernel folds them in
// chunk order, so the result is deterministic run to run.
#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdlib>
#include <type_traits>
#include "common.cuh"

namespace pb {

template <typename T> struct SumAcc { typedef T type; };
template <> struct SumAcc<float> { typedef double type; };
template <> struct SumAcc<bool> { typedef int64_t type; };

template <typename T>
__device__ __forceinline__ bool nan_(T v) { return v != v; }

template <int OP, typename T>
struct Red {
  // accumulator: value (+ index for argmax)
  typedef typename std::conditional<OP == PB_SUM, typename SumAcc<T>::type, T>::type V;
  struct Acc {
    V v;
    int64_t i;
  };
  __device__ __forceinline__ static Acc init() {
    Acc a;
    a.v = V(0);
    a.i = -1;
    return a;
  }
  // fold element x at index idx into a (idx increases along the walk)
  __device__ __forceinline__ static void add(Acc& a, T x, int64_t idx) {
    if (OP == PB_SUM) {
      a.v = (V)(a.v + (V)x);
      return;
    }
    if (a.i < 0) {
      a.v = (V)x;
      a.i = idx;
      return;
    }
    bool take;
    if (OP == PB_RMAX || OP == PB_ARGMAX)
      take = !nan_(a.v) && (nan_((V)x) || (V)x > a.v);
    else
      take = !nan_(a.v) && (nan_((V)x) || (V)x < a.v);
    if (take) {
      a.v = (V)x;
      a.i = idx;
    }
  }
  // combine a (earlier indices) with b (later indices)
  __device__ __forceinline__ static Acc merge(Acc a, Acc b) {
    if (OP == PB_SUM) {
      a.v = (V)(a.v + b.v);
      return a;
    }
    if (b.i < 0) return a;
    if (a.i < 0) return b;
    bool take;
    if (OP == PB_RMAX || OP == PB_ARGMAX)
      take = !nan_(a.v) && (nan_(b.v) || b.v > a.v);
    else
      take = !nan_(a.v) && (nan_(b.v) || b.v < a.v);
    return take ? b : a;
  }
};

template <typename V>
__device__ __forceinline__ V shfl(V v, int src) {
  return __shfl_sync(0xffffffffu, v, src);
}
__device__ __forceinline__ bool shfl(bool v, int src) { return __shfl_sync(0xffffffffu, (int)v, src) != 0; }
__device__ __forceinline__ uint8_t shfl(uint8_t v, int src) { return (uint8_t)__shfl_sync(0xffffffffu, (int)v, src); }

struct RedArgs {
  const void* a;
  void* out;      // final output (chunks == 1) — typed by `dto`
  void* partial;  // [chunks][O] accumulators (chunks > 1)
  int dto;
  int nd;                        // outer (kept) dims, adjacent ones merged when contiguous
  int fast;                      // O < 2^31: decode outputs with 32-bit FastDiv
  int64_t shape[PB_MAX_RANK];    // kept dims, row-major over outputs
  int64_t st[PB_MAX_RANK];       // their strides in a
  FastDiv fd[PB_MAX_RANK];
  int64_t O, R, sR, chunk, chunks;
  int epi, epi_left;  // f32 epilogue: out = op(result, s) or op(s, result); epi < 0: none
  float epi_s;
};

// the f32 result, then the fused scalar op exactly as the elementwise kernel would apply it
__device__ __forceinline__ float epilogue(const RedArgs& r, float v) {
  const float a = r.epi_left ? r.epi_s : v, b = r.epi_left ? v : r.epi_s;
  switch (r.epi) {
    case PB_ADD: return a + b;
    case PB_SUB: return a - b;
    case PB_MUL: return a * b;
    default: return a / b;
  }
}

__device__ __forceinline__ int64_t out_base(const RedArgs& r, int64_t o) {
  int64_t off = 0;
  if (r.fast) {
    uint32_t q = (uint32_t)o;
    for (int k = r.nd - 1; k > 0; --k) {
      uint32_t nq, idx;
      r.fd[k].divmod(q, nq, idx);
      off += (int64_t)idx * r.st[k];
      q = nq;
    }
    return r.nd > 0 ? off + (int64_t)q * r.st[0] : 0;
  }
  for (int k = r.nd - 1; k >= 0; --k) {
    int64_t idx = o % r.shape[k];
    o /= r.shape[k];
    off += idx * r.st[k];
  }
  return off;
}

// fold lane (lane + s)'s accumulator into lane's, for lanes covering [lane, lane + 2s) of an
// interleaved walk: sums add, extrema take the better value with ties (and NaNs) going to the
// lower index, so the result equals a sequential first-wins walk
template <int OP, typename T>
__device__ __forceinline__ void lane_fold(typename Red<OP, T>::Acc& acc, int lane, int s, unsigned mask) {
  typedef Red<OP, T> RD;
  typename RD::Acc other;
  other.v = __shfl_sync(mask, acc.v, (lane + s) & 31);
  other.i = OP == PB_SUM ? 0 : __shfl_sync(mask, acc.i, (lane + s) & 31);
  if ((lane & (2 * s - 1)) != 0) return;
  if (OP == PB_SUM) {
    acc = RD::merge(acc, other);
    return;
  }
  if (other.i < 0) return;
  if (acc.i < 0) {
    acc = other;
    return;
  }
  bool an = nan_(acc.v), bn = nan_(other.v);
  bool take;
  if (an || bn) take = bn && (!an || other.i < acc.i);
  else if (OP == PB_RMAX || OP == PB_ARGMAX) take = other.v > acc.v || (other.v == acc.v && other.i < acc.i);
  else take = other.v < acc.v || (other.v == acc.v && other.i < acc.i);
  if (take) acc = other;
}

template <int OP, typename T>
__device__ __forceinline__ void emit(const RedArgs& r, int64_t o, int64_t c, typename Red<OP, T>::Acc acc) {
  typedef typename Red<OP, T>::Acc Acc;
  if (r.chunks > 1) {
    reinterpret_cast<Acc*>(r.partial)[c * r.O + o] = acc;
    return;
  }
  if (OP == PB_ARGMAX)
    reinterpret_cast<int64_t*>(r.out)[o] = acc.i < 0 ? 0 : acc.i;
  else if (r.epi >= 0)
    reinterpret_cast<float*>(r.out)[o] = epilogue(r, (float)acc.v);
  else
    store_from<typename Red<OP, T>::V>(r.out, r.dto, o, acc.v);
}

// one warp per (output, chunk); reduced axis walked by lanes
template <int OP, typename T>
__global__ void __launch_bounds__(256) red_warp(RedArgs r) {
  typedef Red<OP, T> RD;
  typedef typename RD::Acc Acc;
  const T* a = (const T*)r.a;
  int lane = threadIdx.x & 31;
  int64_t units = r.O * r.chunks;
  int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t u = warp; u < units; u += nwarps) {
    int64_t o = u % r.O, c = u / r.O;
    int64_t base = out_base(r, o);
    int64_t r0 = c * r.chunk, r1 = r0 + r.chunk < r.R ? r0 + r.chunk : r.R;
    Acc acc = RD::init();
    for (int64_t j = r0 + lane; j < r1; j += 32) RD::add(acc, a[base + j * r.sR], j);
    // lanes hold interleaved indices; fold in lane order so ties keep the lowest index
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) lane_fold<OP, T>(acc, lane, s, 0xffffffffu);
    if (lane == 0) emit<OP, T>(r, o, c, acc);
  }
}

// one thread per (output, chunk); the walk issues 8 independent loads at a time
template <int OP, typename T>
__global__ void __launch_bounds__(256) red_thread(RedArgs r) {
  typedef Red<OP, T> RD;
  typedef typename RD::Acc Acc;
  const T* a = (const T*)r.a;
  int64_t units = r.O * r.chunks;
  for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < units; u += (int64_t)gridDim.x * blockDim.x) {
    int64_t o = u % r.O, c = u / r.O;
    int64_t base = out_base(r, o);
    int64_t r0 = c * r.chunk, r1 = r0 + r.chunk < r.R ? r0 + r.chunk : r.R;
    Acc acc = RD::init();
    const T* p = a + base + r0 * r.sR;
    const int64_t sR = r.sR;
    int64_t j = r0;
    if (OP == PB_SUM) {  // independent chains: the dependent f64 add latency bounds the walk
      Acc a1 = RD::init(), a2 = RD::init(), a3 = RD::init();
      for (; j + 8 <= r1; j += 8, p += 8 * sR) {
        T v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = p[q * sR];
        RD::add(acc, v[0], j);
        RD::add(a1, v[1], j);
        RD::add(a2, v[2], j);
        RD::add(a3, v[3], j);
        RD::add(acc, v[4], j);
        RD::add(a1, v[5], j);
        RD::add(a2, v[6], j);
        RD::add(a3, v[7], j);
      }
      acc = RD::merge(RD::merge(acc, a1), RD::merge(a2, a3));
    } else {
      for (; j + 8 <= r1; j += 8, p += 8 * sR) {
        T v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = p[q * sR];
#pragma unroll
        for (int q = 0; q < 8; ++q) RD::add(acc, v[q], j + q);
      }
    }
    for (; j < r1; ++j, p += sR) RD::add(acc, *p, j);
    emit<OP, T>(r, o, c, acc);
  }
}

// short contiguous rows (a + o*R, R <= 128, 4-byte types): the block copies ROWS whole rows
// -- one contiguous span -- into shared memory with coalesced (16-byte when aligned) loads, then
// thread t < ROWS walks row t.  Sums of even-length rows walk the row rotated by t (element
// (j + t) mod R), which makes the strided shared-memory reads bank-conflict free; f32 terms summed in f64
// give the same f32 result in any order (but for rare ties).  Extrema walk in index order.
template <int OP, typename T>
__global__ void __launch_bounds__(256) red_rows(RedArgs r, int rows_per_block, int vec) {
  typedef Red<OP, T> RD;
  typedef typename RD::Acc Acc;
  extern __shared__ float4 rows_smem4[];
  T* buf = reinterpret_cast<T*>(rows_smem4);
  const T* a = (const T*)r.a;
  const int R = (int)r.R;
  for (int64_t o0 = (int64_t)blockIdx.x * rows_per_block; o0 < r.O; o0 += (int64_t)gridDim.x * rows_per_block) {
    const int rows = (int)(r.O - o0 < rows_per_block ? r.O - o0 : rows_per_block);
    const int n = rows * R;
    const T* src = a + o0 * R;
    int e0 = 0;
    if (vec) {  // o0 * R % 4 == 0 and the base is 16-byte aligned
      const int n4 = n >> 2;
      const float4* s4 = reinterpret_cast<const float4*>(src);
      // 4 loads in flight per thread before any shared-memory store
      for (int q0 = threadIdx.x; q0 < n4; q0 += 4 * blockDim.x) {
        float4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int q = q0 + u * blockDim.x;
          if (q < n4) v[u] = __ldg(s4 + q);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int q = q0 + u * blockDim.x;
          if (q < n4) rows_smem4[q] = v[u];
        }
      }
      e0 = n4 << 2;
    }
    for (int e0b = e0 + threadIdx.x; e0b < n; e0b += 4 * blockDim.x) {
      T v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = e0b + u * blockDim.x;
        if (e < n) v[u] = src[e];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = e0b + u * blockDim.x;
        if (e < n) buf[e] = v[u];
      }
    }
    __syncthreads();
    if ((int)threadIdx.x < rows) {
      const int t = threadIdx.x;
      const T* row = buf + t * R;
      Acc acc = RD::init();
      if (OP == PB_SUM) {
        Acc a1 = RD::init(), a2 = RD::init(), a3 = RD::init();
        int j = (R & 1) ? 0 : t % R;  // rotate even rows (odd R is conflict free as is)
        int k = 0;
        for (; k + 4 <= R; k += 4) {
          RD::add(acc, row[j], j);
          j = j + 1 == R ? 0 : j + 1;
          RD::add(a1, row[j], j);
          j = j + 1 == R ? 0 : j + 1;
          RD::add(a2, row[j], j);
          j = j + 1 == R ? 0 : j + 1;
          RD::add(a3, row[j], j);
          j = j + 1 == R ? 0 : j + 1;
        }
        for (; k < R; ++k) {
          RD::add(acc, row[j], j);
          j = j + 1 == R ? 0 : j + 1;
        }
        acc = RD::merge(RD::merge(acc, a1), RD::merge(a2, a3));
      } else {
        for (int j = 0; j < R; ++j) RD::add(acc, row[j], j);
      }
      emit<OP, T>(r, o0 + t, 0, acc);
    }
    __syncthreads();
  }
}

// strided reduced axis (sR > 1), R <= 4096: a block owns 32 consecutive outputs (one per lane,
// so each load instruction is coalesced along the kept inner axis) and splits the reduced axis
// into 8 contiguous slices (one per warp); the slices fold in order through shared memory.
// One launch, deterministic, and each thread walks at most R/8 elements.
template <int OP, typename T>
__global__ void __launch_bounds__(256) red_cols(RedArgs r) {
  typedef Red<OP, T> RD;
  typedef typename RD::Acc Acc;
  __shared__ Acc part[8][32];
  const T* a = (const T*)r.a;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t slice = (r.R + 7) / 8;
  const int64_t j0 = ty * slice, j1 = j0 + slice < r.R ? j0 + slice : r.R;
  for (int64_t o0 = (int64_t)blockIdx.x * 32; o0 < r.O; o0 += (int64_t)gridDim.x * 32) {
    const int64_t o = o0 + tx;
    Acc acc = RD::init();
    if (o < r.O) {
      const T* p = a + out_base(r, o);
      const int64_t sR = r.sR;
#pragma unroll 4
      for (int64_t j = j0; j < j1; ++j) RD::add(acc, p[j * sR], j);
    }
    part[ty][tx] = acc;
    __syncthreads();
    if (ty == 0 && o < r.O) {
#pragma unroll
      for (int t = 1; t < 8; ++t) acc = RD::merge(acc, part[t][tx]);
      emit<OP, T>(r, o, 0, acc);
    }
    __syncthreads();
  }
}

// f32 sum over a strided axis whose innermost kept axis is contiguous (extent % 4 == 0, every
// stride % 4 == 0, 16-byte aligned base): each thread owns 4 consecutive outputs and walks the
// whole reduced axis with float4 loads, 8 in flight (a warp reads 512 contiguous bytes per
// load), summing each output in f64 in index order.  No shared memory, no block barrier.
// This is the reference's _unbroadcast sum(0) over [N, C, H, W] (minml/autograd.py:290-297).
__global__ void __launch_bounds__(256) red_cols4_sum(RedArgs r) {
  const float* a = (const float*)r.a;
  const int64_t O4 = r.O >> 2, R = r.R, sR = r.sR;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < O4; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = q << 2;
    const float* p = a + out_base(r, o);
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int64_t j = 0;
    for (; j + 8 <= R; j += 8) {
      float4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldg(reinterpret_cast<const float4*>(p + (j + u) * sR));
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        s0 += (double)v[u].x;
        s1 += (double)v[u].y;
        s2 += (double)v[u].z;
        s3 += (double)v[u].w;
      }
    }
    for (; j < R; ++j) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(p + j * sR));
      s0 += (double)v.x;
      s1 += (double)v.y;
      s2 += (double)v.z;
      s3 += (double)v.w;
    }
    typedef Red<PB_SUM, float>::Acc Acc;
    Acc c0{s0, -1}, c1{s1, -1}, c2{s2, -1}, c3{s3, -1};
    emit<PB_SUM, float>(r, o, 0, c0);
    emit<PB_SUM, float>(r, o + 1, 0, c1);
    emit<PB_SUM, float>(r, o + 2, 0, c2);
    emit<PB_SUM, float>(r, o + 3, 0, c3);
  }
}

// the same walk for fewer outputs: a block owns 128 consecutive outputs (32 lanes x float4)
// and its 8 warps take consecutive slices of the reduced axis; the slice sums fold in slice
// order through shared memory (the [1, C, H, W] sum(2) and [N, C] sum(0) of _unbroadcast)
__global__ void __launch_bounds__(256) red_cols4s_sum(RedArgs r) {
  __shared__ double part[8][32][4];
  const float* a = (const float*)r.a;
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const int64_t R = r.R, sR = r.sR, slice = (R + 7) / 8;
  const int64_t j0 = wp * slice, j1 = j0 + slice < R ? j0 + slice : R;
  for (int64_t o0 = (int64_t)blockIdx.x * 128; o0 < r.O; o0 += (int64_t)gridDim.x * 128) {
    const int64_t o = o0 + lane * 4;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    if (o < r.O) {
      const float* p = a + out_base(r, o);
      int64_t j = j0;
      for (; j + 4 <= j1; j += 4) {
        float4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = __ldg(reinterpret_cast<const float4*>(p + (j + u) * sR));
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          s0 += (double)v[u].x;
          s1 += (double)v[u].y;
          s2 += (double)v[u].z;
          s3 += (double)v[u].w;
        }
      }
      for (; j < j1; ++j) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(p + j * sR));
        s0 += (double)v.x;
        s1 += (double)v.y;
        s2 += (double)v.z;
        s3 += (double)v.w;
      }
    }
    part[wp][lane][0] = s0;
    part[wp][lane][1] = s1;
    part[wp][lane][2] = s2;
    part[wp][lane][3] = s3;
    __syncthreads();
    if (wp == 0 && o < r.O) {
#pragma unroll
      for (int t = 1; t < 8; ++t) {
        s0 += part[t][lane][0];
        s1 += part[t][lane][1];
        s2 += part[t][lane][2];
        s3 += part[t][lane][3];
      }
      typedef Red<PB_SUM, float>::Acc Acc;
      Acc c0{s0, -1}, c1{s1, -1}, c2{s2, -1}, c3{s3, -1};
      emit<PB_SUM, float>(r, o, 0, c0);
      emit<PB_SUM, float>(r, o + 1, 0, c1);
      emit<PB_SUM, float>(r, o + 2, 0, c2);
      emit<PB_SUM, float>(r, o + 3, 0, c3);
    }
    __syncthreads();
  }
}

// fold chunk partials in chunk order
template <int OP, typename T>
__global__ void __launch_bounds__(256) red_final(RedArgs r) {
  typedef Red<OP, T> RD;
  typedef typename RD::Acc Acc;
  const Acc* part = (const Acc*)r.partial;
  for (int64_t o = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; o < r.O; o += (int64_t)gridDim.x * blockDim.x) {
    Acc acc = part[o];
    for (int64_t c = 1; c < r.chunks; ++c) acc = RD::merge(acc, part[c * r.O + o]);
    if (OP == PB_ARGMAX)
      reinterpret_cast<int64_t*>(r.out)[o] = acc.i < 0 ? 0 : acc.i;
    else if (r.epi >= 0)
      reinterpret_cast<float*>(r.out)[o] = epilogue(r, (float)acc.v);
    else
      store_from<typename RD::V>(r.out, r.dto, o, acc.v);
  }
}

template <int OP, typename T>
static int run_reduce(const pb_tensor* a, int axis, const pb_tensor* out, int epi, float epi_s, int epi_left) {
  typedef typename Red<OP, T>::Acc Acc;
  RedArgs r;
  r.epi = epi;
  r.epi_s = epi_s;
  r.epi_left = epi_left;
  r.a = (const void*)(uintptr_t)a->ptr;
  r.out = (void*)(uintptr_t)out->ptr;
  r.dto = out->dtype;
  r.nd = 0;
  if (axis < 0) {
    if (!is_contiguous(*a)) return fail(PB_ERR_ARG, "pb_reduce: full reduction needs a contiguous input");
    r.R = numel(*a);
    r.sR = 1;
  } else {
    r.R = a->shape[axis];
    r.sR = a->strides[axis];
    for (int k = 0; k < a->ndim; ++k) {
      if (k == axis) continue;
      r.shape[r.nd] = a->shape[k];
      r.st[r.nd] = a->strides[k];
      r.nd++;
    }
  }
  {  // merge kept dim k into k-1 when they are contiguous with each other
    int nd = 0;
    for (int k = 0; k < r.nd; ++k) {
      if (r.shape[k] == 1) continue;
      if (nd > 0 && r.st[nd - 1] == r.st[k] * r.shape[k]) {
        r.shape[nd - 1] *= r.shape[k];
        r.st[nd - 1] = r.st[k];
        continue;
      }
      r.shape[nd] = r.shape[k];
      r.st[nd] = r.st[k];
      ++nd;
    }
    r.nd = nd;
  }
  r.O = 1;
  for (int k = 0; k < r.nd; ++k) r.O *= r.shape[k];
  r.fast = r.O < ((int64_t)1 << 31);
  for (int k = 0; k < r.nd && r.fast; ++k) r.fd[k] = FastDiv((uint32_t)r.shape[k]);
  if (r.O == 0) return PB_OK;
  if (r.R == 0) {  // empty sum -> zeros (max/min/argmax rejected by the planner)
    if (epi >= 0) return fail(PB_ERR_UNSUPPORTED, "pb_reduce_epi: empty reduction");
    pb_scalar z = {1, 0, 0.0, 0};
    return pb_fill(out, &z);
  }
  if (r.R == 1) r.sR = 1;
  cudaStream_t s = compute_stream();
  if (sizeof(T) == 4 && r.sR == 1 && r.R > 1 && r.R <= 128 && r.nd == 1 && r.st[0] == r.R && r.O >= 1024 &&
      r.O * r.R < ((int64_t)1 << 31)) {
    r.chunks = 1;
    r.chunk = r.R;
    r.partial = nullptr;
    static const int rdiv = getenv("PB_RED_ROWS_DIV") ? atoi(getenv("PB_RED_ROWS_DIV")) : 1;  // experiment hook
    const int rows = (r.R <= 32 ? 256 : r.R <= 64 ? 128 : 64) / (rdiv > 0 ? rdiv : 1);
    const size_t smem = (size_t)rows * r.R * 4;
    static bool attr = false;
    if (!attr) {
      PB_CUDA(cudaFuncSetAttribute(red_rows<OP, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
      attr = true;
    }
    const int per_sm = (int)((200 * 1024) / smem) < 8 ? (int)((200 * 1024) / smem) : 8;
    const int64_t blocks = (r.O + rows - 1) / rows;
    const int64_t cap = (int64_t)num_sms() * (per_sm > 0 ? per_sm : 1);
    const int grid = (int)(blocks < cap ? blocks : cap);
    const int vec = (rows * r.R) % 4 == 0 && ((uintptr_t)r.a) % 16 == 0;
    red_rows<OP, T><<<grid, 256, smem, s>>>(r, rows, vec);
    PB_LAUNCHED();
    return PB_OK;
  }
  if (OP == PB_SUM && std::is_same<T, float>::value && r.sR > 1 && r.sR % 4 == 0 && r.nd >= 1 &&
      r.st[r.nd - 1] == 1 && r.shape[r.nd - 1] % 4 == 0 && ((uintptr_t)r.a) % 16 == 0 && r.R <= 4096 &&
      (r.O >= 4096 || r.R <= 64)) {
    bool ok = true;
    for (int k = 0; k + 1 < r.nd; ++k) ok = ok && r.st[k] % 4 == 0;
    if (ok) {
      r.chunks = 1;
      r.chunk = r.R;
      r.partial = nullptr;
      const int64_t threads = r.O / 4;
      static const int64_t thr = getenv("PB_RED_COLS_THR") ? atoll(getenv("PB_RED_COLS_THR")) : 512;  // experiment hook
      if (threads >= (int64_t)num_sms() * thr || r.R < 16) {  // enough outputs: one thread walks all of R
        const int64_t blocks = (threads + 255) / 256;
        const int grid = (int)(blocks < (int64_t)num_sms() * 8 ? blocks : (int64_t)num_sms() * 8);
        red_cols4_sum<<<grid, 256, 0, s>>>(r);
      } else {  // few outputs: 8 warps split R
        const int64_t blocks = (r.O + 127) / 128;
        const int grid = (int)(blocks < (int64_t)num_sms() * 8 ? blocks : (int64_t)num_sms() * 8);
        red_cols4s_sum<<<grid, 256, 0, s>>>(r);
      }
      PB_LAUNCHED();
      return PB_OK;
    }
  }
  if (r.sR > 1 && r.R <= 4096) {
    r.chunks = 1;
    r.chunk = r.R;
    r.partial = nullptr;
    const int64_t blocks = (r.O + 31) / 32;
    const int grid = (int)(blocks < (int64_t)num_sms() * 16 ? blocks : (int64_t)num_sms() * 16);
    red_cols<OP, T><<<grid, 256, 0, s>>>(r);
    PB_LAUNCHED();
    return PB_OK;
  }
  bool warp_mode = (r.sR == 1 && r.R >= 32);
  int64_t target = warp_mode ? (int64_t)num_sms() * 64 : (int64_t)num_sms() * 1024;
  int64_t min_chunk = warp_mode ? 2048 : 128;
  int64_t chunks = (target + r.O - 1) / r.O;
  int64_t max_chunks = (r.R + min_chunk - 1) / min_chunk;
  if (chunks > max_chunks) chunks = max_chunks;
  if (chunks < 1) chunks = 1;
  r.chunks = chunks;
  r.chunk = (r.R + chunks - 1) / chunks;
  if (chunks > 1) {
    r.partial = workspace(sizeof(Acc) * r.O * chunks);
    if (!r.partial) return fail(PB_ERR_OOM, "pb_reduce: no workspace");
  } else {
    r.partial = nullptr;
  }
  int64_t units = r.O * chunks;
  if (warp_mode) {
    int64_t blocks = (units * 32 + 255) / 256;
    int grid = (int)(blocks < (int64_t)num_sms() * 16 ? blocks : (int64_t)num_sms() * 16);
    red_warp<OP, T><<<grid, 256, 0, s>>>(r);
  } else {
    int grid = grid_for(units, 256);
    red_thread<OP, T><<<grid, 256, 0, s>>>(r);
  }
  PB_LAUNCHED();
  if (chunks > 1) {
    red_final<OP, T><<<grid_for(r.O, 256), 256, 0, s>>>(r);
    PB_LAUNCHED();
  }
  return PB_OK;
}

template <int OP>
static int dispatch(const pb_tensor* a, int axis, const pb_tensor* out, int epi = -1, float s = 0.f, int left = 0) {
  if (epi >= 0 && (a->dtype != PB_F32 || out->dtype != PB_F32 || OP == PB_ARGMAX))
    return fail(PB_ERR_UNSUPPORTED, "pb_reduce_epi: f32 sum/max/min only");
  switch (a->dtype) {
    case PB_BOOL: return run_reduce<OP, bool>(a, axis, out, epi, s, left);
    case PB_U8: return run_reduce<OP, uint8_t>(a, axis, out, epi, s, left);
    case PB_I32: return run_reduce<OP, int32_t>(a, axis, out, epi, s, left);
    case PB_I64: return run_reduce<OP, int64_t>(a, axis, out, epi, s, left);
    case PB_F32: return run_reduce<OP, float>(a, axis, out, epi, s, left);
    case PB_F64: return run_reduce<OP, double>(a, axis, out, epi, s, left);
  }
  return fail(PB_ERR_ARG, "pb_reduce: bad dtype");
}

}  // namespace pb

using namespace pb;

extern "C" int pb_reduce(int op, const pb_tensor* a, int axis, const pb_tensor* out) {
  switch (op) {
    case PB_SUM: return dispatch<PB_SUM>(a, axis, out);
    case PB_RMAX: return dispatch<PB_RMAX>(a, axis, out);
    case PB_RMIN: return dispatch<PB_RMIN>(a, axis, out);
    case PB_ARGMAX: return dispatch<PB_ARGMAX>(a, axis, out);
  }
  return fail(PB_ERR_ARG, "pb_reduce: unknown op");
}

// pb_reduce followed by an f32 scalar op on each result -- the reference's mean
// (sum / n, minml/ops.py:33-36) in one launch; bit-identical to the two primitives
extern "C" int pb_reduce_epi(int op, const pb_tensor* a, int axis, const pb_tensor* out, int epi_op, float scalar,
                             int scalar_left) {
  if (epi_op != PB_ADD && epi_op != PB_SUB && epi_op != PB_MUL && epi_op != PB_DIV)
    return fail(PB_ERR_ARG, "pb_reduce_epi: epilogue must be add/sub/mul/div");
  switch (op) {
    case PB_SUM: return dispatch<PB_SUM>(a, axis, out, epi_op, scalar, scalar_left);
    case PB_RMAX: return dispatch<PB_RMAX>(a, axis, out, epi_op, scalar, scalar_left);
    case PB_RMIN: return dispatch<PB_RMIN>(a, axis, out, epi_op, scalar, scalar_left);
  }
  return fail(PB_ERR_ARG, "pb_reduce_epi: unknown op");
}

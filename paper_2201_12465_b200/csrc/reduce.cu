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
  int nd;                        // outer (kept) dims
  int64_t shape[PB_MAX_RANK];    // kept dims, row-major over outputs
  int64_t st[PB_MAX_RANK];       // their strides in a
  int64_t O, R, sR, chunk, chunks;
};

__device__ __forceinline__ int64_t out_base(const RedArgs& r, int64_t o) {
  int64_t off = 0;
  for (int k = r.nd - 1; k >= 0; --k) {
    int64_t idx = o % r.shape[k];
    o /= r.shape[k];
    off += idx * r.st[k];
  }
  return off;
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
    for (int s = 1; s < 32; s <<= 1) {
      Acc other;
      other.v = shfl(acc.v, (lane + s) & 31);
      other.i = __shfl_sync(0xffffffffu, acc.i, (lane + s) & 31);
      if ((lane & (2 * s - 1)) == 0) {
        // lane covers [lane, lane+2s); other covers [lane+s, lane+2s)
        if (OP == PB_SUM) acc = RD::merge(acc, other);
        else {
          // pick by value, tie -> smaller index (indices are interleaved, not ordered)
          if (other.i >= 0) {
            if (acc.i < 0) acc = other;
            else {
              bool an = nan_(acc.v), bn = nan_(other.v);
              bool take;
              if (an || bn) take = bn && (!an || other.i < acc.i);
              else if (OP == PB_RMAX || OP == PB_ARGMAX) take = other.v > acc.v || (other.v == acc.v && other.i < acc.i);
              else take = other.v < acc.v || (other.v == acc.v && other.i < acc.i);
              if (take) acc = other;
            }
          }
        }
      }
    }
    if (lane == 0) emit<OP, T>(r, o, c, acc);
  }
}

// one thread per (output, chunk)
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
    for (int64_t j = r0; j < r1; ++j, p += r.sR) RD::add(acc, *p, j);
    emit<OP, T>(r, o, c, acc);
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
    else
      store_from<typename RD::V>(r.out, r.dto, o, acc.v);
  }
}

template <int OP, typename T>
static int run_reduce(const pb_tensor* a, int axis, const pb_tensor* out) {
  typedef typename Red<OP, T>::Acc Acc;
  RedArgs r;
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
  r.O = 1;
  for (int k = 0; k < r.nd; ++k) r.O *= r.shape[k];
  if (r.O == 0) return PB_OK;
  if (r.R == 0) {  // empty sum -> zeros (max/min/argmax rejected by the planner)
    pb_scalar z = {1, 0, 0.0, 0};
    return pb_fill(out, &z);
  }
  if (r.R == 1) r.sR = 1;
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
  cudaStream_t s = compute_stream();
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
static int dispatch(const pb_tensor* a, int axis, const pb_tensor* out) {
  switch (a->dtype) {
    case PB_BOOL: return run_reduce<OP, bool>(a, axis, out);
    case PB_U8: return run_reduce<OP, uint8_t>(a, axis, out);
    case PB_I32: return run_reduce<OP, int32_t>(a, axis, out);
    case PB_I64: return run_reduce<OP, int64_t>(a, axis, out);
    case PB_F32: return run_reduce<OP, float>(a, axis, out);
    case PB_F64: return run_reduce<OP, double>(a, axis, out);
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

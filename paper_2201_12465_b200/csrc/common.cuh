// Shared plumbing for libpaper_b200.so: error reporting, streams, dtype dispatch and
// numpy-compatible scalar conversions (the value-domain rules of minml/kernels.py:1-32).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <cmath>
#include <string>
#include "../../include/paper_b200.h"

namespace pb {

// ---- errors -------------------------------------------------------------------------
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* where);

#define PB_CUDA(call)                                   \
  do {                                                  \
    cudaError_t e_ = (call);                            \
    if (e_ != cudaSuccess) return ::pb::cuda_fail(e_, #call); \
  } while (0)

#define PB_LAUNCHED()                                                   \
  do {                                                                  \
    ::pb::count_launch();                                               \
    cudaError_t e_ = cudaGetLastError();                                \
    if (e_ != cudaSuccess) return ::pb::cuda_fail(e_, __func__);        \
  } while (0)

// ---- runtime state ------------------------------------------------------------------
cudaStream_t compute_stream();
cudaStream_t comm_stream();
cudaStream_t copy_stream();
int num_sms();
void count_launch();
// grow-only device scratch on the compute stream (stream order makes reuse safe)
void* workspace(size_t bytes);
// n zeroed ticket counters (nullptr if n > kTickCounters); users leave them zero again
constexpr int64_t kTickCounters = 1 << 16;
unsigned* tick_counters(int64_t n);

// ---- dtypes -------------------------------------------------------------------------
inline int itemsize(int dt) {
  switch (dt) {
    case PB_BOOL: case PB_U8: return 1;
    case PB_I32: return 4;
    case PB_I64: return 8;
    case PB_F32: return 4;
    default: return 8;
  }
}

// numpy's unsafe casts as compiled for x86-64: float->int truncates toward zero and
// maps NaN / out-of-range to INT_MIN ("integer indefinite"); float->u8 goes through
// int32 then keeps the low byte; int->int wraps; anything->bool is (x != 0).
template <typename To, typename From>
struct Cvt {
  __host__ __device__ static To run(From v) { return static_cast<To>(v); }
};
template <typename From>
struct Cvt<bool, From> {
  __host__ __device__ static bool run(From v) { return v != From(0); }
};
__host__ __device__ inline int32_t f2i32(double v) {
  if (!(v > -2147483649.0 && v < 2147483648.0)) return INT32_MIN;  // catches NaN
  return (int32_t)v;
}
__host__ __device__ inline int64_t f2i64(double v) {
  if (!(v >= -9223372036854775808.0 && v < 9223372036854775808.0)) return INT64_MIN;
  return (int64_t)v;
}
template <> struct Cvt<int32_t, float> { __host__ __device__ static int32_t run(float v) { return f2i32(v); } };
template <> struct Cvt<int32_t, double> { __host__ __device__ static int32_t run(double v) { return f2i32(v); } };
template <> struct Cvt<int64_t, float> { __host__ __device__ static int64_t run(float v) { return f2i64(v); } };
template <> struct Cvt<int64_t, double> { __host__ __device__ static int64_t run(double v) { return f2i64(v); } };
template <> struct Cvt<uint8_t, float> { __host__ __device__ static uint8_t run(float v) { return (uint8_t)(uint32_t)f2i32(v); } };
template <> struct Cvt<uint8_t, double> { __host__ __device__ static uint8_t run(double v) { return (uint8_t)(uint32_t)f2i32(v); } };
template <> struct Cvt<bool, bool> { __host__ __device__ static bool run(bool v) { return v; } };

template <typename To, typename From>
__host__ __device__ inline To cvt(From v) { return Cvt<To, From>::run(v); }

// load element i (already an element offset) of a runtime-typed buffer as T
template <typename T>
__device__ __forceinline__ T load_as(const void* p, int dt, int64_t i) {
  switch (dt) {
    case PB_BOOL: return cvt<T>(((const bool*)p)[i]);
    case PB_U8: return cvt<T>(((const uint8_t*)p)[i]);
    case PB_I32: return cvt<T>(((const int32_t*)p)[i]);
    case PB_I64: return cvt<T>(((const int64_t*)p)[i]);
    case PB_F32: return cvt<T>(((const float*)p)[i]);
    default: return cvt<T>(((const double*)p)[i]);
  }
}

template <typename T>
__device__ __forceinline__ void store_from(void* p, int dt, int64_t i, T v) {
  switch (dt) {
    case PB_BOOL: ((bool*)p)[i] = cvt<bool>(v); break;
    case PB_U8: ((uint8_t*)p)[i] = cvt<uint8_t>(v); break;
    case PB_I32: ((int32_t*)p)[i] = cvt<int32_t>(v); break;
    case PB_I64: ((int64_t*)p)[i] = cvt<int64_t>(v); break;
    case PB_F32: ((float*)p)[i] = cvt<float>(v); break;
    default: ((double*)p)[i] = cvt<double>(v); break;
  }
}

// scalar operand converted to the compute type on the host (numpy weak-scalar rule)
template <typename T>
inline T scalar_as(const pb_scalar* s) {
  if (s->kind == 0) return cvt<T>(s->f);
  return cvt<T>((int64_t)s->i);
}

// ---- N-d index helpers ----------------------------------------------------------------
struct Dims {
  int ndim;
  int64_t shape[PB_MAX_RANK];
  int64_t st[3][PB_MAX_RANK];  // strides of up to three operands (elements)
};

// merge adjacent axes that are contiguous in every operand; drop extent-1 axes
void coalesce(Dims& d, int nops);
bool is_contiguous(const pb_tensor& t);
int64_t numel(const pb_tensor& t);

template <int N>
__device__ __forceinline__ void offsets(const Dims& d, int64_t linear, int64_t* off, int nops) {
  // last axis fastest
#pragma unroll
  for (int o = 0; o < 3; ++o) off[o] = 0;
  for (int k = d.ndim - 1; k >= 0; --k) {
    int64_t ext = d.shape[k];
    int64_t idx = linear % ext;
    linear /= ext;
#pragma unroll
    for (int o = 0; o < 3; ++o)
      if (o < nops) off[o] += idx * d.st[o][k];
  }
}

// ---- fast unsigned division by a runtime constant (n < 2^31) ------------------------------
struct FastDiv {
  uint32_t d, m, s;
  FastDiv() : d(1), m(0), s(0) {}
  explicit FastDiv(uint32_t dv) : d(dv) {
    s = 0;
    while ((1u << s) < d) ++s;
    m = (uint32_t)((((uint64_t)1 << 32) * (((uint64_t)1 << s) - d)) / d + 1);
  }
  __device__ __forceinline__ uint32_t div(uint32_t n) const { return (__umulhi(n, m) + n) >> s; }
  __device__ __forceinline__ void divmod(uint32_t n, uint32_t& q, uint32_t& r) const {
    q = div(n);
    r = n - q * d;
  }
};

inline int grid_for(int64_t n, int threads, int per_thread = 1) {
  int64_t blocks = (n + (int64_t)threads * per_thread - 1) / ((int64_t)threads * per_thread);
  int64_t cap = (int64_t)num_sms() * 32;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  return (int)blocks;
}

}  // namespace pb

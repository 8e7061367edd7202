// Counter-based RNG fills (minml/rng.py:16-51, kernels.py:65-74).
// word(i) = splitmix64 finalizer of seed + (i+1)*GOLDEN; uniform = (word >> 11) * 2^-53
// in f64, then rounded to the output dtype — bit-exact with the reference.  Normals use
// Box-Muller in f64: pair k takes u1 = U(offset+k), u2 = U(offset+pairs+k) and writes
// r*cos(t) to element 2k and r*sin(t) to element 2k+1 (libm-level agreement, <= 1 ulp f64).
#include <cuda_runtime.h>
#include <stdint.h>
#include "common.cuh"

namespace pb {

__device__ __forceinline__ uint64_t splitmix(uint64_t seed, uint64_t counter) {
  uint64_t z = seed + (counter + 1ull) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ double unit(uint64_t seed, uint64_t counter) {
  return (double)(splitmix(seed, counter) >> 11) * 1.1102230246251565e-16;  // 2^-53
}

// `base` (may be null): a device-resident counter added to `offset` at run time, so a fill
// recorded into a CUDA graph draws fresh counters on every replay (see pb_rand_dev)
template <typename T>
__global__ void __launch_bounds__(256) uniform_kernel(T* out, int64_t n, uint64_t seed, uint64_t offset,
                                                      const uint64_t* base) {
  if (base) offset += *base;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (T)unit(seed, offset + (uint64_t)i);
}

template <typename T>
__global__ void __launch_bounds__(256) normal_kernel(T* out, int64_t n, uint64_t seed, uint64_t offset,
                                                     const uint64_t* base) {
  if (base) offset += *base;
  int64_t pairs = (n + 1) / 2;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < pairs; k += (int64_t)gridDim.x * blockDim.x) {
    double u1 = unit(seed, offset + (uint64_t)k);
    double u2 = unit(seed, offset + (uint64_t)pairs + (uint64_t)k);
    double rad = sqrt(-2.0 * log1p(-u1));
    double th = 2.0 * 3.141592653589793 * u2;
    out[2 * k] = (T)(rad * cos(th));
    if (2 * k + 1 < n) out[2 * k + 1] = (T)(rad * sin(th));
  }
}

}  // namespace pb

using namespace pb;

__global__ void counter_add_kernel(uint64_t* c, uint64_t inc) { *c += inc; }

static int rand_fill(int normal, uint64_t seed, uint64_t offset, const uint64_t* base, const pb_tensor* out) {
  int64_t n = numel(*out);
  if (n == 0) return PB_OK;
  if (!is_contiguous(*out)) return fail(PB_ERR_ARG, "pb_rand: output must be contiguous");
  int grid = grid_for(normal ? (n + 1) / 2 : n, 256, 2);
  cudaStream_t s = compute_stream();
  void* p = (void*)(uintptr_t)out->ptr;
  if (out->dtype == PB_F32) {
    if (normal) normal_kernel<float><<<grid, 256, 0, s>>>((float*)p, n, seed, offset, base);
    else uniform_kernel<float><<<grid, 256, 0, s>>>((float*)p, n, seed, offset, base);
  } else if (out->dtype == PB_F64) {
    if (normal) normal_kernel<double><<<grid, 256, 0, s>>>((double*)p, n, seed, offset, base);
    else uniform_kernel<double><<<grid, 256, 0, s>>>((double*)p, n, seed, offset, base);
  } else {
    return fail(PB_ERR_ARG, "pb_rand: float outputs only");
  }
  PB_LAUNCHED();
  return PB_OK;
}

extern "C" int pb_rand(int normal, uint64_t seed, uint64_t offset, const pb_tensor* out) {
  return rand_fill(normal, seed, offset, nullptr, out);
}

extern "C" int pb_rand_dev(int normal, uint64_t seed, uint64_t base_ptr, uint64_t delta, const pb_tensor* out) {
  if (!base_ptr) return fail(PB_ERR_ARG, "pb_rand_dev: null counter");
  return rand_fill(normal, seed, delta, (const uint64_t*)(uintptr_t)base_ptr, out);
}

extern "C" int pb_counter_add(uint64_t counter_ptr, uint64_t inc) {
  if (!counter_ptr) return fail(PB_ERR_ARG, "pb_counter_add: null counter");
  counter_add_kernel<<<1, 1, 0, compute_stream()>>>((uint64_t*)(uintptr_t)counter_ptr, inc);
  PB_LAUNCHED();
  return PB_OK;
}

// SIMT contraction kernels: matmul (rank-2 / batched rank-3) and conv2d fprop / dgrad /
// wgrad as implicit GEMMs with on-the-fly im2col gathers (minml/kernels.py:166-239).
//
// This is the general path: any dtype (f64 and integer matmuls, mixed-dtype operands that
// numpy promotes to f64), any operand strides (transposed views need no copy), any conv
// stride/padding.  f32 x f32 contractions are routed to the tcgen05 3xTF32 kernels in
// gemm_tc.cu when that path is enabled; this file is their fallback and reference.
// Tile: 128x128 outputs per 256-thread block, 8x8 per thread, K staged 16 at a time
// through shared memory.  wgrad (tiny M*N, huge K = N*Ho*Wo) is split over K into
// deterministic partial sums folded in order by a second kernel.
#include <cuda_runtime.h>
#include <stdint.h>
#include "common.cuh"

namespace pb {

static const int BM = 128, BN = 128, BK = 16, TM = 8, TN = 8;

// f32 operands accumulate in f64: every f32*f32 product is exact in f64, so results match
// the reference's f64 contraction (kernels.py:168-169) to the final f32 rounding.
template <typename T> struct AccOf { typedef T type; };
template <> struct AccOf<float> { typedef double type; };

template <typename T>
struct MatA {  // element (b, r, c) of a strided rank-3 view
  const void* p;
  int dt;
  int64_t sb, sr, sc;
  int R, C;
  __device__ __forceinline__ T get(int b, int r, int c) const {
    if (r >= R || c >= C) return T(0);
    return load_as<T>(p, dt, (int64_t)b * sb + (int64_t)r * sr + (int64_t)c * sc);
  }
};

struct ConvGeom {
  int N, C, H, W, F, KH, KW, SH, SW, PH, PW, HO, WO;
};

// fprop B[k=(c,r,s)][j=(n,ho,wo)] = x[n, c, ho*sh-ph+r, wo*sw-pw+s]
template <typename T>
struct FpropB {
  const void* x;
  int dt;
  ConvGeom g;
  int K, J;
  __device__ __forceinline__ T get(int, int k, int j) const {
    if (k >= K || j >= J) return T(0);
    int s = k % g.KW, t = k / g.KW, r = t % g.KH, c = t / g.KH;
    int wo = j % g.WO, t2 = j / g.WO, ho = t2 % g.HO, n = t2 / g.HO;
    int ih = ho * g.SH - g.PH + r, iw = wo * g.SW - g.PW + s;
    if (ih < 0 || ih >= g.H || iw < 0 || iw >= g.W) return T(0);
    return load_as<T>(x, dt, (((int64_t)n * g.C + c) * g.H + ih) * g.W + iw);
  }
};

// dgrad A[c][k=(f,r,s)] = w[f, c, r, s]
template <typename T>
struct DgradA {
  const void* w;
  int dt;
  ConvGeom g;
  int K;
  __device__ __forceinline__ T get(int, int c, int k) const {
    if (c >= g.C || k >= K) return T(0);
    int s = k % g.KW, t = k / g.KW, r = t % g.KH, f = t / g.KH;
    return load_as<T>(w, dt, (((int64_t)f * g.C + c) * g.KH + r) * g.KW + s);
  }
};

// dgrad B[k=(f,r,s)][j=(n,ih,iw)] = g[n, f, ho, wo] where ih = ho*sh - ph + r
template <typename T>
struct DgradB {
  const void* gr;
  int dt;
  ConvGeom g;
  int K, J;
  __device__ __forceinline__ T get(int, int k, int j) const {
    if (k >= K || j >= J) return T(0);
    int s = k % g.KW, t = k / g.KW, r = t % g.KH, f = t / g.KH;
    int iw = j % g.W, t2 = j / g.W, ih = t2 % g.H, n = t2 / g.H;
    int hn = ih + g.PH - r, wn = iw + g.PW - s;
    if (hn < 0 || wn < 0 || hn % g.SH || wn % g.SW) return T(0);
    int ho = hn / g.SH, wo = wn / g.SW;
    if (ho >= g.HO || wo >= g.WO) return T(0);
    return load_as<T>(gr, dt, (((int64_t)n * g.F + f) * g.HO + ho) * g.WO + wo);
  }
};

// wgrad A[f][k=(n,p)] = g[n, f, p]
template <typename T>
struct WgradA {
  const void* gr;
  int dt;
  ConvGeom g;
  int K;
  __device__ __forceinline__ T get(int, int f, int k) const {
    if (f >= g.F || k >= K) return T(0);
    int P = g.HO * g.WO;
    int p = k % P, n = k / P;
    return load_as<T>(gr, dt, ((int64_t)n * g.F + f) * P + p);
  }
};

// wgrad B[k=(n,ho,wo)][j=(c,r,s)] = x[n, c, ho*sh-ph+r, wo*sw-pw+s]
template <typename T>
struct WgradB {
  const void* x;
  int dt;
  ConvGeom g;
  int K, J;
  __device__ __forceinline__ T get(int, int k, int j) const {
    if (k >= K || j >= J) return T(0);
    int s = j % g.KW, t = j / g.KW, r = t % g.KH, c = t / g.KH;
    int wo = k % g.WO, t2 = k / g.WO, ho = t2 % g.HO, n = t2 / g.HO;
    int ih = ho * g.SH - g.PH + r, iw = wo * g.SW - g.PW + s;
    if (ih < 0 || ih >= g.H || iw < 0 || iw >= g.W) return T(0);
    return load_as<T>(x, dt, (((int64_t)n * g.C + c) * g.H + ih) * g.W + iw);
  }
};

// epilogues
template <typename T>
struct StoreMat {  // C[b][m][n] contiguous, runtime dtype
  void* p;
  int dt;
  int M, N;
  __device__ __forceinline__ void put(int b, int m, int n, T v) const {
    if (m < M && n < N) store_from<T>(p, dt, ((int64_t)b * M + m) * N + n, v);
  }
};

template <typename T>
struct StoreConv {  // rows = channel (F for fprop, C for dgrad), cols = (n, pixel)
  void* p;
  int dt;
  int rows, cols, P;  // P = pixels per image
  const void* bias;   // nullable
  int bdt;
  __device__ __forceinline__ void put(int, int m, int j, T v) const {
    if (m >= rows || j >= cols) return;
    int n = j / P, q = j - n * P;
    if (bias) v = (T)(v + load_as<T>(bias, bdt, m));
    store_from<T>(p, dt, ((int64_t)n * rows + m) * P + q, v);
  }
};

template <typename T>
struct StorePartial {  // ws[split][m][n] in the accumulation type
  T* ws;
  int M, N;
  __device__ __forceinline__ void put(int split, int m, int n, T v) const {
    if (m < M && n < N) ws[((int64_t)split * M + m) * N + n] = v;
  }
};

// C[M,N] (+)= A[M,K] B[K,N]; blockIdx.z = batch (or K split), K range [k0, k1)
template <typename T, class LA, class LB, class ST>
__global__ void __launch_bounds__(256) gemm_kernel(LA la, LB lb, ST st, int M, int N, int K, int ksplit) {
  __shared__ T As[BK][BM + 4];
  __shared__ T Bs[BK][BN + 4];
  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int z = blockIdx.z;
  int batch = z, split = 0;
  int k0 = 0, k1 = K;
  if (ksplit > 1) {
    batch = 0;
    split = z;
    int per = ((K + ksplit - 1) / ksplit + BK - 1) / BK * BK;
    k0 = split * per;
    k1 = min(K, k0 + per);
  }
  typedef typename AccOf<T>::type A;
  A acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = A(0);

  for (int kk = k0; kk < k1; kk += BK) {
    // A tile: 128 x 16, thread -> (k = tid % 16, m = tid / 16 + 16 i)
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      int k = tid % 16, m = tid / 16 + 16 * i;
      int kg = kk + k;
      As[k][m] = kg < k1 ? la.get(batch, m0 + m, kg) : T(0);
    }
    // B tile: 16 x 128, thread -> (n = tid % 128, k = tid / 128 + 2 i)
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      int n = tid % 128, k = tid / 128 + 2 * i;
      int kg = kk + k;
      Bs[k][n] = kg < k1 ? lb.get(batch, kg, n0 + n) : T(0);
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < BK; ++k) {
      T a[TM], b[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) a[i] = As[k][ty * TM + i];
#pragma unroll
      for (int j = 0; j < TN; ++j) b[j] = Bs[k][tx * TN + j];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] += (A)a[i] * (A)b[j];
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) st.put(ksplit > 1 ? split : batch, m0 + ty * TM + i, n0 + tx * TN + j, acc[i][j]);
}

// fold K-split partials in split order and store
template <typename T>
__global__ void fold_kernel(const T* ws, int splits, int64_t MN, void* out, int dt) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < MN; i += (int64_t)gridDim.x * blockDim.x) {
    T v = ws[i];
    for (int s = 1; s < splits; ++s) v += ws[(int64_t)s * MN + i];
    store_from<T>(out, dt, i, v);
  }
}

static ConvGeom geom(const pb_tensor* x_or_shape, const pb_tensor* w_or_shape, const pb_conv* p, const int64_t* xs,
                     const int64_t* ws) {
  (void)x_or_shape;
  (void)w_or_shape;
  ConvGeom g;
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

template <typename T, class LA, class LB, class ST>
static int launch(LA la, LB lb, ST st, int M, int N, int K, int batch) {
  dim3 grid((N + BN - 1) / BN, (M + BM - 1) / BM, batch);
  gemm_kernel<T><<<grid, 256, 0, compute_stream()>>>(la, lb, st, M, N, K, 1);
  PB_LAUNCHED();
  return PB_OK;
}

template <typename T>
static int matmul_t(const pb_tensor* a, const pb_tensor* b, const pb_tensor* out) {
  int r3 = a->ndim == 3;
  int batch = r3 ? (int)a->shape[0] : 1;
  int M = (int)a->shape[r3], K = (int)a->shape[r3 + 1], N = (int)b->shape[r3 + 1];
  MatA<T> la{(const void*)(uintptr_t)a->ptr, a->dtype, r3 ? a->strides[0] : 0, a->strides[r3], a->strides[r3 + 1], M, K};
  MatA<T> lb{(const void*)(uintptr_t)b->ptr, b->dtype, r3 ? b->strides[0] : 0, b->strides[r3], b->strides[r3 + 1], K, N};
  StoreMat<typename AccOf<T>::type> st{(void*)(uintptr_t)out->ptr, out->dtype, M, N};
  if ((int64_t)M * N * batch == 0) return PB_OK;
  if (K == 0) {
    pb_scalar z = {1, 0, 0.0, 0};
    return pb_fill(out, &z);
  }
  return launch<T>(la, lb, st, M, N, K, batch);
}

}  // namespace pb

using namespace pb;

extern "C" int pb_matmul_simt(const pb_tensor* a, const pb_tensor* b, const pb_tensor* out) {
  // numpy semantics (kernels.py:166-173): an f32 result is computed in f64 unless both
  // operands are f32 (then f32 products accumulate in f64 here, 3xTF32 on the tensor cores).
  int dt = out->dtype;
  if (dt == PB_F32 && a->dtype == PB_F32 && b->dtype == PB_F32) return matmul_t<float>(a, b, out);
  if (dt == PB_F32 || dt == PB_F64) return matmul_t<double>(a, b, out);
  switch (dt) {
    case PB_I64: return matmul_t<int64_t>(a, b, out);
    case PB_I32: return matmul_t<int32_t>(a, b, out);
    case PB_U8: return matmul_t<uint8_t>(a, b, out);
  }
  return fail(PB_ERR_UNSUPPORTED, "pb_matmul: unsupported dtype");
}

template <typename T>
static int conv_fprop_t(const pb_tensor* x, const pb_tensor* w, const pb_tensor* bias, const pb_conv* p,
                        const pb_tensor* out) {
  ConvGeom g = geom(x, w, p, x->shape, w->shape);
  int M = g.F, K = g.C * g.KH * g.KW, J = g.N * g.HO * g.WO;
  MatA<T> la{(const void*)(uintptr_t)w->ptr, w->dtype, 0, (int64_t)K, 1, M, K};
  FpropB<T> lb{(const void*)(uintptr_t)x->ptr, x->dtype, g, K, J};
  StoreConv<typename AccOf<T>::type> st{(void*)(uintptr_t)out->ptr, out->dtype, g.F, J, g.HO * g.WO,
                  bias ? (const void*)(uintptr_t)bias->ptr : nullptr, bias ? bias->dtype : 0};
  if ((int64_t)M * J == 0) return PB_OK;
  return launch<T>(la, lb, st, M, J, K, 1);
}

template <typename T>
static int conv_dgrad_t(const pb_tensor* gr, const pb_tensor* w, const pb_conv* p, const pb_tensor* out) {
  ConvGeom g = geom(out, w, p, out->shape, w->shape);
  int M = g.C, K = g.F * g.KH * g.KW, J = g.N * g.H * g.W;
  DgradA<T> la{(const void*)(uintptr_t)w->ptr, w->dtype, g, K};
  DgradB<T> lb{(const void*)(uintptr_t)gr->ptr, gr->dtype, g, K, J};
  StoreConv<typename AccOf<T>::type> st{(void*)(uintptr_t)out->ptr, out->dtype, g.C, J, g.H * g.W, nullptr, 0};
  if ((int64_t)M * J == 0) return PB_OK;
  return launch<T>(la, lb, st, M, J, K, 1);
}

template <typename T>
static int conv_wgrad_t(const pb_tensor* x, const pb_tensor* gr, const pb_conv* p, const pb_tensor* out) {
  ConvGeom g = geom(x, out, p, x->shape, out->shape);
  int M = g.F, J = g.C * g.KH * g.KW, K = g.N * g.HO * g.WO;
  if ((int64_t)M * J == 0) return PB_OK;
  WgradA<T> la{(const void*)(uintptr_t)gr->ptr, gr->dtype, g, K};
  WgradB<T> lb{(const void*)(uintptr_t)x->ptr, x->dtype, g, K, J};
  int tiles = ((M + BM - 1) / BM) * ((J + BN - 1) / BN);
  int splits = (num_sms() * 2 + tiles - 1) / tiles;
  int max_splits = (K + 255) / 256;
  if (splits > max_splits) splits = max_splits;
  if (splits < 1) splits = 1;
  if (splits == 1) {
    StoreMat<typename AccOf<T>::type> st{(void*)(uintptr_t)out->ptr, out->dtype, M, J};
    return launch<T>(la, lb, st, M, J, K, 1);
  }
  typedef typename AccOf<T>::type A;
  A* ws = (A*)workspace(sizeof(A) * (size_t)splits * M * J);
  if (!ws) return fail(PB_ERR_OOM, "conv2d_grad_weight: no workspace");
  StorePartial<A> st{ws, M, J};
  dim3 grid((J + BN - 1) / BN, (M + BM - 1) / BM, splits);
  gemm_kernel<T><<<grid, 256, 0, compute_stream()>>>(la, lb, st, M, J, K, splits);
  PB_LAUNCHED();
  fold_kernel<A><<<grid_for((int64_t)M * J, 256), 256, 0, compute_stream()>>>(ws, splits, (int64_t)M * J,
                                                                              (void*)(uintptr_t)out->ptr, out->dtype);
  PB_LAUNCHED();
  return PB_OK;
}

static bool all_f32(const pb_tensor* a, const pb_tensor* b, const pb_tensor* c) {
  return a->dtype == PB_F32 && b->dtype == PB_F32 && (!c || c->dtype == PB_F32);
}

extern "C" int pb_conv2d_simt(const pb_tensor* x, const pb_tensor* w, const pb_tensor* bias, const pb_conv* p,
                              const pb_tensor* out) {
  if (!is_contiguous(*x) || !is_contiguous(*w)) return fail(PB_ERR_ARG, "pb_conv2d: operands must be contiguous");
  if (out->dtype == PB_F32 && all_f32(x, w, bias)) return conv_fprop_t<float>(x, w, bias, p, out);
  if (out->dtype == PB_F32 || out->dtype == PB_F64) return conv_fprop_t<double>(x, w, bias, p, out);
  if (out->dtype == PB_I64) return conv_fprop_t<int64_t>(x, w, bias, p, out);
  if (out->dtype == PB_I32) return conv_fprop_t<int32_t>(x, w, bias, p, out);
  return fail(PB_ERR_UNSUPPORTED, "pb_conv2d: unsupported dtype");
}

extern "C" int pb_conv2d_grad_input_simt(const pb_tensor* g, const pb_tensor* w, const pb_conv* p, const pb_tensor* out) {
  if (!is_contiguous(*g) || !is_contiguous(*w)) return fail(PB_ERR_ARG, "pb_conv2d_grad_input: operands must be contiguous");
  if (out->dtype == PB_F32 && all_f32(g, w, nullptr)) return conv_dgrad_t<float>(g, w, p, out);
  if (out->dtype == PB_F32 || out->dtype == PB_F64) return conv_dgrad_t<double>(g, w, p, out);
  if (out->dtype == PB_I64) return conv_dgrad_t<int64_t>(g, w, p, out);
  if (out->dtype == PB_I32) return conv_dgrad_t<int32_t>(g, w, p, out);
  return fail(PB_ERR_UNSUPPORTED, "pb_conv2d_grad_input: unsupported dtype");
}

extern "C" int pb_conv2d_grad_weight_simt(const pb_tensor* x, const pb_tensor* g, const pb_conv* p, const pb_tensor* out) {
  if (!is_contiguous(*g) || !is_contiguous(*x)) return fail(PB_ERR_ARG, "pb_conv2d_grad_weight: operands must be contiguous");
  if (out->dtype == PB_F32 && all_f32(x, g, nullptr)) return conv_wgrad_t<float>(x, g, p, out);
  if (out->dtype == PB_F32 || out->dtype == PB_F64) return conv_wgrad_t<double>(x, g, p, out);
  if (out->dtype == PB_I64) return conv_wgrad_t<int64_t>(x, g, p, out);
  if (out->dtype == PB_I32) return conv_wgrad_t<int32_t>(x, g, p, out);
  return fail(PB_ERR_UNSUPPORTED, "pb_conv2d_grad_weight: unsupported dtype");
}

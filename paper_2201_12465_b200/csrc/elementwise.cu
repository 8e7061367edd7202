// Elementwise primitives: broadcast binary ops, unary ops, casts, strided copies
// (reshape / transpose / slice / concat materialisation), pad, fill, arange, checks,
// and the fused multi-tensor SGD update.  Semantics: minml/kernels.py:25-129, 245-269.
//
// Numerics: every op computes in numpy's result type `CT` (chosen on the host), is
// compiled with -fmad=false, and uses IEEE-rounded division/sqrt, so + - * / sqrt and
// all integer/bool/compare/movement ops are bit-exact against numpy; transcendental ops
// use CUDA's libm (<= 2 ulp).
//
// Kernels (all HBM-bound; algorithmic bytes = sum of operand + output bytes):
//   ew_vec   contiguous operands (or a scalar), 16-byte vector loads/stores, grid-stride
//            sized to SMs*resident blocks.
//   ew_rows  any strides: the innermost axis is walked with unit steps per thread
//            (coalesced when it is contiguous), outer axes are decomposed once per tile.
#include <cuda_runtime.h>
#include <stdint.h>
#include <type_traits>
#include <vector>
#include <cstring>
#include <cstdlib>
#include <cuda.h>
#include <dlfcn.h>
#include <mutex>
#include <string>
#include <unordered_map>
#include "common.cuh"

namespace pb {

// ---------------------------------------------------------------------------- operators
template <typename T> __device__ __forceinline__ bool isnan_(T) { return false; }
template <> __device__ __forceinline__ bool isnan_(float v) { return v != v; }
template <> __device__ __forceinline__ bool isnan_(double v) { return v != v; }

template <typename T>
__device__ __forceinline__ T ipow(T base, T e) {
  T r = 1;
  while (e > 0) {
    if (e & 1) r = (T)(r * base);
    base = (T)(base * base);
    e >>= 1;
  }
  return r;
}
__device__ __forceinline__ float pow_(float a, float b) { return powf(a, b); }
__device__ __forceinline__ double pow_(double a, double b) { return pow(a, b); }
__device__ __forceinline__ int32_t pow_(int32_t a, int32_t b) { return ipow<int32_t>(a, b); }
__device__ __forceinline__ int64_t pow_(int64_t a, int64_t b) { return ipow<int64_t>(a, b); }
__device__ __forceinline__ uint8_t pow_(uint8_t a, uint8_t b) { return (uint8_t)ipow<uint32_t>(a, b); }
__device__ __forceinline__ bool pow_(bool a, bool b) { return a || !b; }

template <int OP, typename T>
struct Bin;
#define PB_BIN(OPC, R, EXPR)                                                  \
  template <typename T>                                                       \
  struct Bin<OPC, T> {                                                        \
    typedef R res;                                                            \
    __device__ __forceinline__ static R f(T a, T b) { return EXPR; }         \
  };
PB_BIN(PB_ADD, T, (T)(a + b))
PB_BIN(PB_SUB, T, (T)(a - b))
PB_BIN(PB_MUL, T, (T)(a * b))
PB_BIN(PB_DIV, T, (T)(a / b))
PB_BIN(PB_POW, T, pow_(a, b))
PB_BIN(PB_MIN, T, (isnan_(a) || a <= b) ? a : b)
PB_BIN(PB_MAX, T, (isnan_(a) || a >= b) ? a : b)
PB_BIN(PB_EQ, bool, a == b)
PB_BIN(PB_LT, bool, a < b)
PB_BIN(PB_GT, bool, a > b)
PB_BIN(PB_AND, bool, (bool)a && (bool)b)
PB_BIN(PB_OR, bool, (bool)a || (bool)b)
#undef PB_BIN

// a / b correctly rounded, given r = RN(1/b) (Markstein: q = RN(a*r) is within one ulp of
// a/b, the residual a - q*b is exact with one FMA, and RN(q + residual*r) is RN(a/b)).  The
// theorem needs every intermediate normal: operands outside [2^-60, 2^60] (zeros, subnormals,
// inf, NaN included) take the IEEE division instead.  Checked bit for bit against IEEE
// division in tests/test_gpu_ops.py::test_fast_division_is_ieee_exact.
__device__ __forceinline__ float div_rn_rcp(float a, float b, float r) {
  const float aa = fabsf(a), ab = fabsf(b);
  if (ab >= 0x1p-60f && ab <= 0x1p60f) {
    if (aa >= 0x1p-60f && aa <= 0x1p60f) {
      const float q = __fmul_rn(a, r);
      const float e = __fmaf_rn(-q, b, a);
      return __fmaf_rn(e, r, q);
    }
    if (a == 0.f) return __int_as_float((__float_as_int(a) ^ __float_as_int(b)) & (int)0x80000000);
  }
  return a / b;
}

// IEEE a / b for every input: a normal-range divisor takes its IEEE reciprocal and div_rn_rcp (a
// zero dividend gives the signed zero directly), anything else the hardware division.  The
// hardware sequence's fast-path check (FCHK) sends zero dividends -- half of a ReLU-masked
// gradient -- to its slow subroutine; this path never calls it for them.
__device__ __forceinline__ float div_ieee(float a, float b) {
  const float ab = fabsf(b);
  if (ab >= 0x1p-60f && ab <= 0x1p60f) return div_rn_rcp(a, b, __frcp_rn(b));
  return a / b;
}

template <>
struct Bin<PB_DIV, float> {
  typedef float res;
  __device__ __forceinline__ static float f(float a, float b) { return div_ieee(a, b); }
};

template <typename T> __device__ __forceinline__ T neg_(T v) { return (T)(-v); }
template <> __device__ __forceinline__ bool neg_(bool v) { return v; }
template <typename T> __device__ __forceinline__ T abs_(T v) { return v < 0 ? (T)(-v) : v; }
template <> __device__ __forceinline__ float abs_(float v) { return fabsf(v); }
template <> __device__ __forceinline__ double abs_(double v) { return fabs(v); }
template <> __device__ __forceinline__ uint8_t abs_(uint8_t v) { return v; }
template <> __device__ __forceinline__ bool abs_(bool v) { return v; }

template <typename T> __device__ __forceinline__ T fexp(T v) { return (T)exp((double)v); }
__device__ __forceinline__ float fexp(float v) { return expf(v); }
template <typename T> __device__ __forceinline__ T flog(T v) { return (T)log((double)v); }
__device__ __forceinline__ float flog(float v) { return logf(v); }
template <typename T> __device__ __forceinline__ T fsqrt(T v) { return (T)sqrt((double)v); }
__device__ __forceinline__ float fsqrt(float v) { return sqrtf(v); }
template <typename T> __device__ __forceinline__ T fsin(T v) { return (T)sin((double)v); }
__device__ __forceinline__ float fsin(float v) { return sinf(v); }
template <typename T> __device__ __forceinline__ T fcos(T v) { return (T)cos((double)v); }
__device__ __forceinline__ float fcos(float v) { return cosf(v); }
template <typename T> __device__ __forceinline__ T ftanh(T v) { return (T)tanh((double)v); }
__device__ __forceinline__ float ftanh(float v) { return tanhf(v); }

template <int OP, typename T>
struct Un {
  typedef T res;
  __device__ __forceinline__ static T f(T v) {
    switch (OP) {
      case PB_NEG: return neg_(v);
      case PB_ABS: return abs_(v);
      case PB_EXP: return fexp(v);
      case PB_LOG: return flog(v);
      case PB_SQRT: return fsqrt(v);
      case PB_SIN: return fsin(v);
      case PB_COS: return fcos(v);
      case PB_TANH: return ftanh(v);
      case PB_NOT: return (T)(!(bool)v);
      default: return v;  // PB_CAST: value already converted by load_as
    }
  }
};

// ------------------------------------------------------------------------ vector path
template <typename T> struct Vec { static const int N = 16 / sizeof(T); };

template <typename T, int N>
struct alignas(16) Pack {
  T v[N];
};
template <typename R, int N>
struct alignas(sizeof(R) * N >= 16 ? 16 : sizeof(R) * N) OutPack {
  R v[N];
};

// binary: a/b either full arrays (mode 0) or a scalar (mode 1); out contiguous
template <int OP, typename T, typename R, int AM, int BM>
__global__ void __launch_bounds__(256) ew_vec_bin(const T* __restrict__ a, const T* __restrict__ b, T sa, T sb,
                                                  R* __restrict__ out, int64_t n) {
  const int N = Vec<T>::N;
  int64_t nv = n / N;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += stride) {
    Pack<T, N> pa, pb_;
    if (AM == 0) pa = reinterpret_cast<const Pack<T, N>*>(a)[i];
    if (BM == 0) pb_ = reinterpret_cast<const Pack<T, N>*>(b)[i];
    OutPack<R, N> o;
#pragma unroll
    for (int k = 0; k < N; ++k) {
      T x = AM == 0 ? pa.v[k] : sa;
      T y = BM == 0 ? pb_.v[k] : sb;
      o.v[k] = cvt<R>(Bin<OP, T>::f(x, y));
    }
    *reinterpret_cast<OutPack<R, N>*>(out + i * N) = o;
  }
  for (int64_t i = nv * N + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    T x = AM == 0 ? a[i] : sa;
    T y = BM == 0 ? b[i] : sb;
    out[i] = cvt<R>(Bin<OP, T>::f(x, y));
  }
}

template <int OP, typename T, typename R>
__global__ void __launch_bounds__(256) ew_vec_un(const T* __restrict__ a, R* __restrict__ out, int64_t n) {
  const int N = Vec<T>::N;
  int64_t nv = n / N;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += stride) {
    Pack<T, N> pa = reinterpret_cast<const Pack<T, N>*>(a)[i];
    OutPack<R, N> o;
#pragma unroll
    for (int k = 0; k < N; ++k) o.v[k] = cvt<R>(Un<OP, T>::f(pa.v[k]));
    *reinterpret_cast<OutPack<R, N>*>(out + i * N) = o;
  }
  for (int64_t i = nv * N + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = cvt<R>(Un<OP, T>::f(a[i]));
}

// -------------------------------------------------------------------------- rows path
struct RowArgs {
  const void* a;
  const void* b;
  void* out;
  int dta, dtb, dto;
  Dims d;         // coalesced; st[0]=a, st[1]=b, st[2]=out
  int64_t inner;  // extent of the last axis
  int64_t rows;
  int64_t tiles;  // tiles per row
};

static const int kRowTile = 2048;

template <typename F>
__device__ __forceinline__ void row_walk(const RowArgs& r, F&& body) {
  const int nd = r.d.ndim;
  for (int64_t t = blockIdx.x; t < r.rows * r.tiles; t += gridDim.x) {
    int64_t row = t / r.tiles;
    int64_t c0 = (t - row * r.tiles) * kRowTile;
    int64_t oa = 0, ob = 0, oo = 0;
    if (r.rows <= 0x7fffffff) {
      uint32_t rr = (uint32_t)row;
      for (int k = nd - 2; k >= 0; --k) {
        uint32_t ext = (uint32_t)r.d.shape[k];
        uint32_t q = rr / ext;
        int64_t idx = rr - q * ext;
        rr = q;
        oa += idx * r.d.st[0][k];
        ob += idx * r.d.st[1][k];
        oo += idx * r.d.st[2][k];
      }
    } else {
      int64_t rr = row;
      for (int k = nd - 2; k >= 0; --k) {
        int64_t ext = r.d.shape[k];
        int64_t idx = rr % ext;
        rr /= ext;
        oa += idx * r.d.st[0][k];
        ob += idx * r.d.st[1][k];
        oo += idx * r.d.st[2][k];
      }
    }
    const int64_t sa = r.d.st[0][nd - 1], sb = r.d.st[1][nd - 1], so = r.d.st[2][nd - 1];
    int64_t cend = c0 + kRowTile < r.inner ? c0 + kRowTile : r.inner;
    for (int64_t c = c0 + threadIdx.x; c < cend; c += blockDim.x) body(oa + c * sa, ob + c * sb, oo + c * so);
  }
}

template <int OP, typename CT>
__global__ void __launch_bounds__(256) ew_rows_bin(RowArgs r, CT sa, CT sb, int am, int bm) {
  typedef typename Bin<OP, CT>::res R;
  row_walk(r, [&](int64_t ia, int64_t ib, int64_t io) {
    CT x = am ? sa : load_as<CT>(r.a, r.dta, ia);
    CT y = bm ? sb : load_as<CT>(r.b, r.dtb, ib);
    store_from<R>(r.out, r.dto, io, Bin<OP, CT>::f(x, y));
  });
}

template <int OP, typename CT>
__global__ void __launch_bounds__(256) ew_rows_un(RowArgs r) {
  row_walk(r, [&](int64_t ia, int64_t, int64_t io) {
    store_from<CT>(r.out, r.dto, io, Un<OP, CT>::f(load_as<CT>(r.a, r.dta, ia)));
  });
}


// ------------------------------------------------------------------ f32 broadcast path
// f32 operands (or a scalar) with any broadcast strides over <= 4 coalesced axes into a
// contiguous output.  The reference's hot broadcasts (BatchNorm's per-channel centre /
// scale, the sum-backward spreads g[n,c,1,1] * ones, bias adds) all land here.
// ew_bc4: inner extent % 4 == 0 and every tensor operand's inner stride is 1 (16-byte
//         vector) or 0 (one value per row): 4 float4 per thread, all loads issued first.
// ew_bc1: anything else: 8 scalars per thread, each decomposed with FastDiv.
struct BcArgs {
  const float* a;
  const float* b;
  void* out;
  int nd;               // coalesced rank, 1..4 (axis nd-1 innermost)
  FastDiv ext[4];       // extents
  int64_t sa[4], sb[4]; // element strides
  uint32_t n;           // elements (ew_bc1) or float4s (ew_bc4)
  int va, vb;           // ew_bc4: inner stride 1 (else 0)
};

__device__ __forceinline__ void bc_offsets(const BcArgs& p, uint32_t e, int64_t& oa, int64_t& ob) {
  oa = 0;
  ob = 0;
#pragma unroll
  for (int k = 3; k >= 0; --k) {
    if (k < p.nd) {
      uint32_t q, r;
      if (k > 0) {
        p.ext[k].divmod(e, q, r);
      } else {
        q = 0;
        r = e;
      }
      oa += (int64_t)r * p.sa[k];
      ob += (int64_t)r * p.sb[k];
      e = q;
    }
  }
}

template <typename R> struct Out4 { typedef float4 type; };
template <> struct Out4<bool> { typedef uchar4 type; };
__device__ __forceinline__ float4 mk4(float a, float b, float c, float d) { return make_float4(a, b, c, d); }
__device__ __forceinline__ uchar4 mk4(bool a, bool b, bool c, bool d) { return make_uchar4(a, b, c, d); }

template <int OP, int AM, int BM>
__global__ void __launch_bounds__(256) ew_bc4(BcArgs p, float sa, float sb) {
  typedef typename Bin<OP, float>::res R;
  typedef typename Out4<R>::type O4;
  const uint32_t step = gridDim.x * 1024u;
  for (uint32_t base = blockIdx.x * 1024u + threadIdx.x; base < p.n; base += step) {
    float4 xa[4], xb[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      uint32_t v = base + u * 256u;
      xa[u] = make_float4(sa, sa, sa, sa);
      xb[u] = make_float4(sb, sb, sb, sb);
      if (v < p.n) {
        int64_t oa, ob;
        bc_offsets(p, v * 4u, oa, ob);
        if (!AM) {
          if (p.va) xa[u] = __ldg(reinterpret_cast<const float4*>(p.a + oa));
          else { float t = __ldg(p.a + oa); xa[u] = make_float4(t, t, t, t); }
        }
        if (!BM) {
          if (p.vb) xb[u] = __ldg(reinterpret_cast<const float4*>(p.b + ob));
          else { float t = __ldg(p.b + ob); xb[u] = make_float4(t, t, t, t); }
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      uint32_t v = base + u * 256u;
      if (v < p.n)
        reinterpret_cast<O4*>(p.out)[v] = mk4(Bin<OP, float>::f(xa[u].x, xb[u].x), Bin<OP, float>::f(xa[u].y, xb[u].y),
                                              Bin<OP, float>::f(xa[u].z, xb[u].z), Bin<OP, float>::f(xa[u].w, xb[u].w));
    }
  }
}

template <int OP, int AM, int BM>
__global__ void __launch_bounds__(256) ew_bc1(BcArgs p, float sa, float sb) {
  typedef typename Bin<OP, float>::res R;
  const uint32_t step = gridDim.x * 2048u;
  for (uint32_t base = blockIdx.x * 2048u + threadIdx.x; base < p.n; base += step) {
    float xa[8], xb[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      uint32_t e = base + u * 256u;
      xa[u] = sa;
      xb[u] = sb;
      if (e < p.n) {
        int64_t oa, ob;
        bc_offsets(p, e, oa, ob);
        if (!AM) xa[u] = __ldg(p.a + oa);
        if (!BM) xb[u] = __ldg(p.b + ob);
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      uint32_t e = base + u * 256u;
      if (e < p.n) reinterpret_cast<R*>(p.out)[e] = Bin<OP, float>::f(xa[u], xb[u]);
    }
  }
}


// ------------------------------------------------ per-row broadcast (BatchNorm's pattern)
// out[e] = op(D[e], R[row(e)]) or op(R[row(e)], D[e]) where D is dense in the output's own
// layout and R holds one value per output row (inner stride 0): x - mean, x / std, x * gamma,
// x + beta over [N,C,H,W] with [1,C,1,1] operands.  All index math is 32-bit: one FastDiv for
// the row of each float4, up to three more for R's offset.  A row-broadcast divisor gets its
// IEEE reciprocal once per float4 and each quotient one exact-residual correction
// (div_rn_rcp), which is the correctly rounded a / b.
struct ChanArgs {
  const float* d;
  const float* r;
  void* out;
  uint32_t n4;        // float4s in the output
  FastDiv row_len;    // inner (row) extent, % 4 == 0
  int nouter;         // outer coalesced axes (<= 3)
  FastDiv ext[3];     // their extents, outermost first
  uint32_t rs[3];     // R's element strides along them
};

template <int OP, int RLEFT>
__global__ void __launch_bounds__(256) ew_chan4(ChanArgs p) {
  typedef typename Bin<OP, float>::res R;
  typedef typename Out4<R>::type O4;
  const uint32_t step = gridDim.x * 1024u;
  for (uint32_t base = blockIdx.x * 1024u + threadIdx.x; base < p.n4; base += step) {
    float4 xd[4];
    float xr[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t v = base + u * 256u;
      xd[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      xr[u] = 1.f;
      if (v < p.n4) {
        uint32_t row = p.row_len.div(v * 4u), off = 0;
#pragma unroll
        for (int k = 2; k >= 0; --k) {
          if (k < p.nouter) {
            uint32_t q, rr;
            p.ext[k].divmod(row, q, rr);
            off += rr * p.rs[k];
            row = q;
          }
        }
        xd[u] = __ldg(reinterpret_cast<const float4*>(p.d) + v);
        xr[u] = __ldg(p.r + off);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t v = base + u * 256u;
      if (v >= p.n4) continue;
      const float4 a = xd[u];
      const float b = xr[u];
      if (OP == PB_DIV && !RLEFT) {
        const float rc = __frcp_rn(b);
        reinterpret_cast<float4*>(p.out)[v] =
            make_float4(div_rn_rcp(a.x, b, rc), div_rn_rcp(a.y, b, rc), div_rn_rcp(a.z, b, rc), div_rn_rcp(a.w, b, rc));
      } else if (RLEFT) {
        reinterpret_cast<O4*>(p.out)[v] = mk4(Bin<OP, float>::f(b, a.x), Bin<OP, float>::f(b, a.y),
                                              Bin<OP, float>::f(b, a.z), Bin<OP, float>::f(b, a.w));
      } else {
        reinterpret_cast<O4*>(p.out)[v] = mk4(Bin<OP, float>::f(a.x, b), Bin<OP, float>::f(a.y, b),
                                              Bin<OP, float>::f(a.z, b), Bin<OP, float>::f(a.w, b));
      }
    }
  }
}

// exact-division probe for the tests: out[i] = div_ieee(a[i], b[i]) (div_rn_rcp behind it)
__global__ void fastdiv_probe(const float* a, const float* b, float* out, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = div_ieee(a[i], b[i]);
}

// ------------------------------------------------------------- fused elementwise chains
// Backend-internal fusion (the rule of minml/deferred.py:146-163 restated for
// the GPU): the backend defers f32/bool elementwise primitives and runs a whole linear
// chain  v = head;  v = op_k(v, operand_k) (or op_k(operand_k, v))  in one pass, reading
// each leaf once with broadcast strides and writing only the chain's result.  Every step
// applies the same Bin / Un functor the unfused kernels use, in f32 (bools as 0/1), so a
// fused chain is bit-identical to running its primitives one by one.
static const int kChainLeaves = 8;
static const int kChainSteps = 16;
static const int kChainTaps = 4;

struct ChainStep {
  int16_t op;    // pb_binop, or 64 + pb_unop (PB_CAST: to the step's bool flag)
  int8_t kind;   // 0 unary, 1 leaf, 2 scalar, 3 self (v op v)
  int8_t side;   // binary: 0 -> op(v, x), 1 -> op(x, v)
  int8_t leaf;
  int8_t to_bool;  // cast target (unary PB_CAST)
  float scalar;
};

struct ChainArgs {
  const void* leaf[kChainLeaves];
  int8_t is_bool[kChainLeaves];
  int8_t vec[kChainLeaves];    // chain4: inner stride 1 (else 0)
  int8_t dense[kChainLeaves];  // chain4x: same strides as the (dense) output: offset = index
  int nleaves, nsteps, head_kind;  // head_kind 0: leaf 0, 1: scalar
  float head_scalar;
  ChainStep step[kChainSteps];
  void* out;
  int out_bool;
  int nd;
  FastDiv ext[4];
  int64_t st[kChainLeaves][4];
  uint32_t n;
  // taps (JIT only): after tap_after[i] steps, v is also stored to tap[i] (dense f32, out's shape)
  int ntaps;
  int8_t tap_after[kChainTaps];
  void* tap[kChainTaps];
};

template <int NL>
__device__ __forceinline__ void chain_offsets(const ChainArgs& p, uint32_t e, int64_t* off) {
#pragma unroll
  for (int l = 0; l < NL; ++l) off[l] = 0;
#pragma unroll
  for (int k = 3; k >= 0; --k) {
    if (k < p.nd) {
      uint32_t q, r;
      if (k > 0) {
        p.ext[k].divmod(e, q, r);
      } else {
        q = 0;
        r = e;
      }
#pragma unroll
      for (int l = 0; l < NL; ++l) off[l] += (int64_t)r * p.st[l][k];
      e = q;
    }
  }
}

__device__ __forceinline__ float4 chain_load4(const ChainArgs& p, int l, int64_t off) {
  if (p.is_bool[l]) {
    const uint8_t* b = (const uint8_t*)p.leaf[l] + off;
    if (p.vec[l]) {
      uchar4 u = *reinterpret_cast<const uchar4*>(b);
      return make_float4(u.x ? 1.f : 0.f, u.y ? 1.f : 0.f, u.z ? 1.f : 0.f, u.w ? 1.f : 0.f);
    }
    float t = *b ? 1.f : 0.f;
    return make_float4(t, t, t, t);
  }
  const float* f = (const float*)p.leaf[l] + off;
  if (p.vec[l]) return __ldg(reinterpret_cast<const float4*>(f));
  float t = __ldg(f);
  return make_float4(t, t, t, t);
}

#define PB_LANES4(...)        \
  {                           \
    float a_ = v.x, b_ = o.x; \
    v.x = __VA_ARGS__;        \
    a_ = v.y;                 \
    b_ = o.y;                 \
    v.y = __VA_ARGS__;        \
    a_ = v.z;                 \
    b_ = o.z;                 \
    v.z = __VA_ARGS__;        \
    a_ = v.w;                 \
    b_ = o.w;                 \
    v.w = __VA_ARGS__;        \
    (void)b_;                 \
  }

// one step on 4 lanes; the (warp-uniform) switch is taken once per step, not per lane
__device__ __forceinline__ float4 chain_step4(const ChainStep& st, float4 v, float4 o) {
  if (st.kind == 0) {
    const int op = st.op - 64;
    switch (op) {
      case PB_NEG: PB_LANES4(Un<PB_NEG, float>::f(a_)) break;
      case PB_ABS: PB_LANES4(Un<PB_ABS, float>::f(a_)) break;
      case PB_EXP: PB_LANES4(Un<PB_EXP, float>::f(a_)) break;
      case PB_LOG: PB_LANES4(Un<PB_LOG, float>::f(a_)) break;
      case PB_SQRT: PB_LANES4(Un<PB_SQRT, float>::f(a_)) break;
      case PB_SIN: PB_LANES4(Un<PB_SIN, float>::f(a_)) break;
      case PB_COS: PB_LANES4(Un<PB_COS, float>::f(a_)) break;
      case PB_TANH: PB_LANES4(Un<PB_TANH, float>::f(a_)) break;
      case PB_NOT: PB_LANES4(a_ == 0.f ? 1.f : 0.f) break;
      default:
        if (st.to_bool) PB_LANES4(a_ != 0.f ? 1.f : 0.f)
        break;
    }
    (void)o;
    return v;
  }
  if (st.side) {
    float4 t = v;
    v = o;
    o = t;
  }
  switch (st.op) {
    case PB_ADD: PB_LANES4(Bin<PB_ADD, float>::f(a_, b_)) break;
    case PB_SUB: PB_LANES4(Bin<PB_SUB, float>::f(a_, b_)) break;
    case PB_MUL: PB_LANES4(Bin<PB_MUL, float>::f(a_, b_)) break;
    case PB_DIV: PB_LANES4(Bin<PB_DIV, float>::f(a_, b_)) break;
    case PB_POW: PB_LANES4(Bin<PB_POW, float>::f(a_, b_)) break;
    case PB_MIN: PB_LANES4(Bin<PB_MIN, float>::f(a_, b_)) break;
    case PB_MAX: PB_LANES4(Bin<PB_MAX, float>::f(a_, b_)) break;
    case PB_EQ: PB_LANES4(a_ == b_ ? 1.f : 0.f) break;
    case PB_LT: PB_LANES4(a_ < b_ ? 1.f : 0.f) break;
    case PB_GT: PB_LANES4(a_ > b_ ? 1.f : 0.f) break;
    case PB_AND: PB_LANES4((a_ != 0.f && b_ != 0.f) ? 1.f : 0.f) break;
    default: PB_LANES4((a_ != 0.f || b_ != 0.f) ? 1.f : 0.f) break;
  }
  return v;
}
#undef PB_LANES4

// 4 output elements per thread-iteration (inner extent % 4 == 0, leaves unit- or zero-stride
// inside); NL = number of leaves, so offsets and leaf values stay in registers
// leaf values live in eight named registers: selecting one per step with a compare chain
// (an array here is turned into a local-memory table indexed by st.leaf)
template <int NL, typename V>
__device__ __forceinline__ V pick(int l, const V& x0, const V& x1, const V& x2, const V& x3, const V& x4,
                                  const V& x5, const V& x6, const V& x7) {
  V o = x0;
  if (NL > 1 && l == 1) o = x1;
  if (NL > 2 && l == 2) o = x2;
  if (NL > 3 && l == 3) o = x3;
  if (NL > 4 && l == 4) o = x4;
  if (NL > 5 && l == 5) o = x5;
  if (NL > 6 && l == 6) o = x6;
  if (NL > 7 && l == 7) o = x7;
  return o;
}

// 4 output elements per thread-iteration (inner extent % 4 == 0, leaves unit- or zero-stride
// inside); NL = number of leaves, so offsets and leaf values stay in registers
template <int NL>
__global__ void __launch_bounds__(256) ew_chain4(ChainArgs p) {
  const uint32_t step = gridDim.x * blockDim.x;
  const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
  for (uint32_t v4 = blockIdx.x * blockDim.x + threadIdx.x; v4 < p.n; v4 += step) {
    int64_t off[NL];
    chain_offsets<NL>(p, v4 * 4u, off);
    float4 x0 = chain_load4(p, 0, off[0]);
    float4 x1 = NL > 1 ? chain_load4(p, 1, off[NL > 1 ? 1 : 0]) : z;
    float4 x2 = NL > 2 ? chain_load4(p, 2, off[NL > 2 ? 2 : 0]) : z;
    float4 x3 = NL > 3 ? chain_load4(p, 3, off[NL > 3 ? 3 : 0]) : z;
    float4 x4 = NL > 4 ? chain_load4(p, 4, off[NL > 4 ? 4 : 0]) : z;
    float4 x5 = NL > 5 ? chain_load4(p, 5, off[NL > 5 ? 5 : 0]) : z;
    float4 x6 = NL > 6 ? chain_load4(p, 6, off[NL > 6 ? 6 : 0]) : z;
    float4 x7 = NL > 7 ? chain_load4(p, 7, off[NL > 7 ? 7 : 0]) : z;
    float4 v = p.head_kind == 0 ? x0 : make_float4(p.head_scalar, p.head_scalar, p.head_scalar, p.head_scalar);
    for (int s = 0; s < p.nsteps; ++s) {
      const ChainStep st = p.step[s];
      float4 o = v;
      if (st.kind == 1) o = pick<NL>(st.leaf, x0, x1, x2, x3, x4, x5, x6, x7);
      else if (st.kind == 2) o = make_float4(st.scalar, st.scalar, st.scalar, st.scalar);
      v = chain_step4(st, v, o);
    }
    if (p.out_bool)
      reinterpret_cast<uchar4*>(p.out)[v4] = make_uchar4(v.x != 0.f, v.y != 0.f, v.z != 0.f, v.w != 0.f);
    else
      reinterpret_cast<float4*>(p.out)[v4] = v;
  }
}

// 8 outputs per thread-iteration (inner extent % 8 == 0): the per-step dispatch (step fetch,
// operand select, op switch) is paid once per 8 elements instead of 4
struct F8 {
  float4 a, b;
};
#define PB_L1(C, ...)  \
  {                     \
    float a_ = v.C;     \
    float b_ = o.C;     \
    v.C = __VA_ARGS__;  \
    (void)b_;           \
  }
#define PB_LANES8(...)                                                                          \
  {                                                                                             \
    PB_L1(a.x, __VA_ARGS__) PB_L1(a.y, __VA_ARGS__) PB_L1(a.z, __VA_ARGS__) PB_L1(a.w, __VA_ARGS__) \
    PB_L1(b.x, __VA_ARGS__) PB_L1(b.y, __VA_ARGS__) PB_L1(b.z, __VA_ARGS__) PB_L1(b.w, __VA_ARGS__) \
  }
__device__ __forceinline__ F8 chain_step8(const ChainStep& st, F8 v, F8 o) {
  if (st.kind == 0) {
    const int op = st.op - 64;
    switch (op) {
      case PB_NEG: PB_LANES8(Un<PB_NEG, float>::f(a_)) break;
      case PB_ABS: PB_LANES8(Un<PB_ABS, float>::f(a_)) break;
      case PB_EXP: PB_LANES8(Un<PB_EXP, float>::f(a_)) break;
      case PB_LOG: PB_LANES8(Un<PB_LOG, float>::f(a_)) break;
      case PB_SQRT: PB_LANES8(Un<PB_SQRT, float>::f(a_)) break;
      case PB_SIN: PB_LANES8(Un<PB_SIN, float>::f(a_)) break;
      case PB_COS: PB_LANES8(Un<PB_COS, float>::f(a_)) break;
      case PB_TANH: PB_LANES8(Un<PB_TANH, float>::f(a_)) break;
      case PB_NOT: PB_LANES8(a_ == 0.f ? 1.f : 0.f) break;
      default:
        if (st.to_bool) PB_LANES8(a_ != 0.f ? 1.f : 0.f)
        break;
    }
    return v;
  }
  if (st.side) {
    F8 t = v;
    v = o;
    o = t;
  }
  switch (st.op) {
    case PB_ADD: PB_LANES8(Bin<PB_ADD, float>::f(a_, b_)) break;
    case PB_SUB: PB_LANES8(Bin<PB_SUB, float>::f(a_, b_)) break;
    case PB_MUL: PB_LANES8(Bin<PB_MUL, float>::f(a_, b_)) break;
    case PB_DIV: PB_LANES8(Bin<PB_DIV, float>::f(a_, b_)) break;
    case PB_POW: PB_LANES8(Bin<PB_POW, float>::f(a_, b_)) break;
    case PB_MIN: PB_LANES8(Bin<PB_MIN, float>::f(a_, b_)) break;
    case PB_MAX: PB_LANES8(Bin<PB_MAX, float>::f(a_, b_)) break;
    case PB_EQ: PB_LANES8(a_ == b_ ? 1.f : 0.f) break;
    case PB_LT: PB_LANES8(a_ < b_ ? 1.f : 0.f) break;
    case PB_GT: PB_LANES8(a_ > b_ ? 1.f : 0.f) break;
    case PB_AND: PB_LANES8((a_ != 0.f && b_ != 0.f) ? 1.f : 0.f) break;
    default: PB_LANES8((a_ != 0.f || b_ != 0.f) ? 1.f : 0.f) break;
  }
  return v;
}
#undef PB_LANES8
#undef PB_L1

__device__ __forceinline__ F8 chain_load8(const ChainArgs& p, int l, int64_t off) {
  F8 r;
  if (p.vec[l]) {
    r.a = chain_load4(p, l, off);
    r.b = chain_load4(p, l, off + 4);
  } else {
    r.a = chain_load4(p, l, off);
    r.b = r.a;
  }
  return r;
}

template <int NL>
__global__ void __launch_bounds__(256) ew_chain8(ChainArgs p) {
  const uint32_t step = gridDim.x * blockDim.x;
  F8 z;
  z.a = z.b = make_float4(0.f, 0.f, 0.f, 0.f);
  for (uint32_t v8 = blockIdx.x * blockDim.x + threadIdx.x; v8 < p.n; v8 += step) {
    int64_t off[NL];
    chain_offsets<NL>(p, v8 * 8u, off);
    F8 x0 = chain_load8(p, 0, off[0]);
    F8 x1 = NL > 1 ? chain_load8(p, 1, off[NL > 1 ? 1 : 0]) : z;
    F8 x2 = NL > 2 ? chain_load8(p, 2, off[NL > 2 ? 2 : 0]) : z;
    F8 x3 = NL > 3 ? chain_load8(p, 3, off[NL > 3 ? 3 : 0]) : z;
    F8 x4 = NL > 4 ? chain_load8(p, 4, off[NL > 4 ? 4 : 0]) : z;
    F8 x5 = NL > 5 ? chain_load8(p, 5, off[NL > 5 ? 5 : 0]) : z;
    F8 x6 = NL > 6 ? chain_load8(p, 6, off[NL > 6 ? 6 : 0]) : z;
    F8 x7 = NL > 7 ? chain_load8(p, 7, off[NL > 7 ? 7 : 0]) : z;
    F8 v;
    if (p.head_kind == 0) {
      v = x0;
    } else {
      v.a = v.b = make_float4(p.head_scalar, p.head_scalar, p.head_scalar, p.head_scalar);
    }
    for (int s = 0; s < p.nsteps; ++s) {
      const ChainStep st = p.step[s];
      F8 o = v;
      if (st.kind == 1) {
        o = pick<NL>(st.leaf, x0, x1, x2, x3, x4, x5, x6, x7);
      } else if (st.kind == 2) {
        o.a = o.b = make_float4(st.scalar, st.scalar, st.scalar, st.scalar);
      }
      v = chain_step8(st, v, o);
    }
    if (p.out_bool) {
      uchar4* ob = reinterpret_cast<uchar4*>(p.out) + 2 * v8;
      ob[0] = make_uchar4(v.a.x != 0.f, v.a.y != 0.f, v.a.z != 0.f, v.a.w != 0.f);
      ob[1] = make_uchar4(v.b.x != 0.f, v.b.y != 0.f, v.b.z != 0.f, v.b.w != 0.f);
    } else {
      float4* of = reinterpret_cast<float4*>(p.out) + 2 * v8;
      of[0] = v.a;
      of[1] = v.b;
    }
  }
}

__device__ __forceinline__ float chain_load1(const ChainArgs& p, int l, int64_t off) {
  return p.is_bool[l] ? (((const uint8_t*)p.leaf[l])[off] ? 1.f : 0.f) : __ldg((const float*)p.leaf[l] + off);
}

// one element per thread-iteration, any strides
template <int NL>
__global__ void __launch_bounds__(256) ew_chain1(ChainArgs p) {
  const uint32_t step = gridDim.x * blockDim.x;
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < p.n; e += step) {
    int64_t off[NL];
    chain_offsets<NL>(p, e, off);
    float x0 = chain_load1(p, 0, off[0]);
    float x1 = NL > 1 ? chain_load1(p, 1, off[NL > 1 ? 1 : 0]) : 0.f;
    float x2 = NL > 2 ? chain_load1(p, 2, off[NL > 2 ? 2 : 0]) : 0.f;
    float x3 = NL > 3 ? chain_load1(p, 3, off[NL > 3 ? 3 : 0]) : 0.f;
    float x4 = NL > 4 ? chain_load1(p, 4, off[NL > 4 ? 4 : 0]) : 0.f;
    float x5 = NL > 5 ? chain_load1(p, 5, off[NL > 5 ? 5 : 0]) : 0.f;
    float x6 = NL > 6 ? chain_load1(p, 6, off[NL > 6 ? 6 : 0]) : 0.f;
    float x7 = NL > 7 ? chain_load1(p, 7, off[NL > 7 ? 7 : 0]) : 0.f;
    float v = p.head_kind == 0 ? x0 : p.head_scalar;
    for (int s = 0; s < p.nsteps; ++s) {
      const ChainStep st = p.step[s];
      float o = v;
      if (st.kind == 1) o = pick<NL>(st.leaf, x0, x1, x2, x3, x4, x5, x6, x7);
      else if (st.kind == 2) o = st.scalar;
      float4 r = chain_step4(st, make_float4(v, v, v, v), make_float4(o, o, o, o));
      v = r.x;
    }
    if (p.out_bool)
      ((uint8_t*)p.out)[e] = v != 0.f;
    else
      ((float*)p.out)[e] = v;
  }
}

// 4 consecutive outputs per thread-iteration when rows are not a multiple of 4 (7x7 maps):
// dense leaves load 16 bytes at the output index, the others decode each element's offset
__device__ __forceinline__ float4 chain_load4x(const ChainArgs& p, int l, uint32_t e0) {
  if (p.dense[l]) {
    if (p.is_bool[l]) {
      uchar4 u = *reinterpret_cast<const uchar4*>((const uint8_t*)p.leaf[l] + e0);
      return make_float4(u.x ? 1.f : 0.f, u.y ? 1.f : 0.f, u.z ? 1.f : 0.f, u.w ? 1.f : 0.f);
    }
    return __ldg(reinterpret_cast<const float4*>((const float*)p.leaf[l] + e0));
  }
  float v[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    uint32_t e = e0 + u;
    int64_t off = 0;
#pragma unroll
    for (int k = 3; k >= 0; --k) {
      if (k < p.nd) {
        uint32_t q, r;
        if (k > 0) {
          p.ext[k].divmod(e, q, r);
        } else {
          q = 0;
          r = e;
        }
        off += (int64_t)r * p.st[l][k];
        e = q;
      }
    }
    v[u] = chain_load1(p, l, off);
  }
  return make_float4(v[0], v[1], v[2], v[3]);
}

template <int NL>
__global__ void __launch_bounds__(256) ew_chain4x(ChainArgs p) {
  const uint32_t step = gridDim.x * blockDim.x;
  const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
  for (uint32_t v4 = blockIdx.x * blockDim.x + threadIdx.x; v4 < p.n; v4 += step) {
    const uint32_t e0 = v4 * 4u;
    float4 x0 = chain_load4x(p, 0, e0);
    float4 x1 = NL > 1 ? chain_load4x(p, 1, e0) : z;
    float4 x2 = NL > 2 ? chain_load4x(p, 2, e0) : z;
    float4 x3 = NL > 3 ? chain_load4x(p, 3, e0) : z;
    float4 x4 = NL > 4 ? chain_load4x(p, 4, e0) : z;
    float4 x5 = NL > 5 ? chain_load4x(p, 5, e0) : z;
    float4 x6 = NL > 6 ? chain_load4x(p, 6, e0) : z;
    float4 x7 = NL > 7 ? chain_load4x(p, 7, e0) : z;
    float4 v = p.head_kind == 0 ? x0 : make_float4(p.head_scalar, p.head_scalar, p.head_scalar, p.head_scalar);
    for (int s = 0; s < p.nsteps; ++s) {
      const ChainStep st = p.step[s];
      float4 o = v;
      if (st.kind == 1) o = pick<NL>(st.leaf, x0, x1, x2, x3, x4, x5, x6, x7);
      else if (st.kind == 2) o = make_float4(st.scalar, st.scalar, st.scalar, st.scalar);
      v = chain_step4(st, v, o);
    }
    if (p.out_bool)
      reinterpret_cast<uchar4*>(p.out)[v4] = make_uchar4(v.x != 0.f, v.y != 0.f, v.z != 0.f, v.w != 0.f);
    else
      reinterpret_cast<float4*>(p.out)[v4] = v;
  }
}

template <int NL>
static void launch_chain(ChainArgs& p, int mode, cudaStream_t s) {
  if (mode == 3) ew_chain8<NL><<<grid_for(p.n, 256, 1), 256, 0, s>>>(p);
  else if (mode == 1) ew_chain4<NL><<<grid_for(p.n, 256, 2), 256, 0, s>>>(p);
  else if (mode == 2) ew_chain4x<NL><<<grid_for(p.n, 256, 2), 256, 0, s>>>(p);
  else ew_chain1<NL><<<grid_for(p.n, 256, 4), 256, 0, s>>>(p);
}


// windowed leaves (round 2): the reference scatters a slice's gradient back with zero-stuffing
// pads (minml/autograd.py:667-693, the maxpool backward's 9 windows) and reads strided windows
// of a -inf-padded input in the maxpool forward.  A windowed leaf reads its source through a
// per-axis affine map instead of a materialised pad: for output index i, j = i*mul - off; the
// element is src[j / div] when j >= 0, j % div == 0 and j / div < ext (the source extent), else
// the fill value.  One thread per output element decodes its 4-D index.
struct WinLeaf {
  int32_t mul[4], off[4], shift[4], ext[4];  // div = 1 << shift (the host declines other divisors)
  float fill;
  int on;
};
struct WinArgs {
  ChainArgs c;       // leaves, steps, output (c.st: broadcast strides of the plain leaves, 4-D)
  WinLeaf w[kChainLeaves];
  FastDiv d1, d2, d3;  // output extents of axes 1..3
};

// leaf l at 4 consecutive positions i3 .. i3+3 of the innermost axis: the outer axes' part of
// the window test and offset is computed once per group
__device__ __forceinline__ float4 win_load4(const WinArgs& a, int l, const uint32_t* idx) {
  const ChainArgs& p = a.c;
  const WinLeaf& w = a.w[l];
  float v[4];
  if (w.on) {
    int64_t off = 0;
    bool ok = true;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const int j = (int)idx[d] * w.mul[d] - w.off[d];
      const int q = j >> w.shift[d];
      ok = ok && j >= 0 && !(j & ((1 << w.shift[d]) - 1)) && q < w.ext[d];
      off += (int64_t)q * p.st[l][d];
    }
    const int m3 = (1 << w.shift[3]) - 1;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = (int)(idx[3] + u) * w.mul[3] - w.off[3];
      const int q = j >> w.shift[3];
      if (ok && j >= 0 && !(j & m3) && q < w.ext[3]) {
        const int64_t o = off + (int64_t)q * p.st[l][3];
        v[u] = p.is_bool[l] ? (((const uint8_t*)p.leaf[l])[o] ? 1.f : 0.f) : __ldg((const float*)p.leaf[l] + o);
      } else {
        v[u] = w.fill;
      }
    }
  } else {
    int64_t off = 0;
#pragma unroll
    for (int d = 0; d < 3; ++d) off += (int64_t)idx[d] * p.st[l][d];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t o = off + (int64_t)(idx[3] + u) * p.st[l][3];
      v[u] = p.is_bool[l] ? (((const uint8_t*)p.leaf[l])[o] ? 1.f : 0.f) : __ldg((const float*)p.leaf[l] + o);
    }
  }
  return make_float4(v[0], v[1], v[2], v[3]);
}

__device__ __forceinline__ float win_load1(const WinArgs& a, int l, const uint32_t* idx) {
  const ChainArgs& p = a.c;
  const WinLeaf& w = a.w[l];
  int64_t off = 0;
  if (w.on) {
#pragma unroll
    for (int d = 0; d < 4; ++d) {
      const int j = (int)idx[d] * w.mul[d] - w.off[d];
      if (j < 0 || (j & ((1 << w.shift[d]) - 1))) return w.fill;
      const int q = j >> w.shift[d];
      if (q >= w.ext[d]) return w.fill;
      off += (int64_t)q * p.st[l][d];
    }
  } else {
#pragma unroll
    for (int d = 0; d < 4; ++d) off += (int64_t)idx[d] * p.st[l][d];
  }
  return p.is_bool[l] ? (((const uint8_t*)p.leaf[l])[off] ? 1.f : 0.f) : __ldg((const float*)p.leaf[l] + off);
}

// one output per thread-iteration (inner extents that are not a multiple of 4)
template <int NL>
__global__ void __launch_bounds__(256) ew_chain_win1(WinArgs a) {
  const ChainArgs& p = a.c;
  const uint32_t step = gridDim.x * blockDim.x;
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < p.n; e += step) {
    uint32_t idx[4], q;
    a.d3.divmod(e, q, idx[3]);
    a.d2.divmod(q, q, idx[2]);
    a.d1.divmod(q, idx[0], idx[1]);
    const float x0 = win_load1(a, 0, idx);
    const float x1 = NL > 1 ? win_load1(a, NL > 1 ? 1 : 0, idx) : 0.f;
    const float x2 = NL > 2 ? win_load1(a, NL > 2 ? 2 : 0, idx) : 0.f;
    const float x3 = NL > 3 ? win_load1(a, NL > 3 ? 3 : 0, idx) : 0.f;
    const float x4 = NL > 4 ? win_load1(a, NL > 4 ? 4 : 0, idx) : 0.f;
    const float x5 = NL > 5 ? win_load1(a, NL > 5 ? 5 : 0, idx) : 0.f;
    const float x6 = NL > 6 ? win_load1(a, NL > 6 ? 6 : 0, idx) : 0.f;
    const float x7 = NL > 7 ? win_load1(a, NL > 7 ? 7 : 0, idx) : 0.f;
    float v = p.head_kind == 0 ? x0 : p.head_scalar;
    for (int s = 0; s < p.nsteps; ++s) {
      const ChainStep st = p.step[s];
      float o = v;
      if (st.kind == 1) o = pick<NL>(st.leaf, x0, x1, x2, x3, x4, x5, x6, x7);
      else if (st.kind == 2) o = st.scalar;
      const float4 r = chain_step4(st, make_float4(v, v, v, v), make_float4(o, o, o, o));
      v = r.x;
    }
    if (p.out_bool)
      ((uint8_t*)p.out)[e] = v != 0.f;
    else
      ((float*)p.out)[e] = v;
  }
}

// 4 consecutive outputs along the innermost axis per thread-iteration (its extent % 4 == 0)
template <int NL>
__global__ void __launch_bounds__(256) ew_chain_win(WinArgs a) {
  const ChainArgs& p = a.c;
  const uint32_t step = gridDim.x * blockDim.x;
  const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
  for (uint32_t g = blockIdx.x * blockDim.x + threadIdx.x; g < p.n; g += step) {
    const uint32_t e = g * 4u;
    uint32_t idx[4], q;
    a.d3.divmod(e, q, idx[3]);
    a.d2.divmod(q, q, idx[2]);
    a.d1.divmod(q, idx[0], idx[1]);
    const float4 x0 = win_load4(a, 0, idx);
    const float4 x1 = NL > 1 ? win_load4(a, NL > 1 ? 1 : 0, idx) : z;
    const float4 x2 = NL > 2 ? win_load4(a, NL > 2 ? 2 : 0, idx) : z;
    const float4 x3 = NL > 3 ? win_load4(a, NL > 3 ? 3 : 0, idx) : z;
    const float4 x4 = NL > 4 ? win_load4(a, NL > 4 ? 4 : 0, idx) : z;
    const float4 x5 = NL > 5 ? win_load4(a, NL > 5 ? 5 : 0, idx) : z;
    const float4 x6 = NL > 6 ? win_load4(a, NL > 6 ? 6 : 0, idx) : z;
    const float4 x7 = NL > 7 ? win_load4(a, NL > 7 ? 7 : 0, idx) : z;
    float4 v = p.head_kind == 0 ? x0 : make_float4(p.head_scalar, p.head_scalar, p.head_scalar, p.head_scalar);
    for (int s = 0; s < p.nsteps; ++s) {
      const ChainStep st = p.step[s];
      float4 o = v;
      if (st.kind == 1) o = pick<NL>(st.leaf, x0, x1, x2, x3, x4, x5, x6, x7);
      else if (st.kind == 2) o = make_float4(st.scalar, st.scalar, st.scalar, st.scalar);
      v = chain_step4(st, v, o);
    }
    if (p.out_bool)
      reinterpret_cast<uchar4*>(p.out)[g] = make_uchar4(v.x != 0.f, v.y != 0.f, v.z != 0.f, v.w != 0.f);
    else
      reinterpret_cast<float4*>(p.out)[g] = v;
  }
}


// ------------------------------------------------------------ JIT-specialised chain kernels
// The interpreted chain kernels dispatch every step through a switch: ~68 instructions per
// element for a 3-step chain (ncu: issue-bound at 2.4 IPC, DRAM 41%).  A chain's structure --
// rank, vector width, leaf kinds, the op sequence -- is fixed per call site, so it is compiled
// once with NVRTC (dlopen'd; -fmad=false, the same libdevice and IEEE division as this file) into
// a straight-line kernel and cached by its source text.  Scalars and pointers stay parameters,
// so every instance of a structure shares one kernel.  The functors below are the exact
// expressions of Bin / Un / div_ieee above: results are bit-identical to the interpreter
// (tests/test_gpu_fusion.py).  Disabled with PB_CHAIN_JIT=0, and on any NVRTC failure.
struct JFD {
  uint32_t d, m, s;
};
struct JArgs {
  const void* leaf[kChainLeaves];
  int64_t st[kChainLeaves][4];
  JFD ext[4];
  float sc[kChainSteps];
  float head;
  void* out;
  uint32_t n;
  int pad_;
  void* tap[kChainTaps];
};

static const char* kJitPrelude = R"JIT(
typedef unsigned int uint32_t; typedef long long int64_t; typedef unsigned char uint8_t;
struct JFD { uint32_t d, m, s; };
struct JArgs {
  const void* leaf[8];
  int64_t st[8][4];
  JFD ext[4];
  float sc[16];
  float head;
  void* out;
  uint32_t n;
  int pad_;
  void* tap[4];
};
__device__ __forceinline__ void jdm(const JFD& f, uint32_t n, uint32_t& q, uint32_t& r) {
  q = (__umulhi(n, f.m) + n) >> f.s; r = n - q * f.d;
}
__device__ __forceinline__ float jrcpdiv(float a, float b, float r) {
  const float aa = fabsf(a), ab = fabsf(b);
  if (ab >= 0x1p-60f && ab <= 0x1p60f) {
    if (aa >= 0x1p-60f && aa <= 0x1p60f) {
      const float q = __fmul_rn(a, r);
      const float e = __fmaf_rn(-q, b, a);
      return __fmaf_rn(e, r, q);
    }
    if (a == 0.f) return __int_as_float((__float_as_int(a) ^ __float_as_int(b)) & (int)0x80000000);
  }
  return a / b;
}
__device__ __forceinline__ float jdiv(float a, float b) {
  const float ab = fabsf(b);
  if (ab >= 0x1p-60f && ab <= 0x1p60f) return jrcpdiv(a, b, __frcp_rn(b));
  return a / b;
}
__device__ __forceinline__ float jmin(float a, float b) { return ((a != a) || a <= b) ? a : b; }
__device__ __forceinline__ float jmax(float a, float b) { return ((a != a) || a >= b) ? a : b; }
)JIT";

typedef int (*NvrtcCreate)(void**, const char*, const char*, int, const char* const*, const char* const*);
typedef int (*NvrtcCompile)(void*, int, const char* const*);
typedef int (*NvrtcGetSize)(void*, size_t*);
typedef int (*NvrtcGet)(void*, char*);
typedef int (*NvrtcDestroy)(void**);
typedef CUresult (*CuModuleLoadData)(CUmodule*, const void*);
typedef CUresult (*CuModuleGetFunction)(CUfunction*, CUmodule, const char*);
typedef CUresult (*CuLaunchKernel)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned,
                                   CUstream, void**, void**);
typedef CUresult (*CuOccupancy)(int*, CUfunction, int, size_t);

struct Jit {
  bool ok = false;
  NvrtcCreate create = nullptr;
  NvrtcCompile compile = nullptr;
  NvrtcGetSize cubin_size = nullptr, log_size = nullptr;
  NvrtcGet cubin = nullptr, log = nullptr;
  NvrtcDestroy destroy = nullptr;
  CuModuleLoadData load = nullptr;
  CuModuleGetFunction getfn = nullptr;
  CuLaunchKernel launch = nullptr;
  CuOccupancy occupancy = nullptr;
  std::mutex mu;
  std::unordered_map<std::string, CUfunction> cache;
  std::unordered_map<CUfunction, int> resident;  // 256-thread blocks per SM
};

static Jit& jit() {
  static Jit* j = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    j = new Jit();
    const char* e = getenv("PB_CHAIN_JIT");
    if (e && e[0] == '0') return;
    void* h = dlopen("libnvrtc.so.12", RTLD_NOW | RTLD_LOCAL);
    if (!h) h = dlopen("/usr/local/cuda/lib64/libnvrtc.so.12", RTLD_NOW | RTLD_LOCAL);
    if (!h) return;
    j->create = (NvrtcCreate)dlsym(h, "nvrtcCreateProgram");
    j->compile = (NvrtcCompile)dlsym(h, "nvrtcCompileProgram");
    j->cubin_size = (NvrtcGetSize)dlsym(h, "nvrtcGetCUBINSize");
    j->cubin = (NvrtcGet)dlsym(h, "nvrtcGetCUBIN");
    j->log_size = (NvrtcGetSize)dlsym(h, "nvrtcGetProgramLogSize");
    j->log = (NvrtcGet)dlsym(h, "nvrtcGetProgramLog");
    j->destroy = (NvrtcDestroy)dlsym(h, "nvrtcDestroyProgram");
    void *f1 = nullptr, *f2 = nullptr, *f3 = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuModuleLoadData", &f1, cudaEnableDefault, &q) != cudaSuccess ||
        cudaGetDriverEntryPoint("cuModuleGetFunction", &f2, cudaEnableDefault, &q) != cudaSuccess ||
        cudaGetDriverEntryPoint("cuLaunchKernel", &f3, cudaEnableDefault, &q) != cudaSuccess)
      return;
    j->load = (CuModuleLoadData)f1;
    j->getfn = (CuModuleGetFunction)f2;
    j->launch = (CuLaunchKernel)f3;
    void* f4 = nullptr;
    if (cudaGetDriverEntryPoint("cuOccupancyMaxActiveBlocksPerMultiprocessor", &f4, cudaEnableDefault, &q) ==
        cudaSuccess)
      j->occupancy = (CuOccupancy)f4;
    j->ok = j->create && j->compile && j->cubin_size && j->cubin && j->destroy && j->load && j->getfn && j->launch;
  });
  return *j;
}

static const char* jit_bin(int op) {
  switch (op) {
    case PB_ADD: return "(a+b)";
    case PB_SUB: return "(a-b)";
    case PB_MUL: return "(a*b)";
    case PB_DIV: return "jdiv(a,b)";
    case PB_POW: return "powf(a,b)";
    case PB_MIN: return "jmin(a,b)";
    case PB_MAX: return "jmax(a,b)";
    case PB_EQ: return "(a==b?1.f:0.f)";
    case PB_LT: return "(a<b?1.f:0.f)";
    case PB_GT: return "(a>b?1.f:0.f)";
    case PB_AND: return "((a!=0.f&&b!=0.f)?1.f:0.f)";
    default: return "((a!=0.f||b!=0.f)?1.f:0.f)";
  }
}
static const char* jit_un(int op, int to_bool) {
  switch (op) {
    case PB_NEG: return "(-a)";
    case PB_ABS: return "fabsf(a)";
    case PB_EXP: return "expf(a)";
    case PB_LOG: return "logf(a)";
    case PB_SQRT: return "sqrtf(a)";
    case PB_SIN: return "sinf(a)";
    case PB_COS: return "cosf(a)";
    case PB_TANH: return "tanhf(a)";
    case PB_NOT: return "(a==0.f?1.f:0.f)";
    default: return to_bool ? "(a!=0.f?1.f:0.f)" : "a";
  }
}

// tap stores after `after` steps: output element t*W + u of each tap is this lane's v
static void jit_taps(std::string& s, const ChainArgs& p, int after, int W) {
  for (int i = 0; i < p.ntaps; ++i) {
    if (p.tap_after[i] != after) continue;
    const std::string I = std::to_string(i);
    if (W == 4) s += "    reinterpret_cast<float4*>(p.tap[" + I + "])[t] = make_float4(v0, v1, v2, v3);\n";
    else s += "    ((float*)p.tap[" + I + "])[t] = v0;\n";
  }
}

// the kernel source for a chain structure: W = 4 (16-byte leaves along the inner axis) or 1
static std::string jit_source(const ChainArgs& p, int nleaves, int W) {
  std::string s = kJitPrelude;
  s += "extern \"C\" __global__ void __launch_bounds__(256) ew_chain_jit(JArgs p) {\n";
  s += "  const uint32_t step = gridDim.x * blockDim.x;\n";
  s += "  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < p.n; t += step) {\n";
  // 32-bit offsets when every leaf's largest offset fits (strides non-negative)
  bool small = true;
  for (int l = 0; l < nleaves && small; ++l) {
    int64_t mx = 0;
    for (int k = 0; k < p.nd; ++k) {
      if (p.st[l][k] < 0) small = false;
      mx += (int64_t)(p.ext[k].d - 1) * p.st[l][k];
    }
    small = small && mx + 4 < ((int64_t)1 << 31);
  }
  const char* ot = small ? "uint32_t" : "int64_t";
  s += "    uint32_t e = t * " + std::to_string(W) + "u, q, r;\n";
  for (int l = 0; l < nleaves; ++l) s += std::string("    ") + ot + " o" + std::to_string(l) + " = 0;\n";
  for (int k = p.nd - 1; k >= 0; --k) {
    if (k > 0) s += "    jdm(p.ext[" + std::to_string(k) + "], e, q, r);\n";
    else s += "    q = 0; r = e;\n";
    for (int l = 0; l < nleaves; ++l) {
      const std::string L = std::to_string(l);
      if (p.st[l][k] == 0) continue;
      s += "    o" + L + " += (" + ot + ")r * (" + ot + ")p.st[" + L + "][" + std::to_string(k) + "];\n";
    }
    s += "    e = q;\n";
  }
  // leaf loads: x<l>_<lane>
  for (int l = 0; l < nleaves; ++l) {
    const std::string L = std::to_string(l);
    const bool vec = W == 4 && p.vec[l];
    if (p.is_bool[l]) {
      if (vec) {
        s += "    const uchar4 b" + L + " = *reinterpret_cast<const uchar4*>((const uint8_t*)p.leaf[" + L + "] + o" + L + ");\n";
        const char* c[4] = {"x", "y", "z", "w"};
        for (int u = 0; u < 4; ++u)
          s += "    const float x" + L + "_" + std::to_string(u) + " = b" + L + "." + c[u] + " ? 1.f : 0.f;\n";
      } else {
        s += "    const float x" + L + "_0 = ((const uint8_t*)p.leaf[" + L + "])[o" + L + "] ? 1.f : 0.f;\n";
        for (int u = 1; u < W; ++u) s += "    const float x" + L + "_" + std::to_string(u) + " = x" + L + "_0;\n";
      }
    } else {
      if (vec) {
        s += "    const float4 f" + L + " = __ldg(reinterpret_cast<const float4*>((const float*)p.leaf[" + L + "] + o" + L + "));\n";
        const char* c[4] = {"x", "y", "z", "w"};
        for (int u = 0; u < 4; ++u) s += "    const float x" + L + "_" + std::to_string(u) + " = f" + L + "." + c[u] + ";\n";
      } else {
        s += "    const float x" + L + "_0 = __ldg((const float*)p.leaf[" + L + "] + o" + L + ");\n";
        for (int u = 1; u < W; ++u) s += "    const float x" + L + "_" + std::to_string(u) + " = x" + L + "_0;\n";
      }
    }
  }
  for (int u = 0; u < W; ++u) {
    const std::string U = std::to_string(u);
    s += "    float v" + U + " = " + (p.head_kind == 0 ? "x0_" + U : std::string("p.head")) + ";\n";
  }
  for (int k = 0; k < p.nsteps; ++k) {
    const ChainStep& st = p.step[k];
    // a lane-invariant divisor (a scalar or a broadcast leaf): one IEEE reciprocal per thread
    // iteration, then div_rn_rcp per lane -- the same correctly rounded quotient as jdiv
    const bool udiv = W > 1 && st.kind != 0 && st.op == PB_DIV && !st.side &&
                      (st.kind == 2 || (st.kind == 1 && !(W == 4 && p.vec[st.leaf])));
    if (udiv) {
      const std::string b = st.kind == 2 ? "p.sc[" + std::to_string(k) + "]" : "x" + std::to_string(st.leaf) + "_0";
      s += "    { const float bq = " + b + "; const float ab = fabsf(bq);\n";
      s += "      const bool inr = ab >= 0x1p-60f && ab <= 0x1p60f; const float rq = inr ? __frcp_rn(bq) : 0.f;\n";
      for (int u = 0; u < W; ++u) {
        const std::string U = std::to_string(u);
        s += "      v" + U + " = inr ? jrcpdiv(v" + U + ", bq, rq) : v" + U + " / bq;\n";
      }
      s += "    }\n";
      jit_taps(s, p, k + 1, W);
      continue;
    }
    for (int u = 0; u < W; ++u) {
      const std::string U = std::to_string(u);
      if (st.kind == 0) {
        s += std::string("    { const float a = v") + U + "; v" + U + " = " + jit_un(st.op - 64, st.to_bool) + "; }\n";
        continue;
      }
      std::string o = st.kind == 1 ? "x" + std::to_string(st.leaf) + "_" + U
                     : st.kind == 2 ? "p.sc[" + std::to_string(k) + "]" : "v" + U;
      const std::string a = st.side ? o : "v" + U, b = st.side ? "v" + U : o;
      s += "    { const float a = " + a + ", b = " + b + "; v" + U + " = " + jit_bin(st.op) + "; }\n";
    }
    jit_taps(s, p, k + 1, W);
  }
  if (W == 4) {
    if (p.out_bool)
      s += "    reinterpret_cast<uchar4*>(p.out)[t] = make_uchar4(v0 != 0.f, v1 != 0.f, v2 != 0.f, v3 != 0.f);\n";
    else
      s += "    reinterpret_cast<float4*>(p.out)[t] = make_float4(v0, v1, v2, v3);\n";
  } else {
    s += p.out_bool ? "    ((uint8_t*)p.out)[t] = v0 != 0.f;\n" : "    ((float*)p.out)[t] = v0;\n";
  }
  s += "  }\n}\n";
  return s;
}

static CUfunction jit_get(const std::string& src, const char* name = "ew_chain_jit") {
  Jit& j = jit();
  std::lock_guard<std::mutex> lk(j.mu);
  auto it = j.cache.find(src);
  if (it != j.cache.end()) return it->second;
  CUfunction fn = nullptr;
  void* prog = nullptr;
  if (j.create(&prog, src.c_str(), "pb_chain.cu", 0, nullptr, nullptr) == 0) {
    const char* opts[] = {"--gpu-architecture=sm_100a", "--fmad=false", "-std=c++17", "-default-device"};
    if (j.compile(prog, 4, opts) == 0) {
      size_t n = 0;
      if (j.cubin_size(prog, &n) == 0 && n) {
        std::string bin(n, '\0');
        CUmodule mod = nullptr;
        if (j.cubin(prog, &bin[0]) == 0 && j.load(&mod, bin.data()) == CUDA_SUCCESS) j.getfn(&fn, mod, name);
      }
    }
    j.destroy(&prog);
  }
  j.cache.emplace(src, fn);  // a failure is cached too: that structure stays interpreted
  if (fn) {
    int b = 0;
    if (!j.occupancy || j.occupancy(&b, fn, 256, 0) != CUDA_SUCCESS || b < 1) b = 4;
    j.resident[fn] = b;
  }
  return fn;
}

// one full wave of resident blocks, walked grid-stride (no partial second wave)
static unsigned jit_grid(CUfunction fn, uint32_t units) {
  int b = 4;
  {
    Jit& j = jit();
    std::lock_guard<std::mutex> lk(j.mu);
    auto it = j.resident.find(fn);
    if (it != j.resident.end()) b = it->second;
  }
  static const int waves = getenv("PB_JIT_WAVES") ? atoi(getenv("PB_JIT_WAVES")) : 1;  // experiment hook (0: no cap)
  const uint64_t need = ((uint64_t)units + 255) / 256, wave = (uint64_t)num_sms() * b * (waves > 0 ? waves : 1);
  if (waves <= 0) return (unsigned)(need ? (need < 0x7fffffffu ? need : 0x7fffffffu) : 1);
  return (unsigned)(need < wave ? (need ? need : 1) : wave);
}

// launch the JIT kernel for an interpreter-ready ChainArgs; false -> use the interpreter
static bool jit_chain(const ChainArgs& p, int mode, int nleaves, cudaStream_t s) {
  if (!jit().ok || nleaves < 1) return false;
  const int W = (mode == 1 || mode == 3) ? 4 : 1;  // chain4 / chain8 layouts: 16-byte leaves
  const std::string src = jit_source(p, nleaves, W);
  CUfunction fn = jit_get(src);
  if (!fn) return false;
  JArgs a;
  memset(&a, 0, sizeof(a));
  for (int l = 0; l < nleaves; ++l) {
    a.leaf[l] = p.leaf[l];
    for (int k = 0; k < 4; ++k) a.st[l][k] = p.st[l][k];
  }
  for (int k = 0; k < 4; ++k) a.ext[k] = JFD{p.ext[k].d, p.ext[k].m, p.ext[k].s};
  for (int k = 0; k < p.nsteps; ++k) a.sc[k] = p.step[k].scalar;
  a.head = p.head_scalar;
  a.out = p.out;
  for (int i = 0; i < p.ntaps; ++i) a.tap[i] = p.tap[i];
  // the interpreter's element counts: n/4 for chain4, n/8 (in 8s) for chain8, n for chain1 / chain4x
  uint32_t units = p.n;
  if (mode == 3) units = p.n * 2;       // chain8 counted 8-element units
  else if (mode == 2) units = p.n * 4;  // chain4x counted 4-element units of a scalar walk
  a.n = units;
  void* args[] = {&a};
  const unsigned grid = jit_grid(fn, units);
  return jit().launch(fn, grid, 1, 1, 256, 1, 1, 0, (CUstream)s, args, nullptr) == CUDA_SUCCESS;
}


// windowed chains (pb_ew_chain_win) specialised the same way: window parameters stay arguments
struct JWArgs {
  const void* leaf[kChainLeaves];
  int64_t st[kChainLeaves][4];
  JFD ext[4];
  int32_t wmul[kChainLeaves][4], woff[kChainLeaves][4], wsh[kChainLeaves][4], wext[kChainLeaves][4];
  float fill[kChainLeaves];
  float sc[kChainSteps];
  float head;
  void* out;
  uint32_t n;
  int pad_;
};
static const char* kJitWinDecl = R"JIT(
struct JWArgs {
  const void* leaf[8];
  int64_t st[8][4];
  JFD ext[4];
  int wmul[8][4], woff[8][4], wsh[8][4], wext[8][4];
  float fill[8];
  float sc[16];
  float head;
  void* out;
  uint32_t n;
  int pad_;
};
)JIT";

// ragged (W = 4 over rows whose length is not a multiple of 4 -- the maxpool backward's 114-wide
// padded planes): a thread takes 4 consecutive positions of one row, so the outer-axis window
// checks run once per 4 outputs instead of per output; positions past the row end are masked
// (ext[0] = 4-groups per row, pad_ = the row length)
static std::string jit_win_source(const WinArgs& a, int nleaves, int W, bool ragged) {
  const ChainArgs& p = a.c;
  std::string s = kJitPrelude;
  s += kJitWinDecl;
  s += "extern \"C\" __global__ void __launch_bounds__(256) ew_chain_win_jit(JWArgs p) {\n";
  s += "  const uint32_t step = gridDim.x * blockDim.x;\n";
  s += "  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < p.n; t += step) {\n";
  s += "    uint32_t q, i0, i1, i2, i3;\n";
  if (ragged) {
    s += "    uint32_t row, g;\n";
    s += "    const uint32_t inner = (uint32_t)p.pad_;\n";
    s += "    jdm(p.ext[0], t, row, g);\n";
    s += "    i3 = g * 4u;\n";
    s += "    q = row;\n";
  } else {
    s += "    jdm(p.ext[3], t * " + std::to_string(W) + "u, q, i3);\n";
  }
  s += "    jdm(p.ext[2], q, q, i2);\n";
  s += "    jdm(p.ext[1], q, i0, i1);\n";
  for (int l = 0; l < nleaves; ++l) {
    const std::string L = std::to_string(l);
    const bool isb = p.is_bool[l];
    auto ldx = [&](const std::string& off) {
      return isb ? "(((const uint8_t*)p.leaf[" + L + "])[" + off + "] ? 1.f : 0.f)"
                 : "__ldg((const float*)p.leaf[" + L + "] + " + off + ")";
    };
    if (a.w[l].on) {
      // outer axes once, then each of the W inner positions
      s += "    int64_t b" + L + " = 0; bool ok" + L + " = true;\n";
      for (int d = 0; d < 3; ++d) {
        const std::string D = std::to_string(d);
        s += "    { const int j = (int)i" + D + " * p.wmul[" + L + "][" + D + "] - p.woff[" + L + "][" + D + "];\n";
        s += "      const int qq = j >> p.wsh[" + L + "][" + D + "];\n";
        s += "      ok" + L + " = ok" + L + " && j >= 0 && !(j & ((1 << p.wsh[" + L + "][" + D + "]) - 1)) && qq < p.wext[" + L + "][" + D + "];\n";
        s += "      b" + L + " += (int64_t)qq * p.st[" + L + "][" + D + "]; }\n";
      }
      for (int u = 0; u < W; ++u) {
        const std::string U = std::to_string(u);
        s += "    float x" + L + "_" + U + " = p.fill[" + L + "];\n";
        s += "    { const int j = (int)(i3 + " + U + "u) * p.wmul[" + L + "][3] - p.woff[" + L + "][3];\n";
        s += "      const int qq = j >> p.wsh[" + L + "][3];\n";
        s += "      if (ok" + L + " && j >= 0 && !(j & ((1 << p.wsh[" + L + "][3]) - 1)) && qq < p.wext[" + L + "][3]" +
             (ragged ? " && i3 + " + U + "u < inner" : "") + ")\n";
        s += "        x" + L + "_" + U + " = " + ldx("b" + L + " + (int64_t)qq * p.st[" + L + "][3]") + "; }\n";
      }
    } else {
      s += "    const int64_t b" + L + " = (int64_t)i0 * p.st[" + L + "][0] + (int64_t)i1 * p.st[" + L + "][1] + (int64_t)i2 * p.st[" + L + "][2];\n";
      for (int u = 0; u < W; ++u) {
        const std::string U = std::to_string(u);
        const std::string ld = ldx("b" + L + " + (int64_t)(i3 + " + U + "u) * p.st[" + L + "][3]");
        s += "    const float x" + L + "_" + U + " = " + (ragged ? "i3 + " + U + "u < inner ? " + ld + " : 0.f" : ld) + ";\n";
      }
    }
  }
  for (int u = 0; u < W; ++u) {
    const std::string U = std::to_string(u);
    s += "    float v" + U + " = " + (p.head_kind == 0 ? "x0_" + U : std::string("p.head")) + ";\n";
  }
  for (int k = 0; k < p.nsteps; ++k) {
    const ChainStep& st = p.step[k];
    for (int u = 0; u < W; ++u) {
      const std::string U = std::to_string(u);
      if (st.kind == 0) {
        s += std::string("    { const float a = v") + U + "; v" + U + " = " + jit_un(st.op - 64, st.to_bool) + "; }\n";
        continue;
      }
      std::string o = st.kind == 1 ? "x" + std::to_string(st.leaf) + "_" + U
                     : st.kind == 2 ? "p.sc[" + std::to_string(k) + "]" : "v" + U;
      const std::string x = st.side ? o : "v" + U, y = st.side ? "v" + U : o;
      s += "    { const float a = " + x + ", b = " + y + "; v" + U + " = " + jit_bin(st.op) + "; }\n";
    }
  }
  if (ragged) {
    s += "    const int64_t ob = (int64_t)row * inner + i3;\n";
    for (int u = 0; u < 4; ++u) {
      const std::string U = std::to_string(u);
      s += "    if (i3 + " + U + "u < inner) " +
           (p.out_bool ? "((uint8_t*)p.out)[ob + " + U + "] = v" + U + " != 0.f;\n"
                       : "((float*)p.out)[ob + " + U + "] = v" + U + ";\n");
    }
  } else if (W == 4) {
    if (p.out_bool)
      s += "    reinterpret_cast<uchar4*>(p.out)[t] = make_uchar4(v0 != 0.f, v1 != 0.f, v2 != 0.f, v3 != 0.f);\n";
    else
      s += "    reinterpret_cast<float4*>(p.out)[t] = make_float4(v0, v1, v2, v3);\n";
  } else {
    s += p.out_bool ? "    ((uint8_t*)p.out)[t] = v0 != 0.f;\n" : "    ((float*)p.out)[t] = v0;\n";
  }
  s += "  }\n}\n";
  return s;
}

static bool jit_win(const WinArgs& a, bool vec, int nleaves, const FastDiv& d1, const FastDiv& d2,
                    const FastDiv& d3, cudaStream_t st, uint32_t inner = 0) {
  if (!jit().ok) return false;
  const bool ragged = !vec && inner >= 8;
  const int W = vec || ragged ? 4 : 1;
  const std::string src = jit_win_source(a, nleaves, W, ragged);
  CUfunction fn = jit_get(src, "ew_chain_win_jit");
  if (!fn) return false;
  const ChainArgs& p = a.c;
  JWArgs j;
  memset(&j, 0, sizeof(j));
  for (int l = 0; l < nleaves; ++l) {
    j.leaf[l] = p.leaf[l];
    j.fill[l] = a.w[l].fill;
    for (int d = 0; d < 4; ++d) {
      j.st[l][d] = p.st[l][d];
      j.wmul[l][d] = a.w[l].mul[d];
      j.woff[l][d] = a.w[l].off[d];
      j.wsh[l][d] = a.w[l].shift[d];
      j.wext[l][d] = a.w[l].ext[d];
    }
  }
  j.ext[1] = JFD{d1.d, d1.m, d1.s};
  j.ext[2] = JFD{d2.d, d2.m, d2.s};
  j.ext[3] = JFD{d3.d, d3.m, d3.s};
  for (int k = 0; k < p.nsteps; ++k) j.sc[k] = p.step[k].scalar;
  j.head = p.head_scalar;
  j.out = p.out;
  j.n = p.n;
  if (ragged) {
    const uint32_t groups = (inner + 3) / 4;
    const FastDiv gd(groups);
    j.ext[0] = JFD{gd.d, gd.m, gd.s};
    j.pad_ = (int)inner;
    j.n = p.n / inner * groups;  // (p.n = every output element here)
  }
  void* args[] = {&j};
  const unsigned grid = jit_grid(fn, j.n);
  return jit().launch(fn, grid, 1, 1, 256, 1, 1, 0, (CUstream)st, args, nullptr) == CUDA_SUCCESS;
}

// ----------------------------------------------------------------------- host helpers
static void fill_dims(Dims& d, const pb_tensor* out, const pb_tensor* a, const pb_tensor* b) {
  d.ndim = out->ndim;
  for (int k = 0; k < out->ndim; ++k) {
    d.shape[k] = out->shape[k];
    d.st[2][k] = out->strides[k];
    d.st[0][k] = 0;
    d.st[1][k] = 0;
  }
  // right-align operands; broadcast axes (extent 1) get stride 0
  const pb_tensor* ops[2] = {a, b};
  for (int o = 0; o < 2; ++o) {
    const pb_tensor* t = ops[o];
    if (!t) continue;
    int off = out->ndim - t->ndim;
    for (int k = 0; k < t->ndim; ++k) d.st[o][off + k] = (t->shape[k] == 1) ? 0 : t->strides[k];
  }
}

static RowArgs make_rows(const pb_tensor* out, const pb_tensor* a, const pb_tensor* b) {
  RowArgs r;
  r.a = a ? (const void*)(uintptr_t)a->ptr : nullptr;
  r.b = b ? (const void*)(uintptr_t)b->ptr : nullptr;
  r.out = (void*)(uintptr_t)out->ptr;
  r.dta = a ? a->dtype : 0;
  r.dtb = b ? b->dtype : 0;
  r.dto = out->dtype;
  fill_dims(r.d, out, a, b);
  coalesce(r.d, 3);
  r.inner = r.d.shape[r.d.ndim - 1];
  r.rows = 1;
  for (int k = 0; k < r.d.ndim - 1; ++k) r.rows *= r.d.shape[k];
  r.tiles = (r.inner + kRowTile - 1) / kRowTile;
  return r;
}

static int rows_grid(const RowArgs& r) {
  int64_t units = r.rows * r.tiles;
  int64_t cap = (int64_t)num_sms() * 16;
  return (int)(units < cap ? (units < 1 ? 1 : units) : cap);
}

static bool aligned16(uint64_t p) { return (p & 15) == 0; }

// full-array (same linear index as out) or scalar-like (all strides 0)
static int vec_mode(const pb_tensor* t, const pb_tensor* out) {
  if (!t) return 1;
  bool zero = true;
  for (int k = 0; k < t->ndim; ++k)
    if (t->shape[k] != 1 && t->strides[k] != 0) zero = false;
  if (zero) return 1;
  if (t->ndim != out->ndim) return -1;
  for (int k = 0; k < t->ndim; ++k)
    if (t->shape[k] != out->shape[k]) return -1;
  return is_contiguous(*t) && aligned16(t->ptr) ? 0 : -1;
}

template <typename T>
static T read_scalar_host(const pb_tensor* t, bool* ok);

template <int OP, typename T, typename R>
static int launch_vec_bin(const pb_tensor* a, const pb_tensor* b, int am, int bm, T sa, T sb, const pb_tensor* out,
                          int64_t n) {
  const T* pa = a ? (const T*)(uintptr_t)a->ptr : nullptr;
  const T* pb2 = b ? (const T*)(uintptr_t)b->ptr : nullptr;
  R* po = (R*)(uintptr_t)out->ptr;
  int grid = grid_for(n, 256, Vec<T>::N * 2);
  cudaStream_t s = compute_stream();
  if (am == 0 && bm == 0) ew_vec_bin<OP, T, R, 0, 0><<<grid, 256, 0, s>>>(pa, pb2, sa, sb, po, n);
  else if (am == 0) ew_vec_bin<OP, T, R, 0, 1><<<grid, 256, 0, s>>>(pa, pb2, sa, sb, po, n);
  else ew_vec_bin<OP, T, R, 1, 0><<<grid, 256, 0, s>>>(pa, pb2, sa, sb, po, n);
  PB_LAUNCHED();
  return PB_OK;
}


// f32 broadcast fast path; returns 1 when launched, 0 when the shape does not qualify
template <int OP>
static int try_bcast_f32(const pb_tensor* a, const pb_tensor* b, float sa, float sb, const pb_tensor* out, int* rc) {
  typedef typename Bin<OP, float>::res R;
  const int rt = std::is_same<R, bool>::value ? PB_BOOL : PB_F32;
  if (out->dtype != rt || !is_contiguous(*out) || !aligned16(out->ptr)) return 0;
  if ((a && a->dtype != PB_F32) || (b && b->dtype != PB_F32)) return 0;
  int64_t n = numel(*out);
  if (n <= 0 || n >= ((int64_t)1 << 31)) return 0;
  Dims d;
  fill_dims(d, out, a, b);
  coalesce(d, 3);
  if (d.ndim > 4) return 0;
  BcArgs p;
  p.a = a ? (const float*)(uintptr_t)a->ptr : nullptr;
  p.b = b ? (const float*)(uintptr_t)b->ptr : nullptr;
  p.out = (void*)(uintptr_t)out->ptr;
  p.nd = d.ndim;
  for (int k = 0; k < 4; ++k) {
    p.ext[k] = FastDiv(k < d.ndim ? (uint32_t)d.shape[k] : 1u);
    p.sa[k] = k < d.ndim ? d.st[0][k] : 0;
    p.sb[k] = k < d.ndim ? d.st[1][k] : 0;
  }
  const int in = d.ndim - 1;
  bool v4 = d.shape[in] % 4 == 0;
  const pb_tensor* ops[2] = {a, b};
  int vec[2] = {0, 0};
  for (int o = 0; o < 2 && v4; ++o) {
    if (!ops[o]) continue;
    int64_t is = d.st[o][in];
    if (is == 1) {
      vec[o] = 1;
      if (!aligned16(ops[o]->ptr)) v4 = false;
      for (int k = 0; k < in; ++k)
        if (d.st[o][k] % 4) v4 = false;
    } else if (is != 0) {
      v4 = false;
    }
  }
  cudaStream_t s = compute_stream();
  if (v4 && a && b && d.ndim >= 2 && d.ndim <= 4) {
    // one operand dense in the output's layout, the other constant along each row
    int dense = -1;
    for (int o = 0; o < 2; ++o) {
      bool same = true;
      int64_t acc = 1;
      for (int k = d.ndim - 1; k >= 0; --k) {
        if (d.st[o][k] != acc) same = false;
        acc *= d.shape[k];
      }
      if (same && d.st[1 - o][in] == 0) dense = o;
    }
    bool small = dense >= 0;
    for (int k = 0; small && k < in; ++k)
      if (d.st[1 - dense][k] < 0 || d.st[1 - dense][k] >= ((int64_t)1 << 30)) small = false;
    if (small) {
      ChanArgs c;
      c.d = dense == 0 ? p.a : p.b;
      c.r = dense == 0 ? p.b : p.a;
      c.out = p.out;
      c.n4 = (uint32_t)(n / 4);
      c.row_len = FastDiv((uint32_t)d.shape[in]);
      c.nouter = in;
      for (int k = 0; k < 3; ++k) {
        c.ext[k] = FastDiv(k < in ? (uint32_t)d.shape[k] : 1u);
        c.rs[k] = k < in ? (uint32_t)d.st[1 - dense][k] : 0u;
      }
      int grid = grid_for(c.n4, 1024);
      if (dense == 0) ew_chan4<OP, 0><<<grid, 256, 0, s>>>(c);
      else ew_chan4<OP, 1><<<grid, 256, 0, s>>>(c);
      count_launch();
      cudaError_t e = cudaGetLastError();
      *rc = e == cudaSuccess ? PB_OK : cuda_fail(e, "pb_binary");
      return 1;
    }
  }
  if (v4) {
    p.n = (uint32_t)(n / 4);
    p.va = vec[0];
    p.vb = vec[1];
    int grid = grid_for(p.n, 1024);
    if (a && b) ew_bc4<OP, 0, 0><<<grid, 256, 0, s>>>(p, sa, sb);
    else if (a) ew_bc4<OP, 0, 1><<<grid, 256, 0, s>>>(p, sa, sb);
    else ew_bc4<OP, 1, 0><<<grid, 256, 0, s>>>(p, sa, sb);
  } else {
    p.n = (uint32_t)n;
    p.va = p.vb = 0;
    int grid = grid_for(p.n, 2048);
    if (a && b) ew_bc1<OP, 0, 0><<<grid, 256, 0, s>>>(p, sa, sb);
    else if (a) ew_bc1<OP, 0, 1><<<grid, 256, 0, s>>>(p, sa, sb);
    else ew_bc1<OP, 1, 0><<<grid, 256, 0, s>>>(p, sa, sb);
  }
  count_launch();
  cudaError_t e = cudaGetLastError();
  *rc = e == cudaSuccess ? PB_OK : cuda_fail(e, "pb_binary");
  return 1;
}

template <int OP, typename CT>
static int run_binary(const pb_tensor* a, const pb_tensor* b, const pb_scalar* s, const pb_tensor* out) {
  typedef typename Bin<OP, CT>::res R;
  int64_t n = numel(*out);
  if (n == 0) return PB_OK;
  CT sa = 0, sb = 0;
  int am = a ? 0 : 1, bm = b ? 0 : 1;
  if (!a) sa = scalar_as<CT>(s);
  if (!b) sb = scalar_as<CT>(s);
  // vector fast path: operand dtypes == CT, out dtype == R, contiguous / scalar
  const int ct = std::is_same<CT, float>::value ? PB_F32 : std::is_same<CT, bool>::value ? PB_BOOL : -1;
  const int rt = std::is_same<R, float>::value ? PB_F32 : std::is_same<R, bool>::value ? PB_BOOL : -2;
  if (ct >= 0 && out->dtype == rt && is_contiguous(*out) && aligned16(out->ptr) && (!a || a->dtype == ct) &&
      (!b || b->dtype == ct)) {
    int va = vec_mode(a, out), vb = vec_mode(b, out);
    if (va >= 0 && vb >= 0 && !(va == 1 && vb == 1) && !(a && va == 1) && !(b && vb == 1))
      return launch_vec_bin<OP, CT, R>(a, b, va, vb, sa, sb, out, n);
  }
  if (std::is_same<CT, float>::value) {
    int rc;
    if (try_bcast_f32<OP>(a, b, (float)sa, (float)sb, out, &rc)) return rc;
  }
  RowArgs r = make_rows(out, a, b);
  ew_rows_bin<OP, CT><<<rows_grid(r), 256, 0, compute_stream()>>>(r, sa, sb, am, bm);
  PB_LAUNCHED();
  return PB_OK;
}

template <int OP>
static int dispatch_binary(int compute, const pb_tensor* a, const pb_tensor* b, const pb_scalar* s,
                           const pb_tensor* out) {
  switch (compute) {
    case PB_BOOL: return run_binary<OP, bool>(a, b, s, out);
    case PB_U8: return run_binary<OP, uint8_t>(a, b, s, out);
    case PB_I32: return run_binary<OP, int32_t>(a, b, s, out);
    case PB_I64: return run_binary<OP, int64_t>(a, b, s, out);
    case PB_F32: return run_binary<OP, float>(a, b, s, out);
    case PB_F64: return run_binary<OP, double>(a, b, s, out);
  }
  return fail(PB_ERR_ARG, "pb_binary: bad compute dtype");
}

template <int OP, typename CT>
static int run_unary(const pb_tensor* a, const pb_tensor* out) {
  int64_t n = numel(*out);
  if (n == 0) return PB_OK;
  const int ct = std::is_same<CT, float>::value ? PB_F32 : std::is_same<CT, bool>::value ? PB_BOOL : -1;
  if (ct >= 0 && a->dtype == ct && out->dtype == ct && is_contiguous(*a) && is_contiguous(*out) &&
      aligned16(a->ptr) && aligned16(out->ptr)) {
    ew_vec_un<OP, CT, CT><<<grid_for(n, 256, Vec<CT>::N * 2), 256, 0, compute_stream()>>>(
        (const CT*)(uintptr_t)a->ptr, (CT*)(uintptr_t)out->ptr, n);
    PB_LAUNCHED();
    return PB_OK;
  }
  RowArgs r = make_rows(out, a, nullptr);
  ew_rows_un<OP, CT><<<rows_grid(r), 256, 0, compute_stream()>>>(r);
  PB_LAUNCHED();
  return PB_OK;
}

template <int OP>
static int dispatch_unary(int compute, const pb_tensor* a, const pb_tensor* out) {
  switch (compute) {
    case PB_BOOL: return run_unary<OP, bool>(a, out);
    case PB_U8: return run_unary<OP, uint8_t>(a, out);
    case PB_I32: return run_unary<OP, int32_t>(a, out);
    case PB_I64: return run_unary<OP, int64_t>(a, out);
    case PB_F32: return run_unary<OP, float>(a, out);
    case PB_F64: return run_unary<OP, double>(a, out);
  }
  return fail(PB_ERR_ARG, "pb_unary: bad compute dtype");
}

// cast: bool -> f32 and f32 -> bool are on the ReLU-mask hot path; give them vector kernels
static int run_cast(const pb_tensor* src, const pb_tensor* dst) {
  int64_t n = numel(*dst);
  if (n == 0) return PB_OK;
  bool contig = is_contiguous(*src) && is_contiguous(*dst) && aligned16(src->ptr) && aligned16(dst->ptr) &&
                src->ndim == dst->ndim;
  if (contig && src->dtype == PB_BOOL && dst->dtype == PB_F32) {
    ew_vec_un<PB_CAST, bool, float><<<grid_for(n, 256, 32), 256, 0, compute_stream()>>>(
        (const bool*)(uintptr_t)src->ptr, (float*)(uintptr_t)dst->ptr, n);
    PB_LAUNCHED();
    return PB_OK;
  }
  if (contig && src->dtype == dst->dtype && src->dtype == PB_F32) {
    ew_vec_un<PB_CAST, float, float><<<grid_for(n, 256, 8), 256, 0, compute_stream()>>>(
        (const float*)(uintptr_t)src->ptr, (float*)(uintptr_t)dst->ptr, n);
    PB_LAUNCHED();
    return PB_OK;
  }
  return dispatch_unary<PB_CAST>(dst->dtype, src, dst);
}

// ---------------------------------------------------------------------------- pad / fill
struct PadArgs {
  const void* src;
  void* out;
  int dts, dto, ndim;
  int64_t oshape[PB_MAX_RANK], ostr[PB_MAX_RANK], sshape[PB_MAX_RANK], sstr[PB_MAX_RANK], lo[PB_MAX_RANK];
  int64_t n;
};

template <typename T>
__global__ void __launch_bounds__(256) pad_kernel(PadArgs p, T value) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < p.n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t rem = i, so = 0, oo = 0;
    bool inside = true;
    for (int k = p.ndim - 1; k >= 0; --k) {
      int64_t idx = rem % p.oshape[k];
      rem /= p.oshape[k];
      oo += idx * p.ostr[k];
      int64_t j = idx - p.lo[k];
      if (j < 0 || j >= p.sshape[k]) inside = false;
      so += j * p.sstr[k];
    }
    T v = inside ? load_as<T>(p.src, p.dts, so) : value;
    store_from<T>(p.out, p.dto, oo, v);
  }
}


// 4-byte same-dtype pad into a contiguous output, n < 2^31: FastDiv index decomposition,
// 4 elements per thread with the loads issued first (the reference's max-pool backward is
// chains of these pads over strided views, minml/autograd.py:667-693).
struct PadFast {
  const uint32_t* src;
  uint32_t* out;
  int nd;
  FastDiv ext[PB_MAX_RANK];
  int64_t sstr[PB_MAX_RANK];
  int32_t lo[PB_MAX_RANK], sext[PB_MAX_RANK];
  uint32_t n;
};

__global__ void __launch_bounds__(256) pad_fast(PadFast p, uint32_t value) {
  const uint32_t step = gridDim.x * 1024u;
  for (uint32_t base = blockIdx.x * 1024u + threadIdx.x; base < p.n; base += step) {
    uint32_t v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      uint32_t e = base + u * 256u;
      v[u] = value;
      if (e < p.n) {
        int64_t so = 0;
        bool inside = true;
        for (int k = p.nd - 1; k >= 0; --k) {
          uint32_t q, r;
          p.ext[k].divmod(e, q, r);
          int j = (int)r - p.lo[k];
          inside = inside && j >= 0 && j < p.sext[k];
          so += (int64_t)j * p.sstr[k];
          e = q;
        }
        if (inside) v[u] = __ldg(p.src + so);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      uint32_t e = base + u * 256u;
      if (e < p.n) p.out[e] = v[u];
    }
  }
}

// innermost output extent % 4 == 0: one index decomposition per 4 consecutive outputs of a
// row, 16-byte stores
__device__ __forceinline__ void pad_row(const PadFast& p, uint32_t row, int64_t& so, bool& inside) {
  so = 0;
  inside = true;
  for (int k = p.nd - 2; k >= 0; --k) {
    uint32_t q2, r;
    p.ext[k].divmod(row, q2, r);
    const int j = (int)r - p.lo[k];
    inside = inside && j >= 0 && j < p.sext[k];
    so += (int64_t)j * p.sstr[k];
    row = q2;
  }
}

// 4 consecutive outputs per thread, 16-byte stores (n % 4 == 0): the outer index is decoded
// once per inner-axis row the 4 outputs touch (once when the inner extent is a multiple of 4,
// twice for the max-pool backward's 1 -> 2 interleave pads)
__global__ void __launch_bounds__(256) pad_fast4(PadFast p, uint32_t value) {
  const uint32_t n4 = p.n >> 2;
  const int in = p.nd - 1;
  const int E = (int)p.ext[in].d;
  for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < n4; q += gridDim.x * blockDim.x) {
    uint32_t row, x0;
    p.ext[in].divmod(q << 2, row, x0);
    int64_t so;
    bool inside;
    pad_row(p, row, so, inside);
    int x = (int)x0;
    uint32_t v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (x == E) {  // next inner-axis row
        x = 0;
        pad_row(p, ++row, so, inside);
      }
      const int j = x - p.lo[in];
      v[u] = (inside && j >= 0 && j < p.sext[in]) ? __ldg(p.src + so + (int64_t)j * p.sstr[in]) : value;
      ++x;
    }
    reinterpret_cast<uint4*>(p.out)[q] = make_uint4(v[0], v[1], v[2], v[3]);
  }
}

template <typename T>
__global__ void __launch_bounds__(256) fill_kernel(T* out, int64_t n, T v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = v;
}

__global__ void arange_kernel(int64_t* out, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = i;
}

template <typename T>
__global__ void check_kernel(const void* p, int dt, RowArgs r, int what, int32_t* flag) {
  row_walk(r, [&](int64_t ia, int64_t, int64_t) {
    T v = load_as<T>(p, dt, ia);
    if ((what == 0 && v == 0) || (what == 1 && v < 0)) *flag = 1;
  });
}

// ---------------------------------------------------------------------- fused SGD step
// Multi-tensor launches carry their tensor table in the kernel parameters (no host->device
// metadata copies, so the launch is CUDA-graph capturable).  Each tensor is cut into
// 8192-element work items; blocks find their tensor by binary search over item prefixes.
static const int kMaxTensors = 128;
static const int64_t kItem = 8192;
struct MultiTable {
  float* p[kMaxTensors];        // parameter out (may equal pin)
  const float* pin[kMaxTensors];
  const float* g[kMaxTensors];
  float* v[kMaxTensors];        // velocity out (may equal vin)
  const float* vin[kMaxTensors];
  int64_t n[kMaxTensors];
  int64_t dst[kMaxTensors];    // bucket offsets (pack)
  int32_t first[kMaxTensors + 1];  // prefix of work items
  int count;
};

__device__ __forceinline__ int find_tensor(const MultiTable& t, int item) {
  int lo = 0, hi = t.count - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (t.first[mid] <= item) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// op order matches minml/optim.py:24-33, 64-72, each op rounded separately (no FMA):
//   g' = g + p*wd ; v = v*mu + g' ; p = p - v*lr
__global__ void __launch_bounds__(256) sgd_kernel(const __grid_constant__ MultiTable t, float lr, float mu, float wd,
                                                  int has_mu, int has_wd) {
  int items = t.first[t.count];
  for (int it = blockIdx.x; it < items; it += gridDim.x) {
    int k = find_tensor(t, it);
    int64_t s = (int64_t)(it - t.first[k]) * kItem;
    int64_t e = s + kItem < t.n[k] ? s + kItem : t.n[k];
    float* P = t.p[k];
    const float* PI = t.pin[k];
    const float* G = t.g[k];
    float* V = t.v[k];
    const float* VI = t.vin[k];
    for (int64_t i = s + threadIdx.x; i < e; i += blockDim.x) {
      float g = G[i];
      float p = PI[i];
      if (has_wd) g = __fadd_rn(g, __fmul_rn(p, wd));
      float v = g;
      if (has_mu) {
        v = __fadd_rn(__fmul_rn(VI[i], mu), g);
        V[i] = v;
      }
      P[i] = __fsub_rn(p, __fmul_rn(v, lr));
    }
  }
}

__global__ void __launch_bounds__(256) pack_kernel(const __grid_constant__ MultiTable t, float* bucket) {
  int items = t.first[t.count];
  for (int it = blockIdx.x; it < items; it += gridDim.x) {
    int k = find_tensor(t, it);
    int64_t s = (int64_t)(it - t.first[k]) * kItem;
    int64_t e = s + kItem < t.n[k] ? s + kItem : t.n[k];
    const float* G = t.g[k];
    float* D = bucket + t.dst[k];
    for (int64_t i = s + threadIdx.x; i < e; i += blockDim.x) D[i] = G[i];
  }
}

__global__ void scale_kernel(float* buf, int64_t n, float div) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    buf[i] = __fdiv_rn(buf[i], div);
}


// ------------------------------------------------------- fused multi-stage reductions
// The reference composes per-channel statistics from single-axis f32 sums, each rounded to
// f32 and usually followed by a scalar op: BatchNorm's batch mean is
// x.mean(3).mean(2).mean(0) (minml/nn.py:288-306, mean = sum / n, minml/ops.py:33-36) and
// _unbroadcast reduces a [N, C, H, W] gradient to [1, C, 1, 1] with sum(0).sum(2).sum(3)
// (minml/autograd.py:290-297), usually of a product such as g * xhat.  pb_reduce_chain runs
// such a chain -- source elementwise chain, 2-3 sum stages, their scalar epilogues -- in one
// launch with the same arithmetic per stage: f32 terms summed in f64, rounded to f32, then the
// epilogue in f32.  Only the order of the f64 additions differs from the one-kernel-per-stage
// path, which changes the rounded f32 result only when a partial-sum rounding in f64 (2^-53)
// straddles an f32 rounding boundary.
//   rows mode  stage 1 over the innermost axis (w), stage 2 over h, stage 3 over an outer axis:
//              a sub-warp per row, lanes interleaved (float4 per lane when the rows allow),
//              butterfly fold; stage 2 by one thread per i3 in row order.
//   cols mode  stage 1 over an outer axis (n), stage 3 over the innermost axis (w): a thread
//              per (h, 4 consecutive w) walks n in order with 16-byte loads.
// A block owns one output group (kept index) and a range of stage-3 indices; with several
// blocks per group the stage-2 values go to a workspace and the group's last block (ticket)
// sums them in index order.
struct RCArgs {
  const void* leaf[kChainLeaves];
  int8_t is_bool[kChainLeaves];
  int8_t s_vec[kChainLeaves];  // V4: unit stride along the vector axis (else broadcast)
  int nleaves, nsteps, head_kind;
  float head_scalar;
  ChainStep step[kChainSteps];
  int64_t s1[kChainLeaves], s2[kChainLeaves], s3[kChainLeaves];  // leaf strides along the stage axes
  int64_t ks[kChainLeaves][3];                                     // ... along the kept axes (outer first)
  FastDiv kd1, kd2;                                                // kept extents 1 and 2 (group decode)
  int E1, E2, E3, nst;
  int epi[3], epil[3];
  float epis[3];
  int r3, nsplit;
  int U1, pp, E1p;  // rows: units per row (E1 / 4 or E1), planes per pass, padded smem row pitch
  FastDiv fU1, fE2;
  int P, S;         // cols: pairs per pass, slices of the stage-1 axis
  float* out;
  float* ws;
  unsigned* tick;
};

// B source values -- float4s along the vector axis (V4) or scalars in .x -- with one dispatch per
// chain step for all of them (the interpreter's switch is paid once per B x 4 elements, and the
// kernel holds one copy of it).  The host admits only the steps handled here (no transcendental
// ops), so a step is the same Bin/Un functor the unfused kernels apply: bit-identical values.
template <int NL, int B, bool V4>
__device__ __forceinline__ void rc_eval_batch(const RCArgs& p, const int64_t (&off)[B][NL], const bool (&on)[B],
                                              float4 (&v)[B]) {
  float4 x[NL][B];
#pragma unroll
  for (int l = 0; l < NL; ++l) {
    if (l >= p.nleaves) continue;  // NL is a bucket (1, 2, 3, 4, 8): leaves past nleaves are never read
    const bool vec = V4 && p.s_vec[l];
    if (p.is_bool[l]) {
      const uint8_t* b8 = (const uint8_t*)p.leaf[l];
#pragma unroll
      for (int u = 0; u < B; ++u) {
        if (!on[u]) continue;
        if (vec) {
          const uchar4 c = *reinterpret_cast<const uchar4*>(b8 + off[u][l]);
          x[l][u] = make_float4(c.x ? 1.f : 0.f, c.y ? 1.f : 0.f, c.z ? 1.f : 0.f, c.w ? 1.f : 0.f);
        } else {
          const float t = b8[off[u][l]] ? 1.f : 0.f;
          x[l][u] = make_float4(t, t, t, t);
        }
      }
    } else {
      const float* f = (const float*)p.leaf[l];
#pragma unroll
      for (int u = 0; u < B; ++u) {
        if (!on[u]) continue;
        if (vec) {
          x[l][u] = __ldg(reinterpret_cast<const float4*>(f + off[u][l]));
        } else {
          const float t = __ldg(f + off[u][l]);
          x[l][u] = make_float4(t, t, t, t);
        }
      }
    }
  }
  const float4 hs = make_float4(p.head_scalar, p.head_scalar, p.head_scalar, p.head_scalar);
#pragma unroll
  for (int u = 0; u < B; ++u) v[u] = p.head_kind == 0 ? x[0][u] : hs;
  for (int s = 0; s < p.nsteps; ++s) {
    const ChainStep st = p.step[s];
    float4 o[B];
    if (st.kind == 1) {
      const int sl = st.leaf;
#pragma unroll
      for (int u = 0; u < B; ++u) {
        float4 t = x[0][u];
        if constexpr (NL > 1) t = sl == 1 ? x[NL > 1 ? 1 : 0][u] : t;
        if constexpr (NL > 2) t = sl == 2 ? x[NL > 2 ? 2 : 0][u] : t;
        if constexpr (NL > 3) t = sl == 3 ? x[NL > 3 ? 3 : 0][u] : t;
        if constexpr (NL > 4) t = sl == 4 ? x[NL > 4 ? 4 : 0][u] : t;
        if constexpr (NL > 5) t = sl == 5 ? x[NL > 5 ? 5 : 0][u] : t;
        if constexpr (NL > 6) t = sl == 6 ? x[NL > 6 ? 6 : 0][u] : t;
        if constexpr (NL > 7) t = sl == 7 ? x[NL > 7 ? 7 : 0][u] : t;
        o[u] = t;
      }
    } else if (st.kind == 2) {
#pragma unroll
      for (int u = 0; u < B; ++u) o[u] = make_float4(st.scalar, st.scalar, st.scalar, st.scalar);
    } else {
#pragma unroll
      for (int u = 0; u < B; ++u) o[u] = v[u];
    }
    if (st.kind != 0 && st.side) {
#pragma unroll
      for (int u = 0; u < B; ++u) {
        const float4 t = v[u];
        v[u] = o[u];
        o[u] = t;
      }
    }
#define RC_LANES(...)                                  \
  _Pragma("unroll") for (int u = 0; u < B; ++u) {     \
    float a_, b_;                                      \
    a_ = v[u].x; b_ = o[u].x; v[u].x = (__VA_ARGS__);  \
    a_ = v[u].y; b_ = o[u].y; v[u].y = (__VA_ARGS__);  \
    a_ = v[u].z; b_ = o[u].z; v[u].z = (__VA_ARGS__);  \
    a_ = v[u].w; b_ = o[u].w; v[u].w = (__VA_ARGS__);  \
    (void)b_;                                          \
  }
    if (st.kind == 0) {
      switch (st.op - 64) {
        case PB_NEG: RC_LANES(Un<PB_NEG, float>::f(a_)) break;
        case PB_ABS: RC_LANES(Un<PB_ABS, float>::f(a_)) break;
        case PB_NOT: RC_LANES(a_ == 0.f ? 1.f : 0.f) break;
        default:
          if (st.to_bool) RC_LANES(a_ != 0.f ? 1.f : 0.f)
          break;
      }
      continue;
    }
    switch (st.op) {
      case PB_ADD: RC_LANES(Bin<PB_ADD, float>::f(a_, b_)) break;
      case PB_SUB: RC_LANES(Bin<PB_SUB, float>::f(a_, b_)) break;
      case PB_MUL: RC_LANES(Bin<PB_MUL, float>::f(a_, b_)) break;
      case PB_DIV: RC_LANES(Bin<PB_DIV, float>::f(a_, b_)) break;
      case PB_MIN: RC_LANES(Bin<PB_MIN, float>::f(a_, b_)) break;
      case PB_MAX: RC_LANES(Bin<PB_MAX, float>::f(a_, b_)) break;
      case PB_EQ: RC_LANES(a_ == b_ ? 1.f : 0.f) break;
      case PB_LT: RC_LANES(a_ < b_ ? 1.f : 0.f) break;
      case PB_GT: RC_LANES(a_ > b_ ? 1.f : 0.f) break;
      case PB_AND: RC_LANES((a_ != 0.f && b_ != 0.f) ? 1.f : 0.f) break;
      default: RC_LANES((a_ != 0.f || b_ != 0.f) ? 1.f : 0.f) break;
    }
#undef RC_LANES
  }
}

// plain source (one dense f32 leaf, no steps)
template <int B, bool V4>
__device__ __forceinline__ void rc_load_batch(const RCArgs& p, const int64_t (&off)[B][1], const bool (&on)[B],
                                              float4 (&v)[B]) {
  const float* f = (const float*)p.leaf[0];
#pragma unroll
  for (int u = 0; u < B; ++u) {
    if (!on[u]) continue;
    if (V4) {
      v[u] = __ldg(reinterpret_cast<const float4*>(f + off[u][0]));
    } else {
      const float t = __ldg(f + off[u][0]);
      v[u] = make_float4(t, t, t, t);
    }
  }
}

// product source (round 2): v = x0 * x0 (BatchNorm's c * c) or x0 * x1 (the gamma gradient's
// g * xhat), f32 leaves -- the interpreter's one MUL step without its dispatch and registers
template <int NL, int B, bool V4>
__device__ __forceinline__ void rc_mul_batch(const RCArgs& p, const int64_t (&off)[B][NL], const bool (&on)[B],
                                             float4 (&v)[B]) {
  float4 y[B];
#pragma unroll
  for (int l = 0; l < NL; ++l) {
    const float* f = (const float*)p.leaf[l];
    const bool vec = V4 && p.s_vec[l];
#pragma unroll
    for (int u = 0; u < B; ++u) {
      float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
      if (on[u]) {
        if (vec) {
          t = __ldg(reinterpret_cast<const float4*>(f + off[u][l]));
        } else {
          const float q = __ldg(f + off[u][l]);
          t = make_float4(q, q, q, q);
        }
      }
      if (l == 0) v[u] = t;
      else y[u] = t;
    }
  }
#pragma unroll
  for (int u = 0; u < B; ++u) {
    const float4 w = NL > 1 ? y[u] : v[u];
    v[u] = make_float4(Bin<PB_MUL, float>::f(v[u].x, w.x), Bin<PB_MUL, float>::f(v[u].y, w.y),
                       Bin<PB_MUL, float>::f(v[u].z, w.z), Bin<PB_MUL, float>::f(v[u].w, w.w));
  }
}

// one-step source (round 2): one f32 leaf and one cheap step -- neg / abs, or add / sub / mul
// with a scalar (the sub backward's -g before its _unbroadcast sum); the same functors
__device__ __forceinline__ float rc_one(const ChainStep& st, float a) {
  if (st.kind == 0) return st.op - 64 == PB_NEG ? Un<PB_NEG, float>::f(a) : Un<PB_ABS, float>::f(a);
  const float x = st.side ? st.scalar : a, y = st.side ? a : st.scalar;
  return st.op == PB_ADD ? Bin<PB_ADD, float>::f(x, y)
                         : st.op == PB_SUB ? Bin<PB_SUB, float>::f(x, y) : Bin<PB_MUL, float>::f(x, y);
}
template <int B, bool V4>
__device__ __forceinline__ void rc_one_batch(const RCArgs& p, const int64_t (&off)[B][1], const bool (&on)[B],
                                             float4 (&v)[B]) {
  const float* f = (const float*)p.leaf[0];
  const bool vec = V4 && p.s_vec[0];
  const ChainStep st = p.step[0];
#pragma unroll
  for (int u = 0; u < B; ++u) {
    if (!on[u]) continue;
    if (vec) {
      v[u] = __ldg(reinterpret_cast<const float4*>(f + off[u][0]));
    } else {
      const float q = __ldg(f + off[u][0]);
      v[u] = make_float4(q, q, q, q);
    }
  }
#pragma unroll
  for (int u = 0; u < B; ++u)
    v[u] = make_float4(rc_one(st, v[u].x), rc_one(st, v[u].y), rc_one(st, v[u].z), rc_one(st, v[u].w));
}

// SRC 1: plain source; 2: product source; 3: one-step source; 0: the interpreter
template <int NL, int B, bool V4, int SRC>
__device__ __forceinline__ void rc_source(const RCArgs& p, const int64_t (&off)[B][NL], const bool (&on)[B],
                                          float4 (&v)[B]) {
  if constexpr (SRC == 1) rc_load_batch<B, V4>(p, off, on, v);
  else if constexpr (SRC == 2) rc_mul_batch<NL, B, V4>(p, off, on, v);
  else if constexpr (SRC == 3) rc_one_batch<B, V4>(p, off, on, v);
  else rc_eval_batch<NL, B, V4>(p, off, on, v);
}

__device__ __forceinline__ float rc_epi(const RCArgs& p, int k, float v) {
  const int op = p.epi[k];
  if (op < 0) return v;
  const float a = p.epil[k] ? p.epis[k] : v, b = p.epil[k] ? v : p.epis[k];
  switch (op) {
    case PB_ADD: return a + b;
    case PB_SUB: return a - b;
    case PB_MUL: return a * b;
    default: return a / b;
  }
}

template <int NL>
__device__ __forceinline__ void rc_group_base(const RCArgs& p, int g, int64_t (&gb)[NL]) {
  uint32_t t, k0, k1, k2;
  p.kd2.divmod((uint32_t)g, t, k2);
  p.kd1.divmod(t, k0, k1);
#pragma unroll
  for (int l = 0; l < NL; ++l) gb[l] = (int64_t)k0 * p.ks[l][0] + (int64_t)k1 * p.ks[l][1] + (int64_t)k2 * p.ks[l][2];
}

// rows mode: block (group g, planes [i3a, i3a + np)) evaluates its planes (E2 rows x E1, contiguous
// for dense sources) into shared memory -- several units per thread in flight, 16-byte loads when
// rows allow -- then a thread per row sums it in f64 (4 chains) from the odd-pitch (conflict-free)
// buffer, a warp per plane folds the rows (stage 2), and stage 3 folds the planes: in the block when
// it holds them all, else through the workspace in the group's last block (ticket)
template <int NL, bool V4, int SRC>
__global__ void __launch_bounds__(256) redchain_rows(RCArgs p) {
  extern __shared__ float rc_smem[];
  constexpr int VW = V4 ? 4 : 1;
  float* v1s = rc_smem;                // [np][E2]
  float* v2s = v1s + p.r3 * p.E2;      // [np]
  float* pl = v2s + p.r3;              // [np][E2][E1p]
  const int g = blockIdx.x / p.nsplit, sp = blockIdx.x - g * p.nsplit;
  const int i3a = sp * p.r3, np = min(p.r3, p.E3 - i3a);
  int64_t gb[NL];
  rc_group_base<NL>(p, g, gb);
  constexpr int B = SRC == 1 || SRC == 3 ? 8 : SRC == 2 ? (NL == 1 ? 8 : 4) : (NL <= 3 ? 4 : 2);
  const int units = np * p.E2 * p.U1;
  for (int u0 = threadIdx.x; u0 < units; u0 += B * blockDim.x) {
    float4 v[B];
    int64_t off[B][NL];
    bool on[B];
    int dst[B];
#pragma unroll
    for (int k = 0; k < B; ++k) {
      const int u = u0 + k * blockDim.x;
      on[k] = u < units;
      uint32_t rest, i1u, pi, i2;
      p.fU1.divmod((uint32_t)(on[k] ? u : 0), rest, i1u);
      p.fE2.divmod(rest, pi, i2);
      const int64_t i3 = i3a + (int)pi, i1 = (int64_t)i1u * VW;
#pragma unroll
      for (int l = 0; l < NL; ++l) off[k][l] = gb[l] + i3 * p.s3[l] + (int64_t)i2 * p.s2[l] + i1 * p.s1[l];
      dst[k] = (int)(pi * p.E2 + i2) * p.E1p + (int)i1;
    }
    rc_source<NL, B, V4, SRC>(p, off, on, v);
#pragma unroll
    for (int k = 0; k < B; ++k) {
      if (on[k]) {
        pl[dst[k]] = v[k].x;
        if (V4) {
          pl[dst[k] + 1] = v[k].y;
          pl[dst[k] + 2] = v[k].z;
          pl[dst[k] + 3] = v[k].w;
        }
      }
    }
  }
  __syncthreads();
  for (int r = threadIdx.x; r < np * p.E2; r += blockDim.x) {
    const float* row = pl + r * p.E1p;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    int j = 0;
    for (; j + 4 <= p.E1; j += 4) {
      a0 += (double)row[j];
      a1 += (double)row[j + 1];
      a2 += (double)row[j + 2];
      a3 += (double)row[j + 3];
    }
    for (; j < p.E1; ++j) a0 += (double)row[j];
    v1s[r] = rc_epi(p, 0, (float)((a0 + a1) + (a2 + a3)));
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int pi = wp; pi < np; pi += nw) {  // stage 2: a warp per plane
    double a = 0.0;
    for (int k = lane; k < p.E2; k += 32) a += (double)v1s[pi * p.E2 + k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == 0) {
      const float v2 = rc_epi(p, 1, (float)a);
      if (p.nst < 3) p.out[g] = v2;  // E3 == 1
      else if (p.nsplit == 1) v2s[pi] = v2;
      else p.ws[(int64_t)g * p.E3 + i3a + pi] = v2;
    }
  }
  if (p.nst < 3) return;
  if (p.nsplit == 1) {
    __syncthreads();
    if (threadIdx.x == 0) {
      double a = 0.0;
      for (int t = 0; t < p.E3; ++t) a += (double)v2s[t];
      p.out[g] = rc_epi(p, 2, (float)a);
    }
    return;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned ticket = atomicAdd(p.tick + g, 1u);
    if (ticket == (unsigned)p.nsplit - 1) {  // every block of this group has published
      __threadfence();
      const float* w = p.ws + (int64_t)g * p.E3;
      double a = 0.0;
      for (int t = 0; t < p.E3; ++t) a += (double)__ldcg(w + t);
      p.out[g] = rc_epi(p, 2, (float)a);
      p.tick[g] = 0u;
    }
  }
}

// cols mode (stage 1 over a strided axis, stage 3 over the contiguous one): block (group g, stage-2
// rows [h0, h0 + nh)) gives a thread each (row, 4 consecutive stage-3 indices) and a slice of the
// stage-1 axis, walked with 8 loads in flight -- a warp reads contiguous 512-byte spans; slices fold
// in order through shared memory.  Stage 2 sums the block's rows per column in f64; with several
// blocks per group those f64 partials meet in the group's last block (ticket), which rounds them,
// applies the stage-2 epilogue and folds stage 3.
template <int NL, bool V4, int SRC>
__global__ void __launch_bounds__(256) redchain_cols(RCArgs p) {
  extern __shared__ float rc_smem[];
  constexpr int VW = V4 ? 4 : 1;
  const int hr = p.r3, W = p.E3;
  float* v1s = rc_smem;                                                   // [W][hr]
  float* v2s = v1s + W * hr;                                              // [W]
  double* part = reinterpret_cast<double*>(rc_smem + ((W * hr + W + 1) & ~1));  // [S][P][VW]
  const int g = blockIdx.x / p.nsplit, sp = blockIdx.x - g * p.nsplit;
  const int h0 = sp * hr, nh = min(hr, p.E2 - h0);
  int64_t gb[NL];
  rc_group_base<NL>(p, g, gb);
  const int wu = W / VW;
  const int npairs = nh * wu;
  const int pi = threadIdx.x % p.P, si = threadIdx.x / p.P;
  const int chunk = (p.E1 + p.S - 1) / p.S;
  const int j0 = si * chunk, j1 = min(p.E1, j0 + chunk);
  for (int q0 = 0; q0 < npairs; q0 += p.P) {
    const int q = q0 + pi;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    const bool on = q < npairs;
    const int hl = on ? q / wu : 0, i3 = on ? (q - hl * wu) * VW : 0;
    if (on) {
      int64_t po[NL];
#pragma unroll
      for (int l = 0; l < NL; ++l) po[l] = gb[l] + (int64_t)i3 * p.s3[l] + (int64_t)(h0 + hl) * p.s2[l];
      constexpr int B = SRC == 1 ? 16 : SRC == 3 ? 8 : SRC == 2 ? (NL == 1 ? 8 : 4) : (NL <= 3 ? 4 : 2);
      for (int j = j0; j < j1; j += B) {
        float4 v[B];
        int64_t off[B][NL];
        bool on[B];
#pragma unroll
        for (int u = 0; u < B; ++u) {
          on[u] = j + u < j1;
#pragma unroll
          for (int l = 0; l < NL; ++l) off[u][l] = po[l] + (int64_t)(j + u) * p.s1[l];
        }
        rc_source<NL, B, V4, SRC>(p, off, on, v);
#pragma unroll
        for (int u = 0; u < B; ++u) {
          if (on[u]) {
            a0 += (double)v[u].x;
            if (V4) {
              a1 += (double)v[u].y;
              a2 += (double)v[u].z;
              a3 += (double)v[u].w;
            }
          }
        }
      }
    }
    if (p.S > 1) {
      double* d = part + ((int64_t)si * p.P + pi) * VW;
      d[0] = a0;
      if (V4) {
        d[1] = a1;
        d[2] = a2;
        d[3] = a3;
      }
      __syncthreads();
      if (si == 0 && on) {
        for (int t = 1; t < p.S; ++t) {
          const double* e = part + ((int64_t)t * p.P + pi) * VW;
          a0 += e[0];
          if (V4) {
            a1 += e[1];
            a2 += e[2];
            a3 += e[3];
          }
        }
      }
      __syncthreads();
    }
    if (si == 0 && on) {
      float* d = v1s + i3 * hr + hl;
      d[0] = rc_epi(p, 0, (float)a0);
      if (V4) {
        d[hr] = rc_epi(p, 0, (float)a1);
        d[2 * hr] = rc_epi(p, 0, (float)a2);
        d[3 * hr] = rc_epi(p, 0, (float)a3);
      }
    }
  }
  __syncthreads();
  double* wsd = reinterpret_cast<double*>(p.ws);
  for (int t = threadIdx.x; t < W; t += blockDim.x) {  // stage 2 over this block's rows
    double a = 0.0;
    for (int k = 0; k < nh; ++k) a += (double)v1s[t * hr + k];
    if (p.nsplit == 1) v2s[t] = rc_epi(p, 1, (float)a);
    else wsd[((int64_t)g * p.nsplit + sp) * W + t] = a;
  }
  if (p.nsplit > 1) {
    __threadfence();
    __syncthreads();
    __shared__ unsigned last;
    if (threadIdx.x == 0) last = atomicAdd(p.tick + g, 1u) == (unsigned)p.nsplit - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    for (int t = threadIdx.x; t < W; t += blockDim.x) {
      double a = 0.0;
      for (int k = 0; k < p.nsplit; ++k) a += __ldcg(wsd + ((int64_t)g * p.nsplit + k) * W + t);
      v2s[t] = rc_epi(p, 1, (float)a);
    }
    if (threadIdx.x == 0) p.tick[g] = 0u;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0;
    for (int t = 0; t < W; ++t) a += (double)v2s[t];
    p.out[g] = rc_epi(p, 2, (float)a);
  }
}

template <typename K>
static void rc_smem_attr(K k) {
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 112 * 1024);
}

template <int NL, int SRC>
static void launch_redchain(const RCArgs& p, bool rows, bool v4, int grid, int threads, size_t smem, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    rc_smem_attr(redchain_rows<NL, true, SRC>);
    rc_smem_attr(redchain_rows<NL, false, SRC>);
    rc_smem_attr(redchain_cols<NL, true, SRC>);
    rc_smem_attr(redchain_cols<NL, false, SRC>);
    attr = true;
  }
  if (rows) {
    if (v4) redchain_rows<NL, true, SRC><<<grid, threads, smem, s>>>(p);
    else redchain_rows<NL, false, SRC><<<grid, threads, smem, s>>>(p);
  } else {
    if (v4) redchain_cols<NL, true, SRC><<<grid, threads, smem, s>>>(p);
    else redchain_cols<NL, false, SRC><<<grid, threads, smem, s>>>(p);
  }
}

}  // namespace pb

using namespace pb;

#define PB_CASE_BIN(OPC) \
  case OPC: return dispatch_binary<OPC>(compute, a, b, s, out);
#define PB_CASE_UN(OPC) \
  case OPC: return dispatch_unary<OPC>(compute, a, out);

extern "C" {

int pb_binary(int op, const pb_tensor* a, const pb_tensor* b, const pb_scalar* s, int compute, const pb_tensor* out) {
  if ((!a || !b) && !s) return fail(PB_ERR_ARG, "pb_binary: missing scalar operand");
  switch (op) {
    PB_CASE_BIN(PB_ADD) PB_CASE_BIN(PB_SUB) PB_CASE_BIN(PB_MUL) PB_CASE_BIN(PB_DIV) PB_CASE_BIN(PB_POW)
    PB_CASE_BIN(PB_MIN) PB_CASE_BIN(PB_MAX) PB_CASE_BIN(PB_EQ) PB_CASE_BIN(PB_LT) PB_CASE_BIN(PB_GT)
    PB_CASE_BIN(PB_AND) PB_CASE_BIN(PB_OR)
  }
  return fail(PB_ERR_ARG, "pb_binary: unknown op");
}

int pb_unary(int op, const pb_tensor* a, int compute, const pb_tensor* out) {
  switch (op) {
    PB_CASE_UN(PB_NEG) PB_CASE_UN(PB_ABS) PB_CASE_UN(PB_EXP) PB_CASE_UN(PB_LOG) PB_CASE_UN(PB_SQRT)
    PB_CASE_UN(PB_SIN) PB_CASE_UN(PB_COS) PB_CASE_UN(PB_TANH) PB_CASE_UN(PB_NOT)
    case PB_CAST: return run_cast(a, out);
  }
  return fail(PB_ERR_ARG, "pb_unary: unknown op");
}

int pb_copy(const pb_tensor* src, const pb_tensor* dst) { return run_cast(src, dst); }

int pb_chain_jit_kernels(void) {
  Jit& j = jit();
  if (!j.ok) return -1;
  std::lock_guard<std::mutex> lk(j.mu);
  int n = 0;
  for (auto& kv : j.cache) n += kv.second != nullptr;
  return n;
}

static int ew_chain(int nleaves, const pb_tensor* leaves, int head_kind, double head_scalar, int nsteps,
                    const pb_chain_step* steps, int ntaps, const int* tap_after, const pb_tensor* taps,
                    const pb_tensor* out);

int pb_ew_chain(int nleaves, const pb_tensor* leaves, int head_kind, double head_scalar, int nsteps,
                const pb_chain_step* steps, const pb_tensor* out) {
  return ew_chain(nleaves, leaves, head_kind, head_scalar, nsteps, steps, 0, nullptr, nullptr, out);
}

int pb_ew_chain_taps(int nleaves, const pb_tensor* leaves, int head_kind, double head_scalar, int nsteps,
                     const pb_chain_step* steps, int ntaps, const int* tap_after, const pb_tensor* taps,
                     const pb_tensor* out) {
  if (ntaps < 0 || ntaps > kChainTaps) return fail(PB_ERR_ARG, "pb_ew_chain_taps: 0..4 taps");
  for (int i = 0; i < ntaps; ++i) {
    if (tap_after[i] < 1 || tap_after[i] > nsteps) return fail(PB_ERR_ARG, "pb_ew_chain_taps: tap step out of range");
    if (taps[i].dtype != PB_F32 || !is_contiguous(taps[i]) || numel(taps[i]) != numel(*out) || (taps[i].ptr & 15))
      return fail(PB_ERR_ARG, "pb_ew_chain_taps: a tap is a dense, 16-byte aligned f32 tensor of the output's size");
  }
  return ew_chain(nleaves, leaves, head_kind, head_scalar, nsteps, steps, ntaps, tap_after, taps, out);
}

static int ew_chain(int nleaves, const pb_tensor* leaves, int head_kind, double head_scalar, int nsteps,
                    const pb_chain_step* steps, int ntaps, const int* tap_after, const pb_tensor* taps,
                    const pb_tensor* out) {
  int64_t n = numel(*out);
  if (n == 0) return PB_OK;
  if (nleaves < 0 || nleaves > kChainLeaves || nsteps < 0 || nsteps > kChainSteps ||
      (head_kind == 0 && nleaves == 0))
    return fail(PB_ERR_ARG, "pb_ew_chain: bad chain shape");
  if (n >= ((int64_t)1 << 31) || !is_contiguous(*out) || (out->dtype != PB_F32 && out->dtype != PB_BOOL))
    return fail(PB_ERR_UNSUPPORTED, "pb_ew_chain: output must be a dense f32/bool tensor < 2^31 elements");
  ChainArgs p;
  memset(&p, 0, sizeof(p));
  p.nleaves = nleaves;
  p.nsteps = nsteps;
  p.head_kind = head_kind;
  p.head_scalar = (float)head_scalar;
  p.out = (void*)(uintptr_t)out->ptr;
  p.out_bool = out->dtype == PB_BOOL;
  for (int k = 0; k < nsteps; ++k) {
    const pb_chain_step& c = steps[k];
    if (c.kind == 1 && (c.leaf < 0 || c.leaf >= nleaves)) return fail(PB_ERR_ARG, "pb_ew_chain: bad leaf index");
    p.step[k].op = (int16_t)c.op;
    p.step[k].kind = (int8_t)c.kind;
    p.step[k].side = (int8_t)c.side;
    p.step[k].leaf = (int8_t)c.leaf;
    p.step[k].to_bool = (int8_t)c.to_bool;
    p.step[k].scalar = (float)c.scalar;
  }
  // right-aligned broadcast strides of every leaf over the output, then coalesce
  const int nd0 = out->ndim;
  int64_t shape[PB_MAX_RANK], st[kChainLeaves + 1][PB_MAX_RANK];
  for (int k = 0; k < nd0; ++k) {
    shape[k] = out->shape[k];
    st[kChainLeaves][k] = out->strides[k];
  }
  for (int l = 0; l < nleaves; ++l) {
    const pb_tensor& t = leaves[l];
    if (t.dtype != PB_F32 && t.dtype != PB_BOOL) return fail(PB_ERR_UNSUPPORTED, "pb_ew_chain: leaf dtype");
    p.leaf[l] = (const void*)(uintptr_t)t.ptr;
    p.is_bool[l] = t.dtype == PB_BOOL;
    for (int k = 0; k < nd0; ++k) st[l][k] = 0;
    int off = nd0 - t.ndim;
    if (off < 0) return fail(PB_ERR_ARG, "pb_ew_chain: leaf rank exceeds output rank");
    for (int k = 0; k < t.ndim; ++k) st[l][off + k] = t.shape[k] == 1 ? 0 : t.strides[k];
  }
  // drop extent-1 axes, merge axes contiguous for every operand
  int nd = 0;
  int64_t cs[PB_MAX_RANK], cst[kChainLeaves + 1][PB_MAX_RANK];
  for (int k = 0; k < nd0; ++k) {
    if (shape[k] == 1) continue;
    bool merge = nd > 0;
    for (int l = 0; l <= kChainLeaves && merge; ++l) {
      if (l < nleaves || l == kChainLeaves)
        if (cst[l][nd - 1] != st[l][k] * shape[k]) merge = false;
    }
    if (merge) {
      cs[nd - 1] *= shape[k];
      for (int l = 0; l <= kChainLeaves; ++l) cst[l][nd - 1] = st[l][k];
    } else {
      cs[nd] = shape[k];
      for (int l = 0; l <= kChainLeaves; ++l) cst[l][nd] = st[l][k];
      ++nd;
    }
  }
  if (nd == 0) {
    nd = 1;
    cs[0] = 1;
    for (int l = 0; l <= kChainLeaves; ++l) cst[l][0] = 0;
  }
  if (nd > 4) return fail(PB_ERR_UNSUPPORTED, "pb_ew_chain: more than 4 non-mergeable axes");
  p.nd = nd;
  for (int k = 0; k < 4; ++k) {
    p.ext[k] = FastDiv(k < nd ? (uint32_t)cs[k] : 1u);
    for (int l = 0; l < kChainLeaves; ++l) p.st[l][k] = (k < nd && l < nleaves) ? cst[l][k] : 0;
  }
  bool v4 = cs[nd - 1] % 4 == 0 && ((out->ptr & 15) == 0);
  for (int l = 0; l < nleaves && v4; ++l) {
    int64_t is = cst[l][nd - 1];
    if (is == 1) {
      p.vec[l] = 1;
      uint64_t align = p.is_bool[l] ? 4 : 16;
      if (leaves[l].ptr % align) v4 = false;
      for (int k = 0; k < nd - 1; ++k)
        if (cst[l][k] % 4) v4 = false;
    } else if (is != 0) {
      v4 = false;
    }
  }
  cudaStream_t s = compute_stream();
  int mode = v4 ? 1 : 0;
  if (!v4 && n % 4 == 0 && (out->ptr & 15) == 0) {  // chain4x: dense leaves aligned
    mode = 2;
    for (int l = 0; l < nleaves; ++l) {
      bool dense = true;
      for (int k = 0; k < nd; ++k) dense = dense && cst[l][k] == cst[kChainLeaves][k];
      p.dense[l] = dense;
      if (dense && leaves[l].ptr % (p.is_bool[l] ? 4 : 16)) mode = 0;
    }
  }
  if (mode == 1 && cs[nd - 1] % 8 == 0) {
    // 8-wide pays off when a broadcast leaf makes the per-step operand select the cost
    // (measured: BatchNorm affine chains 58 -> 52 us, all-dense chains 50 -> 53 us)
    bool ok = false, all_vec_ok = true;
    for (int l = 0; l < nleaves; ++l) {
      if (!p.vec[l]) ok = true;
      for (int k = 0; k < nd - 1; ++k)
        if (p.vec[l] && cst[l][k] % 8) all_vec_ok = false;
    }
    if (ok && all_vec_ok) mode = 3;
  }
  if (mode == 3) {
    p.n = (uint32_t)(n / 8);
  } else if (mode == 1) {
    p.n = (uint32_t)(n / 4);
  } else {
    for (int l = 0; l < kChainLeaves; ++l) p.vec[l] = 0;
    p.n = (uint32_t)(mode == 2 ? n / 4 : n);
  }
  p.ntaps = ntaps;
  for (int i = 0; i < ntaps; ++i) {
    p.tap_after[i] = (int8_t)tap_after[i];
    p.tap[i] = (void*)(uintptr_t)taps[i].ptr;
  }
  if (jit_chain(p, mode, nleaves, s)) {
    PB_LAUNCHED();
    return PB_OK;
  }
  if (ntaps) return fail(PB_ERR_UNSUPPORTED, "pb_ew_chain_taps: taps need the JIT chain kernels");
  switch (nleaves) {
    case 0: case 1: launch_chain<1>(p, mode, s); break;
    case 2: launch_chain<2>(p, mode, s); break;
    case 3: launch_chain<3>(p, mode, s); break;
    case 4: launch_chain<4>(p, mode, s); break;
    case 5: launch_chain<5>(p, mode, s); break;
    case 6: launch_chain<6>(p, mode, s); break;
    case 7: launch_chain<7>(p, mode, s); break;
    default: launch_chain<8>(p, mode, s); break;
  }
  PB_LAUNCHED();
  return PB_OK;
}


int pb_reduce_chain(int nleaves, const pb_tensor* leaves, int head_kind, double head_scalar, int nsteps,
                    const pb_chain_step* steps, int src_ndim, const int64_t* src_shape, int nstages,
                    const pb_red_stage* stages, const pb_tensor* out) {
  if (nleaves < 1 || nleaves > kChainLeaves || nsteps < 0 || nsteps > kChainSteps || src_ndim < 1 || src_ndim > 4 ||
      nstages < 1 || nstages > 3)
    return fail(PB_ERR_ARG, "pb_reduce_chain: bad chain shape");
  if (out->dtype != PB_F32 || !is_contiguous(*out)) return fail(PB_ERR_ARG, "pb_reduce_chain: out must be dense f32");
  if (nstages < 2) return fail(PB_ERR_UNSUPPORTED, "pb_reduce_chain: single-stage chains use pb_reduce");
  RCArgs p;
  memset(&p, 0, sizeof(p));
  p.nleaves = nleaves;
  p.nsteps = nsteps;
  p.head_kind = head_kind;
  p.head_scalar = (float)head_scalar;
  p.out = (float*)(uintptr_t)out->ptr;
  for (int k = 0; k < nsteps; ++k) {
    const pb_chain_step& c = steps[k];
    if (c.kind == 1 && (c.leaf < 0 || c.leaf >= nleaves)) return fail(PB_ERR_ARG, "pb_reduce_chain: bad leaf index");
    p.step[k].op = (int16_t)c.op;
    p.step[k].kind = (int8_t)c.kind;
    p.step[k].side = (int8_t)c.side;
    p.step[k].leaf = (int8_t)c.leaf;
    p.step[k].to_bool = (int8_t)c.to_bool;
    p.step[k].scalar = (float)c.scalar;
  }
  // the source index space, left-padded to 4 axes; leaf strides broadcast (right-aligned)
  const int pad = 4 - src_ndim;
  int64_t sh[4], st[kChainLeaves][4];
  for (int k = 0; k < 4; ++k) sh[k] = k < pad ? 1 : src_shape[k - pad];
  for (int l = 0; l < nleaves; ++l) {
    const pb_tensor& t = leaves[l];
    if (t.dtype != PB_F32 && t.dtype != PB_BOOL) return fail(PB_ERR_UNSUPPORTED, "pb_reduce_chain: leaf dtype");
    const int off = 4 - t.ndim;
    if (off < 0) return fail(PB_ERR_ARG, "pb_reduce_chain: leaf rank exceeds the source rank");
    for (int k = 0; k < 4; ++k) st[l][k] = 0;
    for (int k = 0; k < t.ndim; ++k) {
      if (t.shape[k] != 1 && t.shape[k] != sh[off + k]) return fail(PB_ERR_ARG, "pb_reduce_chain: leaf shape");
      st[l][off + k] = t.shape[k] == 1 ? 0 : t.strides[k];
    }
    p.leaf[l] = (const void*)(uintptr_t)t.ptr;
    p.is_bool[l] = t.dtype == PB_BOOL;
  }
  int ax[3] = {-1, -1, -1};
  bool used[4] = {false, false, false, false};
  for (int k = 0; k < nstages; ++k) {
    const int a = stages[k].axis + pad;
    if (a < pad || a > 3 || used[a]) return fail(PB_ERR_ARG, "pb_reduce_chain: bad stage axis");
    used[a] = true;
    ax[k] = a;
    p.epi[k] = stages[k].epi_op;
    p.epil[k] = stages[k].epi_left;
    p.epis[k] = stages[k].scalar;
    if (p.epi[k] >= 0 && p.epi[k] != PB_ADD && p.epi[k] != PB_SUB && p.epi[k] != PB_MUL && p.epi[k] != PB_DIV)
      return fail(PB_ERR_ARG, "pb_reduce_chain: epilogue must be add/sub/mul/div");
  }
  for (int k = nstages; k < 3; ++k) p.epi[k] = -1;
  p.nst = nstages;
  // rows: stage 1 over the innermost axis, stage 2 over the next; cols: stage 3 innermost
  const bool rows = ax[0] == 3 && ax[1] == 2;
  const bool cols = nstages == 3 && ax[2] == 3;
  if (!rows && !cols) return fail(PB_ERR_UNSUPPORTED, "pb_reduce_chain: stage axes");
  p.E1 = (int)sh[ax[0]];
  p.E2 = (int)sh[ax[1]];
  p.E3 = nstages == 3 ? (int)sh[ax[2]] : 1;
  int64_t G = 1;
  int nk = 0, kax[3] = {-1, -1, -1};
  for (int k = 0; k < 4; ++k) {
    if (used[k] || sh[k] == 1) continue;
    if (nk == 3) return fail(PB_ERR_UNSUPPORTED, "pb_reduce_chain: kept axes");
    kax[nk++] = k;
    G *= sh[k];
  }
  {  // right-align the kept axes into slots 0..2 (outer first)
    int64_t kext[3] = {1, 1, 1};
    for (int j = 0; j < nk; ++j) {
      const int slot = 3 - nk + j;
      kext[slot] = sh[kax[j]];
      for (int l = 0; l < nleaves; ++l) p.ks[l][slot] = st[l][kax[j]];
    }
    p.kd1 = FastDiv((uint32_t)kext[1]);
    p.kd2 = FastDiv((uint32_t)kext[2]);
  }
  if (G != numel(*out)) return fail(PB_ERR_ARG, "pb_reduce_chain: output size");
  if (G == 0) return PB_OK;
  if (G >= ((int64_t)1 << 31) || sh[0] * sh[1] * sh[2] * sh[3] >= ((int64_t)1 << 40) || p.E2 * (int64_t)p.E3 > 65536)
    return fail(PB_ERR_UNSUPPORTED, "pb_reduce_chain: extents");
  for (int l = 0; l < nleaves; ++l) {
    p.s1[l] = st[l][ax[0]];
    p.s2[l] = st[l][ax[1]];
    p.s3[l] = nstages == 3 ? st[l][ax[2]] : 0;
  }
  if (p.E1 == 0 || p.E2 == 0 || p.E3 == 0) return fail(PB_ERR_UNSUPPORTED, "pb_reduce_chain: empty stage");
  for (int k = 0; k < nsteps; ++k) {  // the reduction's evaluator runs the cheap (non-libm) steps only
    const int op = steps[k].op;
    const bool ok = steps[k].kind == 0 ? (op == 64 + PB_NEG || op == 64 + PB_ABS || op == 64 + PB_NOT ||
                                          op == 64 + PB_CAST)
                                       : (op != PB_POW && op >= 0 && op <= PB_OR);
    if (!ok) return fail(PB_ERR_UNSUPPORTED, "pb_reduce_chain: step op outside the reduction evaluator");
  }
  // 16-byte vectors along the contiguous axis (stage 1 in rows mode, stage 3 in cols mode)
  const int vax = rows ? ax[0] : ax[2];
  bool v4 = sh[vax] % 4 == 0;
  for (int l = 0; l < nleaves && v4; ++l) {
    const int64_t vs = st[l][vax];
    if (vs == 0) continue;
    if (vs != 1 || leaves[l].ptr % (p.is_bool[l] ? 4 : 16)) v4 = false;
    for (int k = 0; k < 4; ++k)
      if (k != vax && st[l][k] % 4) v4 = false;
  }
  for (int l = 0; l < nleaves; ++l) p.s_vec[l] = v4 && st[l][vax] == 1;
  // Which chains this kernel runs is measured (tools/redchain_bench.py): a chain-fed source saves
  // materialising the chain and always wins; a plain (already materialised) source wins only where
  // launches dominate -- rows mode with few channels or < 2M elements, cols mode on 16-byte rows
  // below 4M elements -- elsewhere the stage-at-a-time kernels stream faster: decline
  static const bool all_sizes = getenv("PB_RC_ALL") != nullptr;  // tools/redchain_bench.py measures both
  const int64_t numel4 = sh[0] * sh[1] * sh[2] * sh[3];
  // chains of more than two leaves or with a division stream slower here than as one chain kernel
  // plus the stage kernels (measured: BatchNorm's grad-of-std chain, 3 leaves and 2 divisions)
  bool heavy = nleaves > 2;
  for (int k = 0; k < nsteps; ++k) heavy = heavy || (steps[k].kind != 0 && steps[k].op == PB_DIV);
  if (!all_sizes && heavy) return fail(PB_ERR_UNSUPPORTED, "pb_reduce_chain: heavy chain");
  static const bool plain_rows = getenv("PB_RC_PLAIN_ROWS") != nullptr;  // experiment hook: fused plain rows
  if (!all_sizes && nleaves == 1 && nsteps == 0 && head_kind == 0 &&
      (rows ? !(plain_rows || G < 256 || numel4 < ((int64_t)1 << 21)) : !(v4 && numel4 < ((int64_t)1 << 22))))
    return fail(PB_ERR_UNSUPPORTED, "pb_reduce_chain: plain source streams faster stage by stage");
  // rows: a block owns one group and `pp` planes (>= ~2K elements); cols: one group and `hr` rows
  // of stage 2 (~256 threads of work)
  const int unit = (!rows && v4) ? 4 : 1;
  int nsplit = 1, r3 = p.E3, threads = 256;
  size_t smem = 0;
  if (rows) {
    p.U1 = v4 ? p.E1 / 4 : p.E1;
    p.E1p = p.E1 | 1;  // odd pitch: a thread per row reads conflict-free
    // whole groups in one block (no ticket) when there are enough groups to fill the SMs, else
    // split the planes so that ~4 blocks per SM run; shared memory caps the planes per block
    const int64_t plane = (int64_t)p.E2 * p.E1p;
    // planes per block: a 48 KB plane budget (4 blocks per SM) measured best -- 96 KB: +0.16 ms per
    // ResNet-50 step, 12-24 KB: more tickets and tail (profiles/r2/experiments/rc_smem_sweep.txt)
    static const int64_t budget = getenv("PB_RC_SMEM_KB") ? atoi(getenv("PB_RC_SMEM_KB")) : 48;  // experiment hooks
    static const int64_t tgt = getenv("PB_RC_TARGET") ? atoi(getenv("PB_RC_TARGET")) : 4;
    const int64_t target = tgt * (int64_t)num_sms();
    int64_t pp = G * 2 >= target ? p.E3 : (p.E3 + (target + G - 1) / G - 1) / ((target + G - 1) / G);
    const int64_t cap = (budget * 1024 / 4 - 2 * (int64_t)p.E3 * (p.E2 + 1)) / plane;
    if (pp > cap) pp = cap > 1 ? cap : 1;
    if (pp > p.E3) pp = p.E3;
    if (pp < 1) pp = 1;
    r3 = (int)pp;
    nsplit = (p.E3 + r3 - 1) / r3;
    p.fU1 = FastDiv((uint32_t)p.U1);
    p.fE2 = FastDiv((uint32_t)p.E2);
    smem = sizeof(float) * (size_t)(r3 * p.E2 + r3 + r3 * plane);
    const int64_t units = (int64_t)r3 * p.E2 * p.U1;
    threads = units >= 1024 ? 256 : units >= 512 ? 128 : 64;
    if (nsplit > 1 && nstages == 3) {
      p.ws = (float*)workspace(sizeof(float) * G * p.E3);
      if (!p.ws) return fail(PB_ERR_OOM, "pb_reduce_chain: workspace");
    }
  } else {
    // one pass of <= 256 (row, column-unit) pairs per block, and >= ~4 blocks per SM: few groups
    // split their rows further (the threads then split the stage-1 axis into slices)
    const int wu = p.E3 / unit;
    static const int pairs = getenv("PB_RC_COLS_PAIRS") ? atoi(getenv("PB_RC_COLS_PAIRS")) : 256;  // experiment hook
    int hr = wu >= pairs ? 1 : pairs / wu;  // one pass of <= `pairs` (row, column-unit) pairs per block
    if (hr > p.E2) hr = p.E2;
    r3 = hr;
    nsplit = (p.E2 + hr - 1) / hr;
    const int64_t npairs = (int64_t)hr * wu;
    int P = (int)(npairs >= 256 ? 256 : (npairs + 31) / 32 * 32);
    int S = 256 / P;
    if (S > p.E1 / 16) S = p.E1 / 16;
    if (S < 1) S = 1;
    p.P = P;
    p.S = S;
    threads = P * S;
    smem = sizeof(float) * (((size_t)p.E3 * hr + p.E3 + 1) & ~(size_t)1);
    if (S > 1) smem += sizeof(double) * (size_t)P * S * unit;
    if (nsplit > 1) {
      p.ws = (float*)workspace(sizeof(double) * G * nsplit * p.E3);
      if (!p.ws) return fail(PB_ERR_OOM, "pb_reduce_chain: workspace");
    }
  }
  p.r3 = r3;
  p.nsplit = nsplit;
  if (nsplit > 1) {
    p.tick = tick_counters(G);
    if (!p.tick) return fail(PB_ERR_UNSUPPORTED, "pb_reduce_chain: more groups than ticket counters");
  }
  if (smem > 112 * 1024) return fail(PB_ERR_UNSUPPORTED, "pb_reduce_chain: stage tile exceeds shared memory");
  const int64_t grid = G * nsplit;
  if (grid >= ((int64_t)1 << 31)) return fail(PB_ERR_UNSUPPORTED, "pb_reduce_chain: grid");
  cudaStream_t s = compute_stream();
  const bool plain = nleaves == 1 && nsteps == 0 && head_kind == 0 && !p.is_bool[0];
  // product: one MUL of leaf 0 by itself (x0 * x0) or by leaf 1 (either side: IEEE a*b == b*a)
  static const bool interp_only = getenv("PB_RC_INTERP") != nullptr;  // experiment hook
  const bool product = !interp_only && nsteps == 1 && head_kind == 0 && steps[0].op == PB_MUL &&
                       ((nleaves == 1 && steps[0].kind == 3) || (nleaves == 2 && steps[0].kind == 1 && steps[0].leaf == 1)) &&
                       !p.is_bool[0] && (nleaves == 1 || !p.is_bool[1]);
  const int so = nsteps == 1 ? steps[0].op : -1, sk = nsteps == 1 ? steps[0].kind : -1;
  const bool one = !interp_only && nleaves == 1 && nsteps == 1 && head_kind == 0 && !p.is_bool[0] &&
                   ((sk == 0 && (so == 64 + PB_NEG || so == 64 + PB_ABS)) ||
                    (sk == 2 && (so == PB_ADD || so == PB_SUB || so == PB_MUL)));
  switch (plain ? 0 : product ? -nleaves : one ? -3 : nleaves) {
    case 0: launch_redchain<1, 1>(p, rows, v4, (int)grid, threads, smem, s); break;
    case -3: launch_redchain<1, 3>(p, rows, v4, (int)grid, threads, smem, s); break;
    case -1: launch_redchain<1, 2>(p, rows, v4, (int)grid, threads, smem, s); break;
    case -2: launch_redchain<2, 2>(p, rows, v4, (int)grid, threads, smem, s); break;
    case 1: launch_redchain<1, 0>(p, rows, v4, (int)grid, threads, smem, s); break;
    case 2: launch_redchain<2, 0>(p, rows, v4, (int)grid, threads, smem, s); break;
    case 3: launch_redchain<3, 0>(p, rows, v4, (int)grid, threads, smem, s); break;
    case 4: launch_redchain<4, 0>(p, rows, v4, (int)grid, threads, smem, s); break;
    default: launch_redchain<8, 0>(p, rows, v4, (int)grid, threads, smem, s); break;
  }
  PB_LAUNCHED();
  return PB_OK;
}


int pb_ew_chain_win(int nleaves, const pb_tensor* leaves, const pb_leaf_window* wins, int head_kind,
                    double head_scalar, int nsteps, const pb_chain_step* steps, const pb_tensor* out) {
  const int64_t n = numel(*out);
  if (n == 0) return PB_OK;
  if (nleaves < 1 || nleaves > kChainLeaves || nsteps < 0 || nsteps > kChainSteps)
    return fail(PB_ERR_ARG, "pb_ew_chain_win: bad chain shape");
  if (n >= ((int64_t)1 << 31) || !is_contiguous(*out) || (out->dtype != PB_F32 && out->dtype != PB_BOOL) ||
      out->ndim > 4 || out->ndim < 1)
    return fail(PB_ERR_UNSUPPORTED, "pb_ew_chain_win: output must be a dense f32/bool tensor of rank <= 4");
  const bool vec = out->shape[out->ndim - 1] % 4 == 0 && (out->ptr & 15) == 0;
  WinArgs a;
  memset(&a, 0, sizeof(a));
  ChainArgs& p = a.c;
  p.nleaves = nleaves;
  p.nsteps = nsteps;
  p.head_kind = head_kind;
  p.head_scalar = (float)head_scalar;
  p.out = (void*)(uintptr_t)out->ptr;
  p.out_bool = out->dtype == PB_BOOL;
  p.n = (uint32_t)(vec ? n / 4 : n);
  for (int k = 0; k < nsteps; ++k) {
    const pb_chain_step& c = steps[k];
    if (c.kind == 1 && (c.leaf < 0 || c.leaf >= nleaves)) return fail(PB_ERR_ARG, "pb_ew_chain_win: bad leaf index");
    p.step[k].op = (int16_t)c.op;
    p.step[k].kind = (int8_t)c.kind;
    p.step[k].side = (int8_t)c.side;
    p.step[k].leaf = (int8_t)c.leaf;
    p.step[k].to_bool = (int8_t)c.to_bool;
    p.step[k].scalar = (float)c.scalar;
  }
  const int pad = 4 - out->ndim;
  int64_t oshape[4];
  for (int d = 0; d < 4; ++d) oshape[d] = d < pad ? 1 : out->shape[d - pad];
  for (int l = 0; l < nleaves; ++l) {
    const pb_tensor& t = leaves[l];
    if (t.dtype != PB_F32 && t.dtype != PB_BOOL) return fail(PB_ERR_UNSUPPORTED, "pb_ew_chain_win: leaf dtype");
    p.leaf[l] = (const void*)(uintptr_t)t.ptr;
    p.is_bool[l] = t.dtype == PB_BOOL;
    const int off = 4 - t.ndim;
    if (off < 0) return fail(PB_ERR_ARG, "pb_ew_chain_win: leaf rank exceeds 4");
    for (int d = 0; d < 4; ++d) p.st[l][d] = 0;
    WinLeaf& w = a.w[l];
    w.on = wins && wins[l].on;
    if (w.on) {
      if (t.ndim != out->ndim) return fail(PB_ERR_ARG, "pb_ew_chain_win: a windowed leaf has the output's rank");
      w.fill = (float)wins[l].fill;
      for (int d = 0; d < 4; ++d) {
        const int k = d - pad;
        const int64_t mul = k < 0 ? 1 : wins[l].mul[k], dv = k < 0 ? 1 : wins[l].div[k];
        const int64_t wo = k < 0 ? 0 : wins[l].off[k], ext = k < 0 ? 1 : t.shape[k];
        if (dv < 1 || (dv & (dv - 1))) return fail(PB_ERR_UNSUPPORTED, "pb_ew_chain_win: window divisor not 2^k");
        // 32-bit index math: |i*mul - off| must fit
        if (mul < 0 || mul * oshape[d] + (wo < 0 ? -wo : wo) >= ((int64_t)1 << 30) || ext >= ((int64_t)1 << 30))
          return fail(PB_ERR_UNSUPPORTED, "pb_ew_chain_win: window coordinates exceed 32 bits");
        int sh = 0;
        while (((int64_t)1 << sh) < dv) ++sh;
        w.mul[d] = (int32_t)mul;
        w.off[d] = (int32_t)wo;
        w.shift[d] = sh;
        w.ext[d] = (int32_t)ext;
        p.st[l][d] = k < 0 ? 0 : t.strides[k];
      }
    } else {
      for (int k = 0; k < t.ndim; ++k) p.st[l][off + k] = t.shape[k] == 1 ? 0 : t.strides[k];
    }
  }
  a.d1 = FastDiv((uint32_t)oshape[1]);
  a.d2 = FastDiv((uint32_t)oshape[2]);
  a.d3 = FastDiv((uint32_t)oshape[3]);
  cudaStream_t s = compute_stream();
  if (jit_win(a, vec, nleaves, a.d1, a.d2, a.d3, s, (uint32_t)oshape[3])) {
    PB_LAUNCHED();
    return PB_OK;
  }
  const int grid = grid_for(p.n, 256, 2);
#define PB_WIN(K)                                              \
  if (vec) ew_chain_win<K><<<grid, 256, 0, s>>>(a);            \
  else ew_chain_win1<K><<<grid, 256, 0, s>>>(a);
  switch (nleaves) {
    case 1: PB_WIN(1) break;
    case 2: PB_WIN(2) break;
    case 3: PB_WIN(3) break;
    case 4: PB_WIN(4) break;
    case 5: PB_WIN(5) break;
    case 6: PB_WIN(6) break;
    case 7: PB_WIN(7) break;
    default: PB_WIN(8) break;
  }
#undef PB_WIN
  PB_LAUNCHED();
  return PB_OK;
}


static bool pad_fast_path(const pb_tensor* src, const int64_t* lo, const pb_scalar* value, const pb_tensor* out,
                          int* rc) {
  int64_t n = numel(*out);
  if (src->dtype != out->dtype || itemsize(out->dtype) != 4 || !is_contiguous(*out) || n >= ((int64_t)1 << 31))
    return false;
  PadFast p;
  p.src = (const uint32_t*)(uintptr_t)src->ptr;
  p.out = (uint32_t*)(uintptr_t)out->ptr;
  // merge an axis into its outer neighbour when neither is padded and src is contiguous across them
  int nd = 0;
  int64_t oext[PB_MAX_RANK], sstr[PB_MAX_RANK], sext[PB_MAX_RANK], l[PB_MAX_RANK];
  for (int k = 0; k < out->ndim; ++k) {
    int64_t e = out->shape[k], st = src->shape[k] == 1 ? 0 : src->strides[k];
    if (nd > 0 && lo[k] == 0 && e == src->shape[k] && l[nd - 1] == 0 && oext[nd - 1] == sext[nd - 1] &&
        sstr[nd - 1] == st * e) {
      oext[nd - 1] *= e;
      sext[nd - 1] *= e;
      sstr[nd - 1] = st;
      continue;
    }
    oext[nd] = e;
    sext[nd] = src->shape[k];
    sstr[nd] = st;
    l[nd] = lo[k];
    ++nd;
  }
  for (int k = 0; k < nd; ++k) {
    if (oext[k] >= ((int64_t)1 << 31) || l[k] >= ((int64_t)1 << 30) || sext[k] >= ((int64_t)1 << 31)) return false;
    p.ext[k] = FastDiv((uint32_t)oext[k]);
    p.sstr[k] = sstr[k];
    p.lo[k] = (int32_t)l[k];
    p.sext[k] = (int32_t)sext[k];
  }
  p.nd = nd;
  p.n = (uint32_t)n;
  uint32_t bits;
  if (out->dtype == PB_F32) {
    float f = scalar_as<float>(value);
    memcpy(&bits, &f, 4);
  } else {
    int32_t i = scalar_as<int32_t>(value);
    memcpy(&bits, &i, 4);
  }
  if (nd > 0 && n % 4 == 0 && out->ptr % 16 == 0)
    pad_fast4<<<grid_for(n / 4, 256), 256, 0, compute_stream()>>>(p, bits);
  else
    pad_fast<<<grid_for(n, 1024), 256, 0, compute_stream()>>>(p, bits);
  count_launch();
  cudaError_t e = cudaGetLastError();
  *rc = e == cudaSuccess ? PB_OK : cuda_fail(e, "pb_pad");
  return true;
}

int pb_pad(const pb_tensor* src, const int64_t* lo, const pb_scalar* value, const pb_tensor* out) {
  if (numel(*out) == 0) return PB_OK;
  {
    int rc;
    if (pad_fast_path(src, lo, value, out, &rc)) return rc;
  }
  PadArgs p;
  p.src = (const void*)(uintptr_t)src->ptr;
  p.out = (void*)(uintptr_t)out->ptr;
  p.dts = src->dtype;
  p.dto = out->dtype;
  p.ndim = out->ndim;
  p.n = numel(*out);
  if (p.n == 0) return PB_OK;
  for (int k = 0; k < out->ndim; ++k) {
    p.oshape[k] = out->shape[k];
    p.ostr[k] = out->strides[k];
    p.sshape[k] = src->shape[k];
    p.sstr[k] = src->strides[k];
    p.lo[k] = lo[k];
  }
  int grid = grid_for(p.n, 256, 4);
  cudaStream_t st = compute_stream();
  switch (out->dtype) {
    case PB_BOOL: pad_kernel<bool><<<grid, 256, 0, st>>>(p, scalar_as<bool>(value)); break;
    case PB_U8: pad_kernel<uint8_t><<<grid, 256, 0, st>>>(p, scalar_as<uint8_t>(value)); break;
    case PB_I32: pad_kernel<int32_t><<<grid, 256, 0, st>>>(p, scalar_as<int32_t>(value)); break;
    case PB_I64: pad_kernel<int64_t><<<grid, 256, 0, st>>>(p, scalar_as<int64_t>(value)); break;
    case PB_F32: pad_kernel<float><<<grid, 256, 0, st>>>(p, scalar_as<float>(value)); break;
    default: pad_kernel<double><<<grid, 256, 0, st>>>(p, scalar_as<double>(value)); break;
  }
  PB_LAUNCHED();
  return PB_OK;
}

int pb_fill(const pb_tensor* out, const pb_scalar* v) {
  int64_t n = numel(*out);
  if (n == 0) return PB_OK;
  int grid = grid_for(n, 256, 4);
  cudaStream_t st = compute_stream();
  void* p = (void*)(uintptr_t)out->ptr;
  switch (out->dtype) {
    case PB_BOOL: fill_kernel<bool><<<grid, 256, 0, st>>>((bool*)p, n, scalar_as<bool>(v)); break;
    case PB_U8: fill_kernel<uint8_t><<<grid, 256, 0, st>>>((uint8_t*)p, n, scalar_as<uint8_t>(v)); break;
    case PB_I32: fill_kernel<int32_t><<<grid, 256, 0, st>>>((int32_t*)p, n, scalar_as<int32_t>(v)); break;
    case PB_I64: fill_kernel<int64_t><<<grid, 256, 0, st>>>((int64_t*)p, n, scalar_as<int64_t>(v)); break;
    case PB_F32: fill_kernel<float><<<grid, 256, 0, st>>>((float*)p, n, scalar_as<float>(v)); break;
    default: fill_kernel<double><<<grid, 256, 0, st>>>((double*)p, n, scalar_as<double>(v)); break;
  }
  PB_LAUNCHED();
  return PB_OK;
}

int pb_arange(const pb_tensor* out) {
  int64_t n = numel(*out);
  if (n == 0) return PB_OK;
  if (out->dtype != PB_I64) return fail(PB_ERR_ARG, "pb_arange: i64 only");
  arange_kernel<<<grid_for(n, 256, 4), 256, 0, compute_stream()>>>((int64_t*)(uintptr_t)out->ptr, n);
  PB_LAUNCHED();
  return PB_OK;
}

int pb_check(int what, const pb_tensor* a, int32_t* result) {
  *result = 0;
  if (numel(*a) == 0) return PB_OK;
  int32_t* flag = (int32_t*)workspace(16);
  if (!flag) return fail(PB_ERR_OOM, "pb_check: no workspace");
  PB_CUDA(cudaMemsetAsync(flag, 0, 4, compute_stream()));
  RowArgs r = make_rows(a, a, nullptr);
  if (a->dtype == PB_F32 || a->dtype == PB_F64)
    check_kernel<double><<<rows_grid(r), 256, 0, compute_stream()>>>(r.a, a->dtype, r, what, flag);
  else
    check_kernel<int64_t><<<rows_grid(r), 256, 0, compute_stream()>>>(r.a, a->dtype, r, what, flag);
  PB_LAUNCHED();
  PB_CUDA(cudaMemcpyAsync(result, flag, 4, cudaMemcpyDeviceToHost, compute_stream()));
  PB_CUDA(cudaStreamSynchronize(compute_stream()));
  return PB_OK;
}

int pb_sgd(int n, const uint64_t* params_in, const uint64_t* params_out, const uint64_t* grads,
           const uint64_t* vels_in, const uint64_t* vels_out, const int64_t* numels, float lr, float momentum,
           float wd) {
  const uint64_t* vels = vels_out;
  const uint64_t* params = params_out;
  for (int base = 0; base < n; base += kMaxTensors) {
    MultiTable t;
    t.count = 0;
    int32_t items = 0;
    for (int i = base; i < n && t.count < kMaxTensors; ++i) {
      int k = t.count++;
      t.p[k] = (float*)(uintptr_t)params[i];
      t.pin[k] = (const float*)(uintptr_t)params_in[i];
      t.g[k] = (const float*)(uintptr_t)grads[i];
      t.v[k] = vels ? (float*)(uintptr_t)vels[i] : nullptr;
      t.vin[k] = vels_in ? (const float*)(uintptr_t)vels_in[i] : nullptr;
      t.n[k] = numels[i];
      t.dst[k] = 0;
      t.first[k] = items;
      items += (int32_t)((numels[i] + kItem - 1) / kItem);
    }
    t.first[t.count] = items;
    if (items == 0) continue;
    int grid = items < num_sms() * 8 ? items : num_sms() * 8;
    sgd_kernel<<<grid, 256, 0, compute_stream()>>>(t, lr, momentum, wd, momentum != 0.0f && vels, wd != 0.0f);
    PB_LAUNCHED();
  }
  return PB_OK;
}

int pb_bucket_pack(int n, const uint64_t* srcs, const int64_t* numels, uint64_t bucket) {
  int64_t acc = 0;
  for (int base = 0; base < n; base += kMaxTensors) {
    MultiTable t;
    t.count = 0;
    int32_t items = 0;
    for (int i = base; i < n && t.count < kMaxTensors; ++i) {
      int k = t.count++;
      t.p[k] = nullptr;
      t.pin[k] = nullptr;
      t.v[k] = nullptr;
      t.vin[k] = nullptr;
      t.g[k] = (const float*)(uintptr_t)srcs[i];
      t.n[k] = numels[i];
      t.dst[k] = acc;
      acc += numels[i];
      t.first[k] = items;
      items += (int32_t)((numels[i] + kItem - 1) / kItem);
    }
    t.first[t.count] = items;
    if (items == 0) continue;
    int grid = items < num_sms() * 8 ? items : num_sms() * 8;
    pack_kernel<<<grid, 256, 0, compute_stream()>>>(t, (float*)(uintptr_t)bucket);
    PB_LAUNCHED();
  }
  return PB_OK;
}

int pb_scale_f32(uint64_t buf, int64_t n, float divisor) {
  if (n <= 0) return PB_OK;
  scale_kernel<<<grid_for(n, 256, 4), 256, 0, compute_stream()>>>((float*)(uintptr_t)buf, n, divisor);
  PB_LAUNCHED();
  return PB_OK;
}

}  // extern "C"

extern "C" int pb_fastdiv_probe(uint64_t a, uint64_t b, uint64_t out, int64_t n) {
  if (n <= 0) return PB_OK;
  fastdiv_probe<<<grid_for(n, 256, 4), 256, 0, compute_stream()>>>((const float*)(uintptr_t)a, (const float*)(uintptr_t)b,
                                                                    (float*)(uintptr_t)out, n);
  PB_LAUNCHED();
  return PB_OK;
}

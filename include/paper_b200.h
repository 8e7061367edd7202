/*
 * paper_b200.h — C ABI of libpaper_b200.so, the B200 backend behind the Flashlight
 * (arXiv 2201.12465) reference's primitive table.
 *
 * The reference's drop-in boundary is Python: ``Backend.execute(OpCall, adapters)``
 * (minml/registry.py:97-141; template minml/eager.py:33-64) dispatching to one numpy
 * kernel per primitive (minml/kernels.py:272-314) with one managed allocation per op
 * (minml/memory.py:126-157).  Each entry point below replaces one row of that table;
 * the Python GpuBackend (paper_2201_12465_b200/gpu/backend.py) binds them with ctypes.
 * INTEGRATION.md shows the equivalent ctypes stub a reference maintainer would add.
 *
 * Conventions: every function returns 0 on success or a nonzero pb_status; the text of
 * the last error on the calling thread is pb_last_error().  Device pointers travel as
 * uint64_t.  Kernels are enqueued on the backend's compute stream (pb_stream(0)) and
 * never block, except the documented host transfers / checks.  No torch types appear.
 */
#ifndef PAPER_B200_H
#define PAPER_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum pb_status { PB_OK = 0, PB_ERR_CUDA = 1, PB_ERR_ARG = 2, PB_ERR_OOM = 3, PB_ERR_ALLOC = 4,
                 PB_ERR_DOMAIN = 5, PB_ERR_NCCL = 6, PB_ERR_UNSUPPORTED = 7,
                 PB_ERR_TIMEOUT = 8 };

/* element types; codes equal the reference's promotion rank (minml/dtypes.py:41-46) */
enum pb_dtype { PB_BOOL = 0, PB_U8 = 1, PB_I32 = 2, PB_I64 = 3, PB_F32 = 4, PB_F64 = 5 };

#define PB_MAX_RANK 8

/* A strided view: element (i0..in-1) lives at ptr + sum(ik * strides[k]) * itemsize. */
typedef struct pb_tensor {
  uint64_t ptr;
  int32_t dtype;
  int32_t ndim;
  int64_t shape[PB_MAX_RANK];
  int64_t strides[PB_MAX_RANK]; /* in elements; 0 marks a broadcast axis */
} pb_tensor;

/* A weak Python scalar operand (minml/_tensor.py:90-102, kernels.py:35-42). */
typedef struct pb_scalar {
  int32_t kind; /* 0 float (f), 1 int (i), 2 bool (i) */
  int32_t pad_;
  double f;
  int64_t i;
} pb_scalar;

/* ---- runtime --------------------------------------------------------------------- */
int pb_init(int device);                 /* select device, create streams */
int pb_device_count(void);               /* 0 when no device / driver */
const char* pb_last_error(void);
int pb_synchronize(void);                /* wait for the compute stream */
uint64_t pb_stream(int which);           /* 0 compute, 1 comm, 2 copy (cudaStream_t) */
int pb_h2d(uint64_t dst, const void* src, uint64_t nbytes); /* pinned staging, async */
int pb_d2h(void* dst, uint64_t src, uint64_t nbytes);       /* blocking */
/* pipelined transfers (training.CapturedStep.run; the reference's read-ahead Prefetch,
   minml/data.py:112-145): h2d through the pinned staging ring on stream `stream`
   (0 compute, 2 copy); d2h posted into pinned slot 0..7 (<= 1 MiB) on the compute stream,
   fetched later (waits for that copy only) */
int pb_h2d_on(uint64_t dst, const void* src, uint64_t nbytes, int stream);
int pb_d2h_post(uint64_t src, uint64_t nbytes, int slot);
int pb_d2h_fetch(int slot, void* dst, uint64_t nbytes);
/* page-locked host buffers: pb_h2d / pb_h2d_on DMA straight from them (no staging copy) */
void* pb_host_alloc(uint64_t nbytes);   /* NULL on failure (pb_last_error) */
int pb_host_free(void* p);
int pb_stream_sync(int stream);          /* wait for one stream (0 compute, 1 comm, 2 copy) */
int pb_d2d(uint64_t dst, uint64_t src, uint64_t nbytes);    /* async */
int pb_event_record(int stream_from, int stream_to);        /* stream_to waits on stream_from */
int pb_graph_begin(void);                 /* start capturing the compute stream */
int pb_graph_end(uint64_t* graph_exec);   /* finish capture, instantiate */
int pb_graph_launch(uint64_t graph_exec);
int pb_graph_destroy(uint64_t graph_exec);
int pb_timer(int op, uint64_t* handle, float* ms); /* 0 create+record start,1 record stop,2 elapsed,3 destroy */

/* ---- caching device allocator (replaces minml/memory.py:86-347) ------------------- */
enum pb_policy { PB_POLICY_NATIVE = 0, PB_POLICY_CACHING = 1, PB_POLICY_SPLIT = 2 };
typedef struct pb_mm_stats {
  uint64_t live_bytes_requested, live_bytes_granted, peak_granted, cache_bytes;
  uint64_t alloc_count, free_count, internal_fragmentation, peak_internal_fragmentation;
  uint64_t live_blocks;
  double external_fragmentation_ratio;
} pb_mm_stats;
typedef struct pb_mm_block {
  uint64_t id, ptr, requested_bytes, granted_bytes, bin_size;
  int32_t op_tag, pool;
} pb_mm_block;

void* pb_mm_create(int policy, uint64_t split_threshold, uint64_t capacity /*0 = none*/, int simulate);
void pb_mm_destroy(void* mm);
int pb_mm_alloc(void* mm, uint64_t nbytes, int32_t op_tag, pb_mm_block* out);
int pb_mm_free(void* mm, uint64_t block_id);
int pb_mm_record_stream(void* mm, uint64_t block_id, int stream);
int pb_mm_stats_get(void* mm, pb_mm_stats* out);
uint64_t pb_mm_flush(void* mm);          /* returns cached blocks released */
int pb_mm_pool(void* mm, int pool);      /* route allocations to a private pool (graphs); 0 = default */
uint64_t pb_bin_size(uint64_t nbytes);
uint64_t pb_round_up(uint64_t nbytes);

/* ---- primitive kernels (minml/kernels.py) ------------------------------------------ */
enum pb_binop { PB_ADD = 0, PB_SUB, PB_MUL, PB_DIV, PB_POW, PB_MIN, PB_MAX, PB_EQ, PB_LT, PB_GT,
                PB_AND, PB_OR };
enum pb_unop { PB_NEG = 0, PB_ABS, PB_EXP, PB_LOG, PB_SQRT, PB_SIN, PB_COS, PB_TANH, PB_NOT, PB_CAST };
enum pb_redop { PB_SUM = 0, PB_RMAX, PB_RMIN, PB_ARGMAX };

/* out = op(a, b) computed in dtype `compute` (numpy's result type), cast to out->dtype.
 * Either operand may be replaced by a scalar: pass a == NULL or b == NULL plus `s`. */
int pb_binary(int op, const pb_tensor* a, const pb_tensor* b, const pb_scalar* s, int compute,
              const pb_tensor* out);                                    /* kernels.py:88-113 */
int pb_unary(int op, const pb_tensor* a, int compute, const pb_tensor* out); /* kernels.py:119-129 */
int pb_copy(const pb_tensor* src, const pb_tensor* dst);   /* strided copy + cast: reshape/transpose/slice/concat */
int pb_pad(const pb_tensor* src, const int64_t* lo, const pb_scalar* value, const pb_tensor* out); /* :265-269 */
int pb_fill(const pb_tensor* out, const pb_scalar* value);                /* kernels.py:54-58 */
int pb_arange(const pb_tensor* out);                                      /* kernels.py:61-62 */
int pb_rand(int normal, uint64_t seed, uint64_t offset, const pb_tensor* out); /* kernels.py:65-74, rng.py */
/* pb_rand with counter offset = *(uint64_t*)base_ptr + delta read on the device: a fill recorded
 * into a CUDA graph draws the counter range the host reserved for each replay
 * (minml/_tensor.py:362-368 reserve, rng.py:16-51); pb_counter_add advances that counter. */
int pb_rand_dev(int normal, uint64_t seed, uint64_t base_ptr, uint64_t delta, const pb_tensor* out);
int pb_counter_add(uint64_t counter_ptr, uint64_t inc);
/* test probe: out[i] = a[i] / b[i] by the reciprocal + exact-residual path the per-row
 * broadcast kernel uses (must equal IEEE division bit for bit) */
int pb_fastdiv_probe(uint64_t a, uint64_t b, uint64_t out, int64_t n);
int pb_reduce(int op, const pb_tensor* a, int axis /* -1 = all */, const pb_tensor* out); /* :139-160 */
/* pb_reduce then out = op(result, scalar) (or op(scalar, result)) in f32, op in add/sub/mul/div:
   the reference's mean = sum / n (minml/ops.py:33-36) fused; backend-internal (planned fusion) */
int pb_reduce_epi(int op, const pb_tensor* a, int axis, const pb_tensor* out, int epi_op, float scalar,
                  int scalar_left);
int pb_check(int what, const pb_tensor* a, int32_t* result); /* 0: any zero, 1: any negative (blocking) */
int pb_matmul(const pb_tensor* a, const pb_tensor* b, const pb_tensor* out); /* kernels.py:166-173 */
typedef struct pb_conv {
  int32_t stride_h, stride_w, pad_h, pad_w;
} pb_conv;
int pb_conv2d(const pb_tensor* x, const pb_tensor* w, const pb_tensor* bias /* nullable */,
              const pb_conv* p, const pb_tensor* out);                     /* kernels.py:197-210 */
int pb_conv2d_grad_input(const pb_tensor* g, const pb_tensor* w, const pb_conv* p,
                         const pb_tensor* out);                            /* kernels.py:213-228 */
int pb_conv2d_grad_weight(const pb_tensor* x, const pb_tensor* g, const pb_conv* p,
                          const pb_tensor* out);                           /* kernels.py:231-239 */
/* Fused elementwise chain (backend-internal fusion, SURVEY §8f f1 / minml/deferred.py:146-163):
 * v = head (leaf 0 broadcast to out, or head_scalar); for each step v = op(v, x) or op(x, v)
 * with x a leaf (broadcast), a scalar, or v itself; unary steps v = op(v).  f32/bool leaves
 * (bool = 0/1), every step in f32 with the unfused kernels' functors: bit-identical to running
 * the primitives one at a time.  out: dense f32 or bool. */
typedef struct pb_chain_step {
  int32_t op;      /* pb_binop, or 64 + pb_unop */
  int32_t kind;    /* 0 unary, 1 leaf, 2 scalar, 3 self */
  int32_t side;    /* 0: op(v, x), 1: op(x, v) */
  int32_t leaf;
  int32_t to_bool; /* PB_CAST target: 1 bool, 0 f32 */
  int32_t pad_;
  double scalar;
} pb_chain_step;
int pb_ew_chain(int nleaves, const pb_tensor* leaves, int head_kind, double head_scalar, int nsteps,
                const pb_chain_step* steps, const pb_tensor* out);
/* The chain above that also stores its running value after tap_after[i] steps (1..nsteps) into
 * taps[i] (dense, 16-byte aligned f32 of out's size): a multi-use intermediate of the chain is
 * written by the pass that consumes it instead of by a pass of its own (round 2 "taps").  JIT
 * kernels only: PB_ERR_UNSUPPORTED, with nothing launched, when the chain cannot be specialised. */
int pb_ew_chain_taps(int nleaves, const pb_tensor* leaves, int head_kind, double head_scalar, int nsteps,
                     const pb_chain_step* steps, int ntaps, const int* tap_after, const pb_tensor* taps,
                     const pb_tensor* out);
/* Chain kernels specialised per structure with NVRTC (straight-line code, the same functors and
 * flags as the interpreter: bit-identical); this returns how many are compiled and cached, or -1
 * when the JIT is off (PB_CHAIN_JIT=0 or libnvrtc missing: the interpreter runs every chain). */
int pb_chain_jit_kernels(void);
/* Fused multi-stage f32 sum over an elementwise chain (minml/nn.py:288-306
 * BatchNorm's x.mean(3).mean(2).mean(0) and minml/autograd.py:290-297 _unbroadcast's
 * sum(0).sum(2).sum(3)): the source is the chain above evaluated over src_shape (a plain tensor
 * is one leaf and no steps); stage k sums source axis stages[k].axis (f64 accumulation, one f32
 * rounding) and applies its optional scalar epilogue, as pb_reduce_epi would.  out: dense f32
 * holding the kept axes in order.  Supported (else PB_ERR_UNSUPPORTED, nothing launched): 2-3
 * stages whose first two are (innermost, next) -- "rows" -- or 3 stages whose last is the
 * innermost axis -- "cols". */
/* Windowed chain leaves: leaf l reads its source through a per-axis affine map, not a
 * materialised pad -- for output index i, j = i*mul - off; the value is src[j / div] when j >= 0,
 * j % div == 0 and j / div < the source extent, else `fill`.  A pad is (mul 1, off lo, div 1),
 * a zero-stuffing pad (minml/autograd.py:667-693) div = step, a strided slice of a padded tensor
 * mul = step.  Leaves with on == 0 broadcast as in pb_ew_chain.  Output rank <= 4. */
typedef struct pb_leaf_window {
  int32_t on;
  int32_t pad_;
  double fill;
  int64_t mul[4], off[4], div[4]; /* per source/output axis */
} pb_leaf_window;
int pb_ew_chain_win(int nleaves, const pb_tensor* leaves, const pb_leaf_window* wins, int head_kind,
                    double head_scalar, int nsteps, const pb_chain_step* steps, const pb_tensor* out);
typedef struct pb_red_stage {
  int32_t axis;     /* source axis */
  int32_t epi_op;   /* -1 none, else PB_ADD/SUB/MUL/DIV */
  int32_t epi_left; /* scalar on the left */
  float scalar;
} pb_red_stage;
int pb_reduce_chain(int nleaves, const pb_tensor* leaves, int head_kind, double head_scalar, int nsteps,
                    const pb_chain_step* steps, int src_ndim, const int64_t* src_shape, int nstages,
                    const pb_red_stage* stages, const pb_tensor* out);
/* In-place multi-tensor SGD (minml/optim.py:64-72 op for op): for each i,
 * g' = g + wd*p (if wd); v = v*mu + g' (if mu, else v := g'); p = p - v*lr.  f32 only. */
int pb_sgd(int n, const uint64_t* params_in, const uint64_t* params_out, const uint64_t* grads,
           const uint64_t* vels_in, const uint64_t* vels_out, const int64_t* numels, float lr,
           float momentum, float weight_decay);  /* out may alias in (in-place update) */
/* Pack / unpack gradient buckets (data-parallel sync) and scale by 1/world. */
int pb_bucket_pack(int n, const uint64_t* srcs, const int64_t* numels, uint64_t bucket);
int pb_scale_f32(uint64_t buf, int64_t n, float divisor); /* buf[i] = buf[i] / divisor */

/* ---- NCCL (replaces minml/distributed.py:129-175) ---------------------------------- */
int pb_nccl_unique_id(uint8_t out[128]);
void* pb_nccl_init(int nranks, int rank, const uint8_t id[128]);
int pb_nccl_destroy(void* comm);
/* op: 0 sum, 1 max, 2 avg; dtype pb_dtype; runs on the comm stream after a fence on compute */
int pb_nccl_allreduce(void* comm, uint64_t sendbuf, uint64_t recvbuf, uint64_t count, int dtype, int op);
int pb_nccl_broadcast(void* comm, uint64_t sendbuf, uint64_t recvbuf, uint64_t count, int dtype, int root);
int pb_nccl_allgather(void* comm, uint64_t sendbuf, uint64_t recvbuf, uint64_t count, int dtype);
int pb_nccl_wait(void* comm);  /* compute stream waits for everything enqueued on the comm stream */
/* Collective watchdog (the reference's CollectiveTimeout, minml/distributed.py:23,93-105): the
 * host waits at most timeout_ms for the comm stream's queued work; on an NCCL async error or the
 * deadline the communicator is aborted (ncclCommAbort -- a hung peer would otherwise block the
 * process forever) and PB_ERR_NCCL / PB_ERR_TIMEOUT is returned.  comm may be NULL (no abort). */
int pb_nccl_sync(void* comm, int64_t timeout_ms);
/* test hook: occupy the comm stream for ms milliseconds (a stand-in for a peer that never arrives) */
int pb_debug_stall_comm(int64_t ms);

/* ---- NVTX ranges: step phases on an Nsight timeline (no-ops unless a tool is attached) ---- */
int pb_nvtx_push(const char* name);
int pb_nvtx_pop(void);

/* ---- introspection ------------------------------------------------------------------ */
uint64_t pb_launch_count(void);  /* kernels launched by this library so far */
int pb_gemm_path(void);          /* 2: tcgen05 with TMA-fed convs (default), 1: SIMT-fed tcgen05 only, 0: SIMT */
int pb_set_gemm_path(int path);

#ifdef __cplusplus
}
#endif
#endif

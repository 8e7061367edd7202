// Runtime plumbing: device selection, streams, errors, scratch, host<->device transfers,
// CUDA-graph capture and event timers.
#include <cuda_runtime.h>
#include <atomic>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>
#include <nvtx3/nvToolsExt.h>
#include "common.cuh"

namespace pb {

static thread_local std::string g_error;
static std::mutex g_mu;
static bool g_inited = false;
static int g_device = -1;
static int g_sms = 148;
static cudaStream_t g_streams[3] = {nullptr, nullptr, nullptr};
static std::atomic<uint64_t> g_launches{0};

void set_error(const std::string& msg) { g_error = msg; }
int fail(int code, const std::string& msg) {
  g_error = msg;
  return code;
}
int cuda_fail(cudaError_t e, const char* where) {
  g_error = std::string(where) + ": " + cudaGetErrorString(e);
  return PB_ERR_CUDA;
}
cudaStream_t compute_stream() { return g_streams[0]; }
cudaStream_t comm_stream() { return g_streams[1]; }
cudaStream_t copy_stream() { return g_streams[2]; }
int num_sms() { return g_sms; }
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

// ---- scratch ---------------------------------------------------------------------------
static void* g_ws = nullptr;
static size_t g_ws_bytes = 0;
static std::vector<void*> g_ws_retired;  // kept alive: CUDA graphs may have recorded them
void* workspace(size_t bytes) {
  if (bytes <= g_ws_bytes) return g_ws;
  size_t want = bytes < ((size_t)64 << 20) ? ((size_t)64 << 20) : bytes + (bytes >> 2);
  if (g_ws) g_ws_retired.push_back(g_ws);
  g_ws = nullptr;
  g_ws_bytes = 0;
  if (cudaMalloc(&g_ws, want) != cudaSuccess) return nullptr;
  g_ws_bytes = want;
  return g_ws;
}

// zeroed per-group ticket counters for single-launch multi-block reductions; every user
// resets the counters it took back to zero, so the buffer is all-zero between kernels
static unsigned* g_ticks = nullptr;
unsigned* tick_counters(int64_t n) { return n <= kTickCounters ? g_ticks : nullptr; }

// ---- index helpers -----------------------------------------------------------------------
int64_t numel(const pb_tensor& t) {
  int64_t n = 1;
  for (int k = 0; k < t.ndim; ++k) n *= t.shape[k];
  return n;
}
bool is_contiguous(const pb_tensor& t) {
  int64_t expect = 1;
  for (int k = t.ndim - 1; k >= 0; --k) {
    if (t.shape[k] != 1 && t.strides[k] != expect) return false;
    expect *= t.shape[k];
  }
  return true;
}
void coalesce(Dims& d, int nops) {
  // drop extent-1 axes
  int w = 0;
  for (int k = 0; k < d.ndim; ++k) {
    if (d.shape[k] == 1) continue;
    d.shape[w] = d.shape[k];
    for (int o = 0; o < nops; ++o) d.st[o][w] = d.st[o][k];
    ++w;
  }
  d.ndim = w;
  if (d.ndim <= 1) {
    if (d.ndim == 0) {
      d.ndim = 1;
      d.shape[0] = 1;
      for (int o = 0; o < nops; ++o) d.st[o][0] = 0;
    }
    return;
  }
  // merge axis k-1 into k when every operand steps contiguously across the boundary
  w = 0;
  for (int k = 1; k < d.ndim; ++k) {
    bool ok = true;
    for (int o = 0; o < nops; ++o)
      if (d.st[o][w] != d.st[o][k] * d.shape[k]) ok = false;
    if (ok) {
      d.shape[w] *= d.shape[k];
      for (int o = 0; o < nops; ++o) d.st[o][w] = d.st[o][k];
    } else {
      ++w;
      d.shape[w] = d.shape[k];
      for (int o = 0; o < nops; ++o) d.st[o][w] = d.st[o][k];
    }
  }
  d.ndim = w + 1;
}

// ---- pinned staging ring for host->device copies --------------------------------------
struct Stage {
  void* host = nullptr;
  size_t cap = 0;
  cudaEvent_t ev = nullptr;
  bool pending = false;
};
static const int kStages = 4;
static const size_t kStageBytes = (size_t)32 << 20;
static Stage g_stage[kStages];
static int g_stage_next = 0;
// ---- posted device->host result slots ------------------------------------------------
struct Post {
  void* host = nullptr;
  cudaEvent_t ev = nullptr;
  uint64_t bytes = 0;
};
static const int kPostSlots = 8;
static const size_t kPostBytes = (size_t)1 << 20;
static Post g_post[kPostSlots];

}  // namespace pb

using namespace pb;

extern "C" {

int pb_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int pb_init(int device) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_inited) {
    if (device != g_device) return fail(PB_ERR_ARG, "pb_init: already initialised on another device");
    return PB_OK;
  }
  PB_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  PB_CUDA(cudaGetDeviceProperties(&prop, device));
  g_sms = prop.multiProcessorCount;
  for (int i = 0; i < 3; ++i) PB_CUDA(cudaStreamCreateWithFlags(&g_streams[i], cudaStreamNonBlocking));
  for (int i = 0; i < kStages; ++i) {
    PB_CUDA(cudaHostAlloc(&g_stage[i].host, kStageBytes, cudaHostAllocDefault));
    g_stage[i].cap = kStageBytes;
    PB_CUDA(cudaEventCreateWithFlags(&g_stage[i].ev, cudaEventDisableTiming));
  }
  PB_CUDA(cudaMalloc(&g_ticks, sizeof(unsigned) * kTickCounters));
  PB_CUDA(cudaMemset(g_ticks, 0, sizeof(unsigned) * kTickCounters));
  g_device = device;
  g_inited = true;
  return PB_OK;
}

const char* pb_last_error(void) { return g_error.c_str(); }

int pb_synchronize(void) {
  PB_CUDA(cudaStreamSynchronize(g_streams[0]));
  PB_CUDA(cudaStreamSynchronize(g_streams[1]));
  return PB_OK;
}

uint64_t pb_stream(int which) { return (uint64_t)(uintptr_t)g_streams[(which >= 0 && which < 3) ? which : 0]; }

uint64_t pb_launch_count(void) { return g_launches.load(); }

int pb_h2d(uint64_t dst, const void* src, uint64_t nbytes) { return pb_h2d_on(dst, src, nbytes, 0); }

int pb_h2d_on(uint64_t dst, const void* src, uint64_t nbytes, int stream) {
  if (stream < 0 || stream > 2) return fail(PB_ERR_ARG, "pb_h2d_on: stream must be 0, 1 or 2");
  if (nbytes == 0) return PB_OK;
  cudaPointerAttributes attr;
  if (cudaPointerGetAttributes(&attr, src) == cudaSuccess && attr.type == cudaMemoryTypeHost) {
    // page-locked source (pb_host_alloc): one DMA, no staging copy on the host
    PB_CUDA(cudaMemcpyAsync((void*)(uintptr_t)dst, src, nbytes, cudaMemcpyHostToDevice, g_streams[stream]));
    return PB_OK;
  }
  cudaGetLastError();
  const char* s = (const char*)src;
  uint64_t off = 0;
  while (off < nbytes) {
    Stage& st = g_stage[g_stage_next];
    g_stage_next = (g_stage_next + 1) % kStages;
    if (st.pending) PB_CUDA(cudaEventSynchronize(st.ev));
    size_t len = (size_t)(nbytes - off) < st.cap ? (size_t)(nbytes - off) : st.cap;
    std::memcpy(st.host, s + off, len);
    PB_CUDA(cudaMemcpyAsync((void*)(uintptr_t)(dst + off), st.host, len, cudaMemcpyHostToDevice, g_streams[stream]));
    PB_CUDA(cudaEventRecord(st.ev, g_streams[stream]));
    st.pending = true;
    off += len;
  }
  return PB_OK;
}

int pb_d2h(void* dst, uint64_t src, uint64_t nbytes) {
  if (nbytes == 0) return PB_OK;
  PB_CUDA(cudaMemcpyAsync(dst, (const void*)(uintptr_t)src, nbytes, cudaMemcpyDeviceToHost, g_streams[0]));
  PB_CUDA(cudaStreamSynchronize(g_streams[0]));
  return PB_OK;
}

// posted device->host reads: a pinned slot per outstanding result, completed by an event, so
// the host can read step i's loss while step i+1 is already queued behind it
int pb_d2h_post(uint64_t src, uint64_t nbytes, int slot) {
  if (slot < 0 || slot >= kPostSlots || nbytes > kPostBytes) return fail(PB_ERR_ARG, "pb_d2h_post: bad slot or size");
  Post& p = g_post[slot];
  if (!p.host) {
    // every slot at once: a page-locked allocation is slow and can stall the host, which must
    // not happen inside a pipelined run that first touches slot k at step k
    for (int i = 0; i < kPostSlots; ++i) {
      if (g_post[i].host) continue;
      PB_CUDA(cudaHostAlloc(&g_post[i].host, kPostBytes, cudaHostAllocDefault));
      PB_CUDA(cudaEventCreateWithFlags(&g_post[i].ev, cudaEventDisableTiming));
    }
  }
  if (nbytes) PB_CUDA(cudaMemcpyAsync(p.host, (const void*)(uintptr_t)src, nbytes, cudaMemcpyDeviceToHost, g_streams[0]));
  PB_CUDA(cudaEventRecord(p.ev, g_streams[0]));
  p.bytes = nbytes;
  return PB_OK;
}

void* pb_host_alloc(uint64_t nbytes) {
  void* p = nullptr;
  if (cudaHostAlloc(&p, nbytes ? nbytes : 1, cudaHostAllocDefault) != cudaSuccess) {
    cudaGetLastError();
    set_error("pb_host_alloc: cudaHostAlloc failed");
    return nullptr;
  }
  return p;
}

int pb_host_free(void* p) {
  if (p) PB_CUDA(cudaFreeHost(p));
  return PB_OK;
}

int pb_stream_sync(int stream) {
  if (stream < 0 || stream > 2) return fail(PB_ERR_ARG, "pb_stream_sync: stream must be 0, 1 or 2");
  PB_CUDA(cudaStreamSynchronize(g_streams[stream]));
  return PB_OK;
}

int pb_d2h_fetch(int slot, void* dst, uint64_t nbytes) {
  if (slot < 0 || slot >= kPostSlots || !g_post[slot].host || nbytes > g_post[slot].bytes)
    return fail(PB_ERR_ARG, "pb_d2h_fetch: slot not posted or size too large");
  PB_CUDA(cudaEventSynchronize(g_post[slot].ev));
  std::memcpy(dst, g_post[slot].host, nbytes);
  return PB_OK;
}

int pb_d2d(uint64_t dst, uint64_t src, uint64_t nbytes) {
  if (nbytes == 0) return PB_OK;
  PB_CUDA(cudaMemcpyAsync((void*)(uintptr_t)dst, (const void*)(uintptr_t)src, nbytes, cudaMemcpyDeviceToDevice,
                          g_streams[0]));
  return PB_OK;
}

int pb_event_record(int from, int to) {
  cudaEvent_t ev;
  PB_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  PB_CUDA(cudaEventRecord(ev, g_streams[from]));
  PB_CUDA(cudaStreamWaitEvent(g_streams[to], ev, 0));
  PB_CUDA(cudaEventDestroy(ev));
  return PB_OK;
}

int pb_graph_begin(void) {
  PB_CUDA(cudaStreamBeginCapture(g_streams[0], cudaStreamCaptureModeRelaxed));
  return PB_OK;
}

int pb_graph_end(uint64_t* exec_out) {
  cudaGraph_t g;
  PB_CUDA(cudaStreamEndCapture(g_streams[0], &g));
  cudaGraphExec_t ex;
  PB_CUDA(cudaGraphInstantiate(&ex, g, 0));
  PB_CUDA(cudaGraphDestroy(g));
  *exec_out = (uint64_t)(uintptr_t)ex;
  return PB_OK;
}

int pb_graph_launch(uint64_t exec) {
  PB_CUDA(cudaGraphLaunch((cudaGraphExec_t)(uintptr_t)exec, g_streams[0]));
  return PB_OK;
}

int pb_graph_destroy(uint64_t exec) {
  PB_CUDA(cudaGraphExecDestroy((cudaGraphExec_t)(uintptr_t)exec));
  return PB_OK;
}

// op 0: create two events, record start; 1: record stop; 2: elapsed ms (syncs stop); 3: destroy
int pb_timer(int op, uint64_t* handle, float* ms) {
  cudaEvent_t* evs;
  if (op == 0) {
    evs = new cudaEvent_t[2];
    PB_CUDA(cudaEventCreate(&evs[0]));
    PB_CUDA(cudaEventCreate(&evs[1]));
    PB_CUDA(cudaEventRecord(evs[0], g_streams[0]));
    *handle = (uint64_t)(uintptr_t)evs;
    return PB_OK;
  }
  evs = (cudaEvent_t*)(uintptr_t)*handle;
  if (op == 1) {
    PB_CUDA(cudaEventRecord(evs[1], g_streams[0]));
  } else if (op == 2) {
    PB_CUDA(cudaEventSynchronize(evs[1]));
    PB_CUDA(cudaEventElapsedTime(ms, evs[0], evs[1]));
  } else {
    cudaEventDestroy(evs[0]);
    cudaEventDestroy(evs[1]);
    delete[] evs;
  }
  return PB_OK;
}

}  // extern "C"

// ---- NVTX ranges (named phases of a step on the timeline; no-ops without a tool attached) ----
extern "C" int pb_nvtx_push(const char* name) {
  nvtxRangePushA(name ? name : "");
  return PB_OK;
}
extern "C" int pb_nvtx_pop(void) {
  nvtxRangePop();
  return PB_OK;
}

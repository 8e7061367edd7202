// NCCL collectives on device buffers (replaces the thread-rank ring of
// minml/distributed.py:129-175).  Collectives run on the comm stream after an event fence
// on the compute stream; pb_nccl_wait makes the compute stream wait for them.
#include <nccl.h>
#include <chrono>
#include <cstring>
#include <thread>
#include "common.cuh"

using namespace pb;

static ncclDataType_t nccl_type(int dt) {
  switch (dt) {
    case PB_U8: case PB_BOOL: return ncclUint8;
    case PB_I32: return ncclInt32;
    case PB_I64: return ncclInt64;
    case PB_F32: return ncclFloat32;
    default: return ncclFloat64;
  }
}

#define PB_NCCL(call)                                                                  \
  do {                                                                                 \
    ncclResult_t r_ = (call);                                                          \
    if (r_ != ncclSuccess) return fail(PB_ERR_NCCL, std::string(#call) + ": " + ncclGetErrorString(r_)); \
  } while (0)

// two persistent fence events (created once; a wait binds to the record before it, so one
// event per direction can be re-recorded freely, also while a graph is being captured)
static cudaEvent_t g_to_comm = nullptr, g_to_compute = nullptr;

static int fence(cudaEvent_t* ev, cudaStream_t from, cudaStream_t to) {
  if (!*ev) PB_CUDA(cudaEventCreateWithFlags(ev, cudaEventDisableTiming));
  PB_CUDA(cudaEventRecord(*ev, from));
  PB_CUDA(cudaStreamWaitEvent(to, *ev, 0));
  return PB_OK;
}

static int fence_compute_to_comm() { return fence(&g_to_comm, compute_stream(), comm_stream()); }

// spins on the global nanosecond timer (pb_debug_stall_comm)
__global__ void stall_kernel(uint64_t ns) {
  uint64_t t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    __nanosleep(1000);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while (t - t0 < ns);
}

extern "C" {

int pb_nccl_unique_id(uint8_t out[128]) {
  ncclUniqueId id;
  PB_NCCL(ncclGetUniqueId(&id));
  std::memcpy(out, id.internal, 128);
  return PB_OK;
}

void* pb_nccl_init(int nranks, int rank, const uint8_t id_bytes[128]) {
  ncclUniqueId id;
  std::memcpy(id.internal, id_bytes, 128);
  ncclComm_t comm;
  ncclResult_t r = ncclCommInitRank(&comm, nranks, id, rank);
  if (r != ncclSuccess) {
    set_error(std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
    return nullptr;
  }
  return (void*)comm;
}

int pb_nccl_destroy(void* comm) {
  PB_NCCL(ncclCommDestroy((ncclComm_t)comm));
  return PB_OK;
}

int pb_nccl_allreduce(void* comm, uint64_t send, uint64_t recv, uint64_t count, int dtype, int op) {
  int rc = fence_compute_to_comm();
  if (rc) return rc;
  ncclRedOp_t o = op == 1 ? ncclMax : (op == 2 ? ncclAvg : ncclSum);
  PB_NCCL(ncclAllReduce((const void*)(uintptr_t)send, (void*)(uintptr_t)recv, count, nccl_type(dtype), o,
                        (ncclComm_t)comm, comm_stream()));
  return PB_OK;
}

int pb_nccl_broadcast(void* comm, uint64_t send, uint64_t recv, uint64_t count, int dtype, int root) {
  int rc = fence_compute_to_comm();
  if (rc) return rc;
  PB_NCCL(ncclBroadcast((const void*)(uintptr_t)send, (void*)(uintptr_t)recv, count, nccl_type(dtype), root,
                        (ncclComm_t)comm, comm_stream()));
  return PB_OK;
}

int pb_nccl_allgather(void* comm, uint64_t send, uint64_t recv, uint64_t count, int dtype) {
  int rc = fence_compute_to_comm();
  if (rc) return rc;
  PB_NCCL(ncclAllGather((const void*)(uintptr_t)send, (void*)(uintptr_t)recv, count, nccl_type(dtype),
                        (ncclComm_t)comm, comm_stream()));
  return PB_OK;
}

int pb_nccl_wait(void* comm) {
  (void)comm;
  return fence(&g_to_compute, comm_stream(), compute_stream());
}

int pb_nccl_sync(void* comm, int64_t timeout_ms) {
  static cudaEvent_t done = nullptr;
  if (!done) PB_CUDA(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
  PB_CUDA(cudaEventRecord(done, comm_stream()));
  const auto deadline = std::chrono::steady_clock::now() + std::chrono::milliseconds(timeout_ms);
  for (;;) {
    const cudaError_t q = cudaEventQuery(done);
    if (q == cudaSuccess) return PB_OK;
    if (q != cudaErrorNotReady) return cuda_fail(q, "pb_nccl_sync");
    if (comm) {
      ncclResult_t ar = ncclSuccess;
      ncclCommGetAsyncError((ncclComm_t)comm, &ar);
      if (ar != ncclSuccess && ar != ncclInProgress) {
        ncclCommAbort((ncclComm_t)comm);
        return fail(PB_ERR_NCCL, std::string("collective failed: ") + ncclGetErrorString(ar) +
                                     " (communicator aborted)");
      }
    }
    if (std::chrono::steady_clock::now() >= deadline) {
      if (comm) ncclCommAbort((ncclComm_t)comm);
      return fail(PB_ERR_TIMEOUT, "collective did not complete within " + std::to_string(timeout_ms) +
                                      " ms" + (comm ? " (communicator aborted)" : ""));
    }
    std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
}

int pb_debug_stall_comm(int64_t ms) {
  stall_kernel<<<1, 1, 0, comm_stream()>>>((uint64_t)ms * 1000000ull);
  PB_LAUNCHED();
  return PB_OK;
}

}  // extern "C"

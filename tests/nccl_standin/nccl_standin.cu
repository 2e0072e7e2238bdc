// TEST INFRASTRUCTURE ONLY: an in-process stand-in for libnccl.so.2 so the
// data-parallel path of the trainer (rank >= 1 shard offsets, ZeRO-1
// reduce-scatter / shard AdamW / all-gather, bucketed all-reduce) can execute
// on a machine with ONE GPU, where real NCCL refuses two ranks on one device.
//
// Ranks are host threads of one process (one DraftTrainer per thread, each
// with its own streams, all on the same device).  Every collective is matched
// by call order per communicator: the i-th call of every rank forms one
// operation.  Each caller records a "ready" event on its stream and waits on
// a host barrier; the last rank to arrive enqueues the operation on the
// group's own stream (wait on every ready event -> reduce / gather into a
// scratch buffer -> copy the result into every rank's output) and records a
// "done" event that every rank's stream then waits on.  Sums are computed in
// rank order (deterministic).  Only what specsim's trainer calls is provided
// (nccl_dyn.h): GetUniqueId, CommInitRank, AllReduce / ReduceScatter (sum of
// float, double, int64), AllGather (any type), CommDestroy, GetErrorString.
// Streams being captured into a CUDA graph are rejected (set
// SPECSIM_NO_GRAPH=1): the cross-stream wait on another rank's event cannot
// be captured.
//
// Loaded by the library through SPECSIM_NCCL_LIB (nccl_dyn.cpp).
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

namespace {

enum Kind { K_ALLREDUCE, K_REDUCESCATTER, K_ALLGATHER };

struct Call {
  Kind kind;
  const void* send;
  void* recv;
  size_t count;  // elements received by each rank (ReduceScatter / AllGather: per-rank chunk)
  ncclDataType_t type;
  cudaEvent_t ready;
};

struct Group {
  int nranks = 0, arrived_init = 0, device = 0;
  std::mutex mu;
  std::condition_variable cv;
  cudaStream_t stream = nullptr;
  void* scratch = nullptr;
  size_t scratch_bytes = 0;
  std::vector<int64_t> issued;            // per rank: calls issued
  std::map<int64_t, std::vector<Call>> pending;  // op index -> per-rank call
  std::map<int64_t, cudaEvent_t> done;           // op index -> completion event
  std::map<int64_t, int> consumed;               // op index -> ranks that waited on done
  int live = 0;
};

std::mutex g_mu;
std::map<std::string, std::shared_ptr<Group>> g_groups;
std::atomic<uint64_t> g_ids{1};

struct Comm {
  std::shared_ptr<Group> g;
  int rank;
};

size_t type_size(ncclDataType_t t) {
  switch (t) {
    case ncclInt8: case ncclUint8: return 1;
    case ncclFloat16: case ncclBfloat16: return 2;
    case ncclInt32: case ncclUint32: case ncclFloat32: return 4;
    case ncclInt64: case ncclUint64: case ncclFloat64: return 8;
    default: return 0;
  }
}

template <class T>
__global__ void sum_kernel(const T* const* ins, int n, T* out, size_t count) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    T s = ins[0][i];
    for (int k = 1; k < n; ++k) s += ins[k][i];  // rank order
    out[i] = s;
  }
}

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess) {                                                         \
      std::fprintf(stderr, "nccl_standin: %s: %s\n", #x, cudaGetErrorString(e_));    \
      return ncclUnhandledCudaError;                                                 \
    }                                                                                \
  } while (0)

// Runs one complete operation (all ranks' calls present) on the group stream.
ncclResult_t execute(Group& g, std::vector<Call>& calls, cudaEvent_t done) {
  const int n = g.nranks;
  const Call& c0 = calls[0];
  const size_t es = type_size(c0.type);
  for (const Call& c : calls)
    if (c.kind != c0.kind || c.count != c0.count || c.type != c0.type) return ncclInvalidUsage;
  const size_t chunk = c0.count * es;
  // scratch: n input-sized slots (inputs staged first, so in-place calls are safe)
  const size_t in_elems = c0.kind == K_ALLREDUCE ? c0.count : c0.kind == K_REDUCESCATTER
                                                                  ? c0.count * n
                                                                  : c0.count;
  const size_t need = in_elems * es * (n + 1) + 64 * sizeof(void*);
  if (need > g.scratch_bytes) {
    CK(cudaStreamSynchronize(g.stream));
    if (g.scratch) CK(cudaFree(g.scratch));
    CK(cudaMalloc(&g.scratch, need));
    g.scratch_bytes = need;
  }
  char* base = static_cast<char*>(g.scratch);
  for (const Call& c : calls) CK(cudaStreamWaitEvent(g.stream, c.ready, 0));
  for (int r = 0; r < n; ++r)
    CK(cudaMemcpyAsync(base + r * in_elems * es, calls[r].send, in_elems * es,
                       cudaMemcpyDeviceToDevice, g.stream));
  char* result = base + n * in_elems * es;
  if (c0.kind == K_ALLGATHER) {
    // result = concat of the staged inputs in rank order
    result = base;
  } else {
    const void** ptrs = reinterpret_cast<const void**>(result + in_elems * es);
    std::vector<const void*> h(n);
    for (int r = 0; r < n; ++r) h[r] = base + r * in_elems * es;
    CK(cudaMemcpyAsync(ptrs, h.data(), n * sizeof(void*), cudaMemcpyHostToDevice, g.stream));
    const unsigned blocks = static_cast<unsigned>(std::min<size_t>((in_elems + 255) / 256, 4096));
    switch (c0.type) {
      case ncclFloat32:
        sum_kernel<float><<<blocks, 256, 0, g.stream>>>(
            reinterpret_cast<const float* const*>(ptrs), n, reinterpret_cast<float*>(result), in_elems);
        break;
      case ncclFloat64:
        sum_kernel<double><<<blocks, 256, 0, g.stream>>>(
            reinterpret_cast<const double* const*>(ptrs), n, reinterpret_cast<double*>(result),
            in_elems);
        break;
      case ncclInt64:
        sum_kernel<long long><<<blocks, 256, 0, g.stream>>>(
            reinterpret_cast<const long long* const*>(ptrs), n,
            reinterpret_cast<long long*>(result), in_elems);
        break;
      default:
        return ncclInvalidArgument;
    }
    CK(cudaGetLastError());
    // the host vector h must outlive the async copy
    CK(cudaStreamSynchronize(g.stream));
  }
  for (int r = 0; r < n; ++r) {
    const char* src = c0.kind == K_REDUCESCATTER ? result + r * chunk : result;
    const size_t bytes = c0.kind == K_ALLGATHER ? chunk * n : chunk;
    CK(cudaMemcpyAsync(calls[r].recv, src, bytes, cudaMemcpyDeviceToDevice, g.stream));
  }
  CK(cudaEventRecord(done, g.stream));
  return ncclSuccess;
}

ncclResult_t collective(ncclComm_t comm_, Kind kind, const void* send, void* recv, size_t count,
                        ncclDataType_t type, ncclRedOp_t op, cudaStream_t stream) {
  Comm* comm = reinterpret_cast<Comm*>(comm_);
  if (!comm) return ncclInvalidArgument;
  if (kind != K_ALLGATHER && op != ncclSum) return ncclInvalidArgument;
  if (type_size(type) == 0) return ncclInvalidArgument;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  CK(cudaStreamIsCapturing(stream, &cap));
  if (cap != cudaStreamCaptureStatusNone) {
    std::fprintf(stderr, "nccl_standin: stream capture is not supported (SPECSIM_NO_GRAPH=1)\n");
    return ncclInvalidUsage;
  }
  Group& g = *comm->g;
  Call c{kind, send, recv, count, type, nullptr};
  CK(cudaEventCreateWithFlags(&c.ready, cudaEventDisableTiming));
  CK(cudaEventRecord(c.ready, stream));
  std::unique_lock<std::mutex> lk(g.mu);
  const int64_t idx = g.issued[comm->rank]++;
  auto& slot = g.pending[idx];
  if (slot.empty()) slot.resize(g.nranks, Call{kind, nullptr, nullptr, 0, type, nullptr});
  slot[comm->rank] = c;
  int present = 0;
  for (const Call& x : slot) present += x.ready != nullptr;
  ncclResult_t rc = ncclSuccess;
  if (present == g.nranks) {
    cudaEvent_t done;
    if (cudaEventCreateWithFlags(&done, cudaEventDisableTiming) != cudaSuccess)
      return ncclUnhandledCudaError;
    rc = execute(g, slot, done);
    for (Call& x : slot) cudaEventDestroy(x.ready);  // destroyed after the waits were enqueued
    g.pending.erase(idx);
    g.done[idx] = rc == ncclSuccess ? done : nullptr;
    g.cv.notify_all();
  } else {
    g.cv.wait(lk, [&] { return g.done.count(idx) != 0; });
  }
  cudaEvent_t done = g.done[idx];
  if (!done) return ncclInternalError;
  const cudaError_t e = cudaStreamWaitEvent(stream, done, 0);
  if (++g.consumed[idx] == g.nranks) {
    cudaEventDestroy(done);
    g.done.erase(idx);
    g.consumed.erase(idx);
  }
  if (e != cudaSuccess) return ncclUnhandledCudaError;
  return rc;
}

}  // namespace

extern "C" {

ncclResult_t ncclGetUniqueId(ncclUniqueId* id) {
  if (!id) return ncclInvalidArgument;
  std::memset(id, 0, sizeof(*id));
  std::snprintf(id->internal, sizeof(id->internal), "standin-%llu",
                static_cast<unsigned long long>(g_ids.fetch_add(1)));
  return ncclSuccess;
}

ncclResult_t ncclCommInitRank(ncclComm_t* out, int nranks, ncclUniqueId id, int rank) {
  if (!out || nranks < 1 || rank < 0 || rank >= nranks) return ncclInvalidArgument;
  std::shared_ptr<Group> g;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto& slot = g_groups[std::string(id.internal, strnlen(id.internal, sizeof(id.internal)))];
    if (!slot) {
      slot = std::make_shared<Group>();
      slot->nranks = nranks;
      slot->issued.assign(nranks, 0);
      if (cudaGetDevice(&slot->device) != cudaSuccess) return ncclUnhandledCudaError;
      if (cudaStreamCreateWithFlags(&slot->stream, cudaStreamNonBlocking) != cudaSuccess)
        return ncclUnhandledCudaError;
    }
    g = slot;
  }
  if (g->nranks != nranks) return ncclInvalidUsage;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev != g->device) return ncclInvalidUsage;
  {
    std::unique_lock<std::mutex> lk(g->mu);
    ++g->arrived_init;
    ++g->live;
    g->cv.notify_all();
    g->cv.wait(lk, [&] { return g->arrived_init >= g->nranks; });
  }
  *out = reinterpret_cast<ncclComm_t>(new Comm{g, rank});
  return ncclSuccess;
}

ncclResult_t ncclAllReduce(const void* send, void* recv, size_t count, ncclDataType_t type,
                           ncclRedOp_t op, ncclComm_t comm, cudaStream_t stream) {
  return collective(comm, K_ALLREDUCE, send, recv, count, type, op, stream);
}

ncclResult_t ncclReduceScatter(const void* send, void* recv, size_t recvcount,
                               ncclDataType_t type, ncclRedOp_t op, ncclComm_t comm,
                               cudaStream_t stream) {
  return collective(comm, K_REDUCESCATTER, send, recv, recvcount, type, op, stream);
}

ncclResult_t ncclAllGather(const void* send, void* recv, size_t sendcount, ncclDataType_t type,
                           ncclComm_t comm, cudaStream_t stream) {
  return collective(comm, K_ALLGATHER, send, recv, sendcount, type, ncclSum, stream);
}

ncclResult_t ncclCommDestroy(ncclComm_t comm_) {
  Comm* comm = reinterpret_cast<Comm*>(comm_);
  if (!comm) return ncclInvalidArgument;
  {
    std::lock_guard<std::mutex> lk(comm->g->mu);
    if (--comm->g->live == 0) {
      cudaStreamSynchronize(comm->g->stream);
      if (comm->g->scratch) cudaFree(comm->g->scratch);
      cudaStreamDestroy(comm->g->stream);
      comm->g->scratch = nullptr;
    }
  }
  delete comm;
  return ncclSuccess;
}

const char* ncclGetErrorString(ncclResult_t r) {
  switch (r) {
    case ncclSuccess: return "no error (stand-in)";
    case ncclUnhandledCudaError: return "unhandled cuda error (stand-in)";
    case ncclInvalidArgument: return "invalid argument (stand-in)";
    case ncclInvalidUsage: return "invalid usage (stand-in)";
    default: return "internal error (stand-in)";
  }
}

}  // extern "C"

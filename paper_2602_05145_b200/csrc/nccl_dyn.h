// NCCL resolved at run time (dlopen) instead of at link time, so loading this
// library never pins a libnccl.so.2 into the process before the host
// framework (e.g. torch, which ships a newer NCCL) loads its own.  Only the
// entry points the data-parallel exchange needs are bound.
#pragma once

#include <nccl.h>

namespace specsim {
namespace nccl {

struct Api {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t);
  ncclResult_t (*ReduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t,
                                ncclComm_t, cudaStream_t);
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  const char* (*GetErrorString)(ncclResult_t);
};

// Throws NcclError if no libnccl.so.2 can be found.  Prefers
// $SPECSIM_NCCL_LIB, then an already loaded copy, then the loader search path.
const Api& api();

}  // namespace nccl
}  // namespace specsim

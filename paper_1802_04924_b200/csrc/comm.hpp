// comm.hpp — NCCL, loaded at run time (dlopen) only when a context joins a
// multi-GPU communicator.  The library therefore has no link-time NCCL
// dependency and shares whichever libnccl.so.2 the process already loaded
// (e.g. PyTorch's).  Used for the row-sharded plan (plan.cu): all-gathers of
// derived tables at re-association points and of the argmin / final tables.
#pragma once

#include <nccl.h>

#include <cstddef>

namespace pp {

struct Nccl {
  ncclResult_t (*GetUniqueId)(ncclUniqueId *);
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*Broadcast)(const void *, void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  const char *(*GetErrorString)(ncclResult_t);
};

// Throws pp::Error(PP_ERR_CUDA) when libnccl.so.2 cannot be loaded.
const Nccl &nccl();

} // namespace pp

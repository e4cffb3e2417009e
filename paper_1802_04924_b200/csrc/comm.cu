// comm.cu — run-time NCCL binding and the communicator C ABI.
#include "comm.hpp"
#include "device.hpp"

#include <dlfcn.h>

#include <cstdlib>
#include <cstring>
#include <mutex>

namespace pp {

const Nccl &nccl() {
  static Nccl n{};
  static std::string err;
  static std::once_flag once;
  std::call_once(once, [] {
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD); // already loaded (e.g. by torch)
    if (!h && std::getenv("PARPLAN_NCCL")) h = dlopen(std::getenv("PARPLAN_NCCL"), RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      err = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
    auto sym = [&](const char *name) {
      void *p = dlsym(h, name);
      if (!p) err = std::string("libnccl.so.2 lacks ") + name;
      return p;
    };
    n.GetUniqueId = reinterpret_cast<decltype(n.GetUniqueId)>(sym("ncclGetUniqueId"));
    n.CommInitRank = reinterpret_cast<decltype(n.CommInitRank)>(sym("ncclCommInitRank"));
    n.CommDestroy = reinterpret_cast<decltype(n.CommDestroy)>(sym("ncclCommDestroy"));
    n.AllGather = reinterpret_cast<decltype(n.AllGather)>(sym("ncclAllGather"));
    n.Broadcast = reinterpret_cast<decltype(n.Broadcast)>(sym("ncclBroadcast"));
    n.AllReduce = reinterpret_cast<decltype(n.AllReduce)>(sym("ncclAllReduce"));
    n.GroupStart = reinterpret_cast<decltype(n.GroupStart)>(sym("ncclGroupStart"));
    n.GroupEnd = reinterpret_cast<decltype(n.GroupEnd)>(sym("ncclGroupEnd"));
    n.GetErrorString = reinterpret_cast<decltype(n.GetErrorString)>(sym("ncclGetErrorString"));
  });
  if (!err.empty()) fail(PP_ERR_CUDA, err);
  return n;
}

} // namespace pp

using pp::guard;

#define PP_NCCL(call)                                                                                                  \
  do {                                                                                                                 \
    ncclResult_t r_ = (call);                                                                                          \
    if (r_ != ncclSuccess) ::pp::fail(PP_ERR_CUDA, std::string(#call) + ": " + ::pp::nccl().GetErrorString(r_));       \
  } while (0)

extern "C" {

pp_status pp_comm_unique_id(void *id128) {
  return guard([&] {
    PP_REQUIRE(id128, "null argument");
    ncclUniqueId id;
    PP_NCCL(pp::nccl().GetUniqueId(&id));
    std::memcpy(id128, &id, sizeof id);
  });
}

pp_status pp_context_attach_comm(pp_context *ctx, int32_t nranks, int32_t rank, const void *id128) {
  return guard([&] {
    PP_REQUIRE(ctx && id128, "null argument");
    PP_REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks, "bad rank / world size");
    PP_REQUIRE(!ctx->comm, "context already has a communicator");
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof id);
    PP_CUDA(cudaSetDevice(ctx->device));
    ncclComm_t c = nullptr;
    PP_NCCL(pp::nccl().CommInitRank(&c, nranks, id, rank));
    ctx->comm = c;
    ctx->nranks = nranks;
    ctx->rank = rank;
  });
}

} // extern "C"

namespace pp {

void comm_destroy(pp_context *ctx) {
  if (ctx->comm) {
    nccl().CommDestroy(static_cast<ncclComm_t>(ctx->comm));
    ctx->comm = nullptr;
  }
}

void all_gather(pp_context *ctx, const void *send, void *recv, size_t bytes, cudaStream_t st) {
  PP_NCCL(nccl().AllGather(send, recv, bytes, ncclUint8, static_cast<ncclComm_t>(ctx->comm), st));
}

void broadcast(pp_context *ctx, void *buf, size_t bytes, int root, cudaStream_t st) {
  PP_NCCL(nccl().Broadcast(buf, buf, bytes, ncclUint8, root, static_cast<ncclComm_t>(ctx->comm), st));
}

void all_reduce_max(pp_context *ctx, int32_t *buf, size_t count, cudaStream_t st) {
  PP_NCCL(nccl().AllReduce(buf, buf, count, ncclInt32, ncclMax, static_cast<ncclComm_t>(ctx->comm), st));
}

void group_start() { PP_NCCL(nccl().GroupStart()); }
void group_end() { PP_NCCL(nccl().GroupEnd()); }

} // namespace pp

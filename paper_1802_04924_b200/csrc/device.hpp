// device.hpp — CUDA plumbing shared by the device translation units.
#pragma once

#include "internal.hpp"

#include <cuda_runtime.h>

#include <cstring>
#include <memory>
#include <string>
#include <vector>

#define PP_CUDA(call)                                                                                                  \
  do {                                                                                                                 \
    cudaError_t err_ = (call);                                                                                         \
    if (err_ != cudaSuccess)                                                                                           \
      ::pp::fail(PP_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(err_));                                   \
  } while (0)

namespace pp {

// Device allocation: owning (alloc/ensure) or a non-owning view into a pool.
template <class T> struct DBuf {
  T *p = nullptr;
  size_t n = 0;
  bool own = true;
  DBuf() = default;
  explicit DBuf(size_t count) { alloc(count); }
  DBuf(const DBuf &) = delete;
  DBuf &operator=(const DBuf &) = delete;
  DBuf(DBuf &&o) noexcept : p(o.p), n(o.n), own(o.own) { o.p = nullptr, o.n = 0; }
  DBuf &operator=(DBuf &&o) noexcept {
    if (this != &o) {
      release();
      p = o.p, n = o.n, own = o.own;
      o.p = nullptr, o.n = 0;
    }
    return *this;
  }
  ~DBuf() { release(); }
  void alloc(size_t count) {
    release();
    own = true;
    // whole 256-byte granules: 16-byte-rounded bulk copies of a table's byte
    // range (chain_item) stay inside the allocation
    if (count) PP_CUDA(cudaMalloc(reinterpret_cast<void **>(&p), (count * sizeof(T) + 255) / 256 * 256));
    n = count;
  }
  void ensure(size_t count) {
    if (count > n || !own) alloc(count);
  }
  void view(void *ptr, size_t count) {
    release();
    p = static_cast<T *>(ptr), n = count, own = false;
  }
  void release() {
    if (p && own) cudaFree(p);
    p = nullptr, n = 0, own = true;
  }
  size_t bytes() const { return n * sizeof(T); }
};

// Pinned host staging buffer (grown on demand).
struct PinnedBuf {
  void *p = nullptr;
  size_t cap = 0;
  PinnedBuf() = default;
  PinnedBuf(const PinnedBuf &) = delete;
  PinnedBuf &operator=(const PinnedBuf &) = delete;
  ~PinnedBuf() {
    if (p) cudaFreeHost(p);
  }
  void *ensure(size_t bytes) {
    if (bytes > cap) {
      if (p) cudaFreeHost(p);
      p = nullptr;
      PP_CUDA(cudaMallocHost(&p, bytes));
      cap = bytes;
    }
    return p;
  }
};

// Packs heterogeneous host arrays into one byte image (16-byte aligned
// sections) so a whole call's descriptors cross PCIe in one copy.
struct Packer {
  std::vector<unsigned char> bytes;
  template <class T> size_t put(const T *src, size_t count) {
    const size_t off = (bytes.size() + 15) & ~size_t(15);
    bytes.resize(off + count * sizeof(T));
    if (count) std::memcpy(bytes.data() + off, src, count * sizeof(T));
    return off;
  }
  template <class T> size_t put(const std::vector<T> &v) { return put(v.data(), v.size()); }
  size_t size() const { return bytes.size(); }
};

} // namespace pp

// One CUDA device + stream; all calls on a context are stream-ordered and
// synchronous at the API boundary.
struct pp_context {
  int device = 0;
  int sms = 0;
  cudaStream_t stream = nullptr;
  bool external_stream = false;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  int precision = PP_PRECISION_AUTO;
  bool no_minplus = false; // kernel policy bit 0: generic tiled fold only (parity tests)
  bool no_fused = false;   // kernel policy bit 1: one launch per wave instead of the fused kernel
  bool mp_conservative = false; // kernel policy bit 2: min-plus folds with proven operand caps only
  // multi-GPU (pp_context_attach_comm): plans are row-sharded across the ranks
  void *comm = nullptr; // ncclComm_t
  int nranks = 1, rank = 0;
  int64_t launches = 0;
  pp::DBuf<unsigned char> desc;  // device image of the current call's descriptors
  pp::PinnedBuf staging;         // pinned host side of desc + results
  pp::DBuf<unsigned char> scratch;
  // grow-only pools for one-shot plans (pp_plan / pp_plan_with_tables): no
  // cudaMalloc/cudaFree on the steady-state path
  pp::DBuf<unsigned char> plan_pool;
  pp::DBuf<unsigned char> plan_scratch; // device-only buffers of one-shot plans
  pp::PinnedBuf plan_pinned;
  size_t last_image_bytes = 0;          // reserve hint for the next descriptor image
  size_t last_pool_bytes = 0;           // largest one-shot plan pool so far (early table builds)
  pp::DBuf<unsigned int> gbar;          // fused kernel: grid-barrier word [0], build chunk counter [32..33] (zeroed once)
  // prepared plans of repeated one-shot pp_plan calls (plan.cu PlanCache)
  std::shared_ptr<void> plan_cache;

  void begin() const; // cudaSetDevice + record ev0
  double end_ms();    // record ev1, sync, elapsed
  // uploads a packed descriptor image; returns its device base pointer
  unsigned char *upload(const pp::Packer &pk);
};

namespace pp {
// comm.cu
void comm_destroy(pp_context *ctx);
void all_gather(pp_context *ctx, const void *send, void *recv, size_t bytes, cudaStream_t st);
void broadcast(pp_context *ctx, void *buf, size_t bytes, int root, cudaStream_t st); // in place
void all_reduce_max(pp_context *ctx, int32_t *buf, size_t count, cudaStream_t st);   // in place
void group_start();
void group_end();

inline void check_launch(pp_context *ctx, int n = 1) {
  PP_CUDA(cudaGetLastError());
  ctx->launches += n;
}
} // namespace pp

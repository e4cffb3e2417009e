// dp.cu — single-step DP execution (ReducedGraph step API), the standalone
// enumeration (ReducedGraph::enumerate_final, brute force) and table
// downloads.  The batched plan executor is in plan.cu; kernels in kernels.cuh.
#include "dp.hpp"
#include "kernels.cuh"

#include <algorithm>
#include <cstring>

namespace pp {

template <class T>
static void enumerate_impl(pp_context *ctx, const std::vector<EnumNode> &en, const std::vector<EnumEdge> &ee,
                           int shift, int32_t *digits, double *cost) {
  const int K = static_cast<int>(en.size());
  PP_REQUIRE(K <= kMaxEnumNodes, "too many nodes for the enumeration kernel");
  int64_t space = 1;
  for (const EnumNode &n : en) {
    PP_REQUIRE(space <= INT64_MAX / std::max(1, n.count), "enumeration space overflows");
    space *= n.count;
  }
  const int64_t lanes = int64_t(ctx->sms) * 8 * kEnumThreads;
  const int64_t per_thread = std::max<int64_t>(1, (space + lanes - 1) / lanes);
  const int64_t threads = (space + per_thread - 1) / per_thread;
  const int nblk = static_cast<int>((threads + kEnumThreads - 1) / kEnumThreads);
  using A = typename Acc<T>::type;
  Packer pk;
  const size_t oN = pk.put(en), oE = pk.put(ee), oBV = pk.put(std::vector<A>(static_cast<size_t>(nblk))),
               oBI = pk.put(std::vector<int64_t>(static_cast<size_t>(nblk)));
  const size_t oOut = pk.put(std::vector<unsigned char>(static_cast<size_t>(K) * 4 + 16));
  const size_t oFC = (oOut + static_cast<size_t>(K) * 4 + 7) & ~size_t(7);
  ctx->begin();
  unsigned char *b = ctx->upload(pk);
  enum_kernel<T><<<nblk, kEnumThreads, 0, ctx->stream>>>(reinterpret_cast<const EnumNode *>(b + oN), K,
                                                          reinterpret_cast<const EnumEdge *>(b + oE),
                                                          static_cast<int>(ee.size()), space, per_thread,
                                                          reinterpret_cast<A *>(b + oBV),
                                                          reinterpret_cast<int64_t *>(b + oBI));
  check_launch(ctx);
  FinishArgs fa{};
  fa.blk_val = b + oBV;
  fa.blk_idx = reinterpret_cast<const int64_t *>(b + oBI);
  fa.nblk = nblk;
  fa.nodes = reinterpret_cast<const EnumNode *>(b + oN);
  fa.k = K;
  fa.digits = reinterpret_cast<int32_t *>(b + oOut);
  fa.final_cost = reinterpret_cast<double *>(b + oFC);
  fa.shift = shift;
  fa.n_rec = -1;
  finish_kernel<T><<<1, kFinishThreads, 0, ctx->stream>>>(fa);
  check_launch(ctx);
  unsigned char *h = static_cast<unsigned char *>(ctx->staging.p);
  PP_CUDA(cudaMemcpyAsync(h + oOut, b + oOut, oFC + 8 - oOut, cudaMemcpyDeviceToHost, ctx->stream));
  ctx->end_ms();
  std::memcpy(digits, h + oOut, static_cast<size_t>(K) * 4);
  std::memcpy(cost, h + oFC, 8);
}

void run_enumerate(pp_context *ctx, int mode, int shift, const std::vector<const void *> &node_tabs,
                   const std::vector<int32_t> &counts, const std::vector<const void *> &edge_tabs,
                   const std::vector<int32_t> &eps, const std::vector<int32_t> &epd, const std::vector<int32_t> &ecols,
                   int32_t *digits, double *cost) {
  std::vector<EnumNode> en;
  for (size_t d = 0; d < node_tabs.size(); ++d) en.push_back(EnumNode{node_tabs[d], counts[d], 0});
  std::vector<EnumEdge> ee;
  for (size_t e = 0; e < edge_tabs.size(); ++e) ee.push_back(EnumEdge{edge_tabs[e], eps[e], epd[e], ecols[e], 0});
  if (mode == kFP64)
    enumerate_impl<double>(ctx, en, ee, 0, digits, cost);
  else
    enumerate_impl<int32_t>(ctx, en, ee, shift, digits, cost);
}

template <class T>
static void single_op(pp_context *ctx, const Op &op, const void *t1, const void *t2, const void *w, void *out,
                      uint16_t *am, int nu, int nw, int nv) {
  Packer pk;
  int64_t tiles = 0, blocks = 0;
  size_t off;
  if (!op.type) {
    FoldDesc<T> f{static_cast<const T *>(t1), static_cast<const T *>(t2), static_cast<const T *>(w),
                  static_cast<T *>(out), am, nu, nw, nv, (nv + kTile - 1) / kTile, 0};
    tiles = static_cast<int64_t>((nu + kTile - 1) / kTile) * f.tiles_k;
    off = pk.put(&f, 1);
  } else {
    MergeDesc<T> m{static_cast<const T *>(t1), static_cast<const T *>(t2), static_cast<T *>(out),
                   static_cast<int64_t>(nu) * nv, 0};
    blocks = (m.n + kMergePerBlock - 1) / kMergePerBlock;
    off = pk.put(&m, 1);
  }
  ctx->begin();
  unsigned char *b = ctx->upload(pk);
  const int64_t grid = tiles + blocks;
  if (grid) {
    wave_kernel<T><<<static_cast<unsigned>(grid), kFoldThreads, 0, ctx->stream>>>(
        reinterpret_cast<const FoldDesc<T> *>(b + off), op.type ? 0 : 1, tiles,
        reinterpret_cast<const MergeDesc<T> *>(b + off), op.type ? 1 : 0);
    check_launch(ctx);
  }
  ctx->end_ms();
}

void run_single_op(pp_context *ctx, int mode, const Op &op, const void *t1, const void *t2, const void *w, void *out,
                   uint16_t *am, int nu, int nw, int nv) {
  if (mode == kFP64)
    single_op<double>(ctx, op, t1, t2, w, out, am, nu, nw, nv);
  else
    single_op<int32_t>(ctx, op, t1, t2, w, out, am, nu, nw, nv);
}

void download_table(pp_context *ctx, int mode, int shift, const void *src, int64_t n, double *out) {
  if (!n) return;
  ctx->begin();
  if (mode == kFP64) {
    PP_CUDA(cudaMemcpyAsync(out, src, static_cast<size_t>(n) * 8, cudaMemcpyDeviceToHost, ctx->stream));
  } else {
    DBuf<double> tmp(static_cast<size_t>(n));
    to_double_kernel<int32_t><<<ctx->sms * 4, 256, 0, ctx->stream>>>(static_cast<const int32_t *>(src), tmp.p, n, shift);
    check_launch(ctx);
    PP_CUDA(cudaMemcpyAsync(out, tmp.p, static_cast<size_t>(n) * 8, cudaMemcpyDeviceToHost, ctx->stream));
    PP_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  ctx->end_ms();
}

void download_argmin(pp_context *ctx, const uint16_t *src, int64_t n, int32_t *out) {
  if (!n) return;
  ctx->begin();
  DBuf<int32_t> tmp(static_cast<size_t>(n));
  widen_u16_kernel<<<ctx->sms * 4, 256, 0, ctx->stream>>>(src, tmp.p, n);
  check_launch(ctx);
  PP_CUDA(cudaMemcpyAsync(out, tmp.p, static_cast<size_t>(n) * 4, cudaMemcpyDeviceToHost, ctx->stream));
  PP_CUDA(cudaStreamSynchronize(ctx->stream));
  ctx->end_ms();
}

} // namespace pp

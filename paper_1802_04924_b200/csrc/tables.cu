// tables.cu — contexts and the cost-table builders.
//
//   K2 node-cost fill   compute_cost + sync_cost (cost.hpp:60-94), one thread per (layer, config)
//   K1 xfer builder     transfer_profile (cost.hpp:103-131), one thread per (edge, c_src, c_dst) cell
//
// Both run in ONE launch (block ranges) over descriptors uploaded in one copy.
// K1 never enumerates partition pairs when the link bandwidth is uniform: the
// intersection volume factorises per dimension and the max over source
// partitions p != q is taken in O(1) per dimension (geometry.hpp:
// max_offdiag_volume); RN(4*maxvol/bw) equals the reference's max of
// per-pair RN(4*vol/bw) by monotonicity of correctly rounded division.  With a
// non-uniform bandwidth matrix K1 walks the pairs and divides per pair.
// Compiled with --fmad=false: every FP64 expression keeps the reference's
// operation order and rounding.
#include "tables.hpp"

#include <functional>

#include <type_traits>
#include "build.cuh"

#include "parplan/geometry.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>

using pp::DBuf;
using pp::guard;
namespace geo = parplan::geo;

// ---------------------------------------------------------------------------
// context
// ---------------------------------------------------------------------------

void pp_context::begin() const {
  PP_CUDA(cudaSetDevice(device));
  PP_CUDA(cudaEventRecord(ev0, stream));
}

double pp_context::end_ms() {
  PP_CUDA(cudaEventRecord(ev1, stream));
  PP_CUDA(cudaEventSynchronize(ev1));
  float ms = 0.f;
  PP_CUDA(cudaEventElapsedTime(&ms, ev0, ev1));
  return ms;
}

unsigned char *pp_context::upload(const pp::Packer &pk) {
  const size_t n = pk.size();
  desc.ensure(n + 16);
  void *h = staging.ensure(n + 16);
  std::memcpy(h, pk.bytes.data(), n);
  PP_CUDA(cudaMemcpyAsync(desc.p, h, n, cudaMemcpyHostToDevice, stream));
  return desc.p;
}

extern "C" {

pp_status pp_device_count(int32_t *count) {
  return guard([&] {
    PP_REQUIRE(count, "null argument");
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) n = 0;
    cudaGetLastError();
    int usable = 0;
    for (int d = 0; d < n; ++d) {
      cudaDeviceProp p;
      if (cudaGetDeviceProperties(&p, d) == cudaSuccess && p.major >= 10) ++usable;
    }
    *count = usable;
  });
}

pp_status pp_context_create(int32_t device, pp_context **out) {
  return guard([&] {
    PP_REQUIRE(out, "null argument");
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0)
      pp::fail(PP_ERR_CUDA, std::string("no CUDA device available (libparplan_cuda has no CPU fallback): ") +
                                cudaGetErrorString(e));
    PP_REQUIRE(device >= 0 && device < n, "device index out of range");
    cudaDeviceProp prop;
    PP_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10)
      pp::fail(PP_ERR_CUDA, "device " + std::to_string(device) + " is sm_" + std::to_string(prop.major) +
                                std::to_string(prop.minor) + "; this build targets sm_100a (B200)");
    auto ctx = std::make_unique<pp_context>();
    ctx->device = device;
    ctx->sms = prop.multiProcessorCount;
    PP_CUDA(cudaSetDevice(device));
    PP_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    PP_CUDA(cudaEventCreate(&ctx->ev0));
    PP_CUDA(cudaEventCreate(&ctx->ev1));
    *out = ctx.release();
  });
}

pp_status pp_context_create_on_stream(int32_t device, void *stream, pp_context **out) {
  pp_context *ctx = nullptr;
  pp_status st = pp_context_create(device, &ctx);
  if (st != PP_OK) return st;
  cudaStreamDestroy(ctx->stream);
  ctx->stream = static_cast<cudaStream_t>(stream);
  ctx->external_stream = true;
  *out = ctx;
  return PP_OK;
}

pp_status pp_context_stream(const pp_context *ctx, void **stream) {
  return guard([&] {
    PP_REQUIRE(ctx && stream, "null argument");
    *stream = ctx->stream;
  });
}

pp_status pp_context_release_pools(pp_context *ctx) {
  return guard([&] {
    PP_REQUIRE(ctx, "null context");
    PP_CUDA(cudaSetDevice(ctx->device));
    PP_CUDA(cudaStreamSynchronize(ctx->stream));
    ctx->plan_cache.reset();
    ctx->plan_pool.release();
    ctx->plan_scratch.release();
    ctx->scratch.release();
    ctx->last_pool_bytes = 0;
  });
}

pp_status pp_context_destroy(pp_context *ctx) {
  if (!ctx) return PP_OK;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  ctx->plan_cache.reset();
  ctx->desc.release();
  ctx->scratch.release();
  ctx->plan_pool.release();
  pp::comm_destroy(ctx);
  if (ctx->ev0) cudaEventDestroy(ctx->ev0);
  if (ctx->ev1) cudaEventDestroy(ctx->ev1);
  if (ctx->stream && !ctx->external_stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
  return PP_OK;
}

pp_status pp_context_set_precision(pp_context *ctx, int32_t policy) {
  return guard([&] {
    PP_REQUIRE(ctx, "null context");
    PP_REQUIRE(policy == PP_PRECISION_AUTO || policy == PP_PRECISION_FP64, "unknown precision policy");
    ctx->precision = policy;
  });
}

pp_status pp_context_set_kernel_policy(pp_context *ctx, int32_t policy) {
  return guard([&] {
    PP_REQUIRE(ctx, "null context");
    PP_REQUIRE(policy >= 0 && policy <= 7, "unknown kernel policy");
    ctx->no_minplus = (policy & 1) != 0;
    ctx->no_fused = (policy & 2) != 0;
    ctx->mp_conservative = (policy & 4) != 0;
  });
}

pp_status pp_context_launch_count(const pp_context *ctx, int64_t *n) {
  return guard([&] {
    PP_REQUIRE(ctx && n, "null argument");
    *n = ctx->launches;
  });
}

} // extern "C"

// ---------------------------------------------------------------------------
// K1 + K2
// ---------------------------------------------------------------------------

namespace pp {

__global__ void __launch_bounds__(kBuildThreads, 8) build_tables_kernel(BuildArgs a) {
  const int b = blockIdx.x;
  if (b < a.node_blocks) {
    const int64_t gi = static_cast<int64_t>(b) * kBuildThreads + threadIdx.x;
    if (gi < a.ncells) node_cost_cell(a, gi);
    return;
  }
  const int64_t eb = b - a.node_blocks + a.edge_block0;
  // edge of this block: binary search over the edges' first blocks, staged
  // in shared memory (independent loads instead of a chain of dependent ones)
  constexpr int kStaged = 2048;
  __shared__ int32_t first_blk[kStaged];
  const bool staged = a.ne <= kStaged;
  if (staged) {
    for (int e = threadIdx.x; e < a.ne; e += kBuildThreads) first_blk[e] = static_cast<int32_t>(a.edges[e].blk_begin);
    __syncthreads();
  }
  int lo = 0, hi = a.ne - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if ((staged ? first_blk[mid] : a.edges[mid].blk_begin) <= eb)
      lo = mid;
    else
      hi = mid - 1;
  }
  const EdgeDev &E = a.edges[lo];
  const int64_t cell = (eb - E.blk_begin) * kBuildThreads + threadIdx.x;
  xfer_cells_warp(a, cell < E.cells ? lo : -1, cell);
}

// Seeded synthetic tables (config-5 sweep at sizes the host generator cannot
// feed): value = (splitmix64(seed ^ stream) % 641) units of 1/64.
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}

// FP64 synthetic tables that the fixed-point certificate rejects: (k + u) / 64,
// k = splitmix % 641, u a 53-bit fraction (measured-cost-like values)
__global__ void synth64_kernel(double *out, int64_t n, uint64_t seed, uint64_t stream) {
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint64_t x = splitmix64(seed ^ stream ^ static_cast<uint64_t>(k) * 0x9E3779B97F4A7C15ULL);
    out[k] = (static_cast<double>(x % 641) + static_cast<double>(x >> 11) * 0x1p-53) / 64.0;
  }
}

__global__ void synth_kernel(int32_t *out, int64_t n, uint64_t seed, uint64_t stream) {
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[k] = static_cast<int32_t>(splitmix64(seed * 0x100000001B3ULL + stream + static_cast<uint64_t>(k)) % 641u);
}

__global__ void widen_kernel(const int32_t *in, double *out, int64_t n, int shift) {
  for (int64_t k = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[k] = ldexp(static_cast<double>(in[k]), -shift);
}

// evaluate_strategy by index (cost.hpp:235-246): one thread, pinned order.
template <class T>
__global__ void total_cost_kernel(const T *node, const T *xfer, const int64_t *cat_off, const int64_t *xoff,
                                  const int32_t *esrc, const int32_t *edst, const int32_t *counts,
                                  const int32_t *idx, int nl, int ne, int shift, double *out) {
  double t = 0.0;
  for (int l = 0; l < nl; ++l) t += ldexp(static_cast<double>(node[cat_off[l] + idx[l]]), -shift);
  for (int e = 0; e < ne; ++e)
    t += ldexp(static_cast<double>(xfer[xoff[e] + static_cast<int64_t>(idx[esrc[e]]) * counts[edst[e]] + idx[edst[e]]]),
               -shift);
  *out = t;
}

// Batched evaluation (evaluate_strategy / evaluate_components totals,
// cost.hpp:235-293) of n strategies given as config indices [n][nl]: one
// thread per strategy, each total summed from 0.0 in the reference's order
// (nodes by layer, then edges by id; node and transfer totals separately).
template <class T>
__global__ void evaluate_batch_kernel(const T *node, const T *xfer, const int64_t *cat_off, const int64_t *xoff,
                                      const int32_t *esrc, const int32_t *edst, const int32_t *counts,
                                      const int32_t *idx, int64_t n, int nl, int ne, int shift, double *cost,
                                      double *node_total, double *xfer_total) {
  for (int64_t s = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; s < n;
       s += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t *ix = idx + s * nl;
    double t = 0.0, tn = 0.0, tx = 0.0;
    for (int l = 0; l < nl; ++l) {
      const double v = ldexp(static_cast<double>(node[cat_off[l] + ix[l]]), -shift);
      t += v;
      tn += v;
    }
    for (int e = 0; e < ne; ++e) {
      const double v =
          ldexp(static_cast<double>(xfer[xoff[e] + static_cast<int64_t>(ix[esrc[e]]) * counts[edst[e]] + ix[edst[e]]]), -shift);
      t += v;
      tx += v;
    }
    cost[s] = t;
    if (node_total) node_total[s] = tn;
    if (xfer_total) xfer_total[s] = tx;
  }
}

// ---------------------------------------------------------------------------

static void init_layout(Tables &t, const Graph &g, const std::vector<int32_t> &counts) {
  t.nl = g.nl;
  t.ne = g.ne;
  t.esrc = g.esrc;
  t.edst = g.edst;
  t.counts = counts;
  t.cat_off.assign(static_cast<size_t>(g.nl) + 1, 0);
  for (int l = 0; l < g.nl; ++l) t.cat_off[static_cast<size_t>(l) + 1] = t.cat_off[static_cast<size_t>(l)] + counts[static_cast<size_t>(l)];
  t.ncells = t.cat_off.back();
  t.xoff.assign(static_cast<size_t>(g.ne) + 1, 0);
  for (int e = 0; e < g.ne; ++e)
    t.xoff[static_cast<size_t>(e) + 1] =
        t.xoff[static_cast<size_t>(e)] + static_cast<int64_t>(counts[static_cast<size_t>(g.esrc[static_cast<size_t>(e)])]) *
                                             counts[static_cast<size_t>(g.edst[static_cast<size_t>(e)])];
  t.xcells = t.xoff.back();
}

bool certify_fixed_point(const std::vector<double> &node, const std::vector<int64_t> &node_off,
                         const std::vector<double> &xfer, const std::vector<int64_t> &xoff,
                         const std::vector<int32_t> &counts, const std::vector<int> &esrc,
                         const std::vector<int> &edst, int *shift) {
  (void)counts, (void)esrc, (void)edst;
  // smallest s with every value an integer multiple of 2^-s
  int s = 0;
  auto need = [&](double v) -> bool {
    if (!std::isfinite(v)) return false;
    while (s <= 24) {
      const double u = std::ldexp(v, s);
      if (u == std::floor(u) && std::fabs(u) < 2147483647.0) return true;
      ++s;
    }
    return false;
  };
  for (double v : node)
    if (!need(v)) return false;
  for (double v : xfer)
    if (!need(v)) return false;
  // every DP value is a sum of at most one entry per original table
  double bound = 0.0;
  for (size_t l = 0; l + 1 < node_off.size(); ++l) {
    double m = 0.0;
    for (int64_t k = node_off[l]; k < node_off[l + 1]; ++k) m = std::max(m, std::fabs(node[static_cast<size_t>(k)]));
    bound += std::ldexp(m, s);
  }
  for (size_t e = 0; e + 1 < xoff.size(); ++e) {
    double m = 0.0;
    for (int64_t k = xoff[e]; k < xoff[e + 1]; ++k) m = std::max(m, std::fabs(xfer[static_cast<size_t>(k)]));
    bound += std::ldexp(m, s);
  }
  if (!(bound < 2147483647.0)) return false;
  *shift = s;
  return true;
}

void compute_spans_fixed(Tables &t, const std::vector<int32_t> &nu, const std::vector<int32_t> &xu) {
  t.node_span.assign(static_cast<size_t>(t.nl), 0);
  t.absmax_node.assign(static_cast<size_t>(t.nl), 0);
  for (int l = 0; l < t.nl; ++l) {
    int64_t lo = INT64_MAX, hi = INT64_MIN, am = 0;
    for (int64_t k = t.cat_off[static_cast<size_t>(l)]; k < t.cat_off[static_cast<size_t>(l) + 1]; ++k) {
      lo = std::min<int64_t>(lo, nu[static_cast<size_t>(k)]);
      hi = std::max<int64_t>(hi, nu[static_cast<size_t>(k)]);
      am = std::max<int64_t>(am, std::abs(static_cast<int64_t>(nu[static_cast<size_t>(k)])));
    }
    t.node_span[static_cast<size_t>(l)] = hi >= lo ? hi - lo : 0;
    t.absmax_node[static_cast<size_t>(l)] = am;
  }
  t.row_span.assign(static_cast<size_t>(t.ne), 0);
  t.col_span.assign(static_cast<size_t>(t.ne), 0);
  t.absmax_edge.assign(static_cast<size_t>(t.ne), 0);
  for (int e = 0; e < t.ne; ++e) {
    const int R = t.counts[static_cast<size_t>(t.esrc[static_cast<size_t>(e)])];
    const int Cc = t.counts[static_cast<size_t>(t.edst[static_cast<size_t>(e)])];
    const int32_t *m = xu.data() + t.xoff[static_cast<size_t>(e)];
    std::vector<int64_t> cmin(static_cast<size_t>(Cc), INT64_MAX), cmax(static_cast<size_t>(Cc), INT64_MIN);
    int64_t rs = 0, am = 0;
    for (int i = 0; i < R; ++i) {
      int64_t lo = INT64_MAX, hi = INT64_MIN;
      for (int j = 0; j < Cc; ++j) {
        const int64_t v = m[static_cast<int64_t>(i) * Cc + j];
        lo = std::min(lo, v), hi = std::max(hi, v);
        cmin[static_cast<size_t>(j)] = std::min(cmin[static_cast<size_t>(j)], v);
        cmax[static_cast<size_t>(j)] = std::max(cmax[static_cast<size_t>(j)], v);
        am = std::max(am, std::abs(v));
      }
      if (Cc) rs = std::max(rs, hi - lo);
    }
    int64_t cs = 0;
    if (R)
      for (int j = 0; j < Cc; ++j) cs = std::max(cs, cmax[static_cast<size_t>(j)] - cmin[static_cast<size_t>(j)]);
    t.row_span[static_cast<size_t>(e)] = rs;
    t.col_span[static_cast<size_t>(e)] = cs;
    t.absmax_edge[static_cast<size_t>(e)] = am;
  }
}

} // namespace pp

using namespace pp;

extern "C" {

pp_status pp_tables_build(pp_context *ctx, const pp_graph *gh, const pp_device_desc *dev, pp_tables **out) {
  return guard([&] {
    PP_REQUIRE(ctx && gh && dev && out, "pp_tables_build: null argument");
    auto tp = std::make_unique<pp_tables>();
    Tables &t = tp->impl;
    t.ctx = ctx;
    const BuildPlan bp = plan_build(t, gh->impl, dev);
    Packer pk;
    const size_t oL = pk.put(bp.L), oE = pk.put(bp.E), oC = pk.put(*bp.cfg32);
    const size_t oR = pk.put(dev->compute_rates, static_cast<size_t>(bp.D));
    const size_t oB = pk.put(dev->bandwidth, static_cast<size_t>(bp.D) * bp.D);
    t.node.alloc(static_cast<size_t>(t.ncells));
    t.compute.alloc(static_cast<size_t>(t.ncells));
    t.sync.alloc(static_cast<size_t>(t.ncells));
    t.xfer64.alloc(static_cast<size_t>(t.xcells));
    ctx->begin();
    unsigned char *base = ctx->upload(pk);
    BuildArgs a{};
    a.layers = reinterpret_cast<const LayerDev *>(base + oL);
    a.edges = reinterpret_cast<const EdgeDev *>(base + oE);
    a.cfg = reinterpret_cast<const int32_t *>(base + oC);
    a.rates = reinterpret_cast<const double *>(base + oR);
    a.bw = reinterpret_cast<const double *>(base + oB);
    a.node = t.node.p, a.compute = t.compute.p, a.sync = t.sync.p, a.xfer = t.xfer64.p;
    a.ncells = t.ncells;
    a.nl = t.nl, a.ne = t.ne, a.D = bp.D;
    a.node_blocks = static_cast<int32_t>(bp.node_blocks);
    a.bw_uniform = bp.bw_uniform;
    launch_build(ctx, ctx->stream, a, bp.grid);
    t.build_ms = ctx->end_ms();
    *out = tp.release();
  });
}

} // extern "C"

namespace pp {

void launch_build(pp_context *ctx, cudaStream_t st, const BuildArgs &a, int64_t grid) {
  if (grid <= 0) return;
  build_tables_kernel<<<static_cast<unsigned>(grid), kBuildThreads, 0, st>>>(a);
  check_launch(ctx);
}

BuildPlan plan_build(Tables &t, const Graph &g, const pp_device_desc *dev, bool host_configs) {
  const int D = dev->count;
  if (D < 1) throw parplan::InputError("device graph: need at least one device");
  // DeviceGraph validation (graph.hpp:193-214)
  const parplan::DeviceGraph dg(std::vector<double>(dev->compute_rates, dev->compute_rates + D),
                                std::vector<double>(dev->bandwidth, dev->bandwidth + static_cast<size_t>(D) * D));
  for (int l = 0; l < g.nl; ++l) { // K1 runs its region arithmetic on int32 coordinates
    const int64_t *s = &g.shape[static_cast<size_t>(l) * 4];
    // K1 divides coordinates by piece sizes with a float reciprocal + exact
    // correction, valid below 2^22 (build.cuh: div_fast)
    PP_REQUIRE(s[1] * s[2] * s[3] < (int64_t(1) << 22) && s[0] < (int64_t(1) << 22),
               "layer '" + g.g.layer(l).id + "': tensor extents exceed the 2^22 range of the table builder");
  }
  const Graph::Catalogs &cats = g.catalogs(D); // cached per (graph, D)
  const std::vector<int32_t> &counts = cats.counts;
  if (host_configs) t.configs = cats.configs; // kept for pp_tables_download only
  init_layout(t, g, counts);
  t.mode = kFP64;
  t.analytic = true;
  BuildPlan bp;
  bp.D = D;
  bp.cfg32 = &cats.configs32;

  double bw_uniform = dev->bandwidth[D > 1 ? 1 : 0];
    for (int p = 0; p < D; ++p)
      for (int q = 0; q < D; ++q)
        if (p != q && dev->bandwidth[static_cast<size_t>(p) * D + q] != bw_uniform) bw_uniform = -1.0;
    if (D == 1) bw_uniform = 1.0; // no off-diagonal pairs: every table is zero

    std::vector<LayerDev> L(static_cast<size_t>(g.nl));
    for (int l = 0; l < g.nl; ++l) {
      LayerDev &x = L[static_cast<size_t>(l)];
      std::memcpy(x.shape, &g.shape[static_cast<size_t>(l) * 4], sizeof x.shape);
      const auto &ins = g.g.in_edges(l);
      const int src = ins.empty() ? l : g.esrc[static_cast<size_t>(ins.front())]; // Input: in = out (cost.hpp:181-182)
      std::memcpy(x.in_shape, &g.shape[static_cast<size_t>(src) * 4], sizeof x.in_shape);
      std::memcpy(x.params, &g.params[static_cast<size_t>(l) * 7], sizeof x.params);
      x.cat_off = t.cat_off[static_cast<size_t>(l)];
      x.kind = g.kind[static_cast<size_t>(l)];
      x.count = counts[static_cast<size_t>(l)];
    }
    std::vector<EdgeDev> E(static_cast<size_t>(g.ne));
    int64_t blocks = 0;
    for (int e = 0; e < g.ne; ++e) {
      EdgeDev &x = E[static_cast<size_t>(e)];
      const int s = g.esrc[static_cast<size_t>(e)], d = g.edst[static_cast<size_t>(e)];
      std::memcpy(x.sshape, &g.shape[static_cast<size_t>(s) * 4], sizeof x.sshape);
      std::memcpy(x.dshape, &g.shape[static_cast<size_t>(d) * 4], sizeof x.dshape);
      std::memcpy(x.params, &g.params[static_cast<size_t>(d) * 7], sizeof x.params);
      x.band = g.band_offset[static_cast<size_t>(e)];
      x.kind = g.kind[static_cast<size_t>(d)];
      x.nu = counts[static_cast<size_t>(s)];
      x.nv = counts[static_cast<size_t>(d)];
      x.cat_u = t.cat_off[static_cast<size_t>(s)];
      x.cat_v = t.cat_off[static_cast<size_t>(d)];
      x.out_off = t.xoff[static_cast<size_t>(e)];
      x.cells = static_cast<int64_t>(x.nu) * x.nv;
      x.blk_begin = blocks;
      blocks += (x.cells + kBuildThreads - 1) / kBuildThreads;
    }
    const int64_t node_blocks = (t.ncells + kBuildThreads - 1) / kBuildThreads;
    PP_REQUIRE(node_blocks + blocks < (int64_t(1) << 31), "cost tables too large for one launch");
    bp.L = std::move(L);
    bp.E = std::move(E);
    bp.node_blocks = node_blocks;
    bp.grid = node_blocks + blocks;
    bp.bw_uniform = bw_uniform;
    return bp;
}

} // namespace pp

extern "C" {

pp_status pp_tables_upload(pp_context *ctx, const pp_graph *gh, const int32_t *counts, const int64_t *configs,
                           const double *node, const double *xfer, pp_tables **out) {
  return guard([&] {
    PP_REQUIRE(ctx && gh && counts && node && out, "pp_tables_upload: null argument");
    const Graph &g = gh->impl;
    auto tp = std::make_unique<pp_tables>();
    Tables &t = tp->impl;
    t.ctx = ctx;
    std::vector<int32_t> cnt(counts, counts + g.nl);
    for (int32_t c : cnt) PP_REQUIRE(c >= 1 && c <= 65535, "every layer needs 1..65535 configs");
    init_layout(t, g, cnt);
    PP_REQUIRE(t.xcells == 0 || xfer, "pp_tables_upload: null xfer");
    if (configs)
      t.configs.assign(configs, configs + 4 * t.ncells);
    else
      t.configs.assign(static_cast<size_t>(4 * t.ncells), 1);
    std::vector<double> nd(node, node + t.ncells), xf(xfer, xfer + t.xcells);
    int shift = 0;
    const bool fixed = ctx->precision == PP_PRECISION_AUTO &&
                       certify_fixed_point(nd, t.cat_off, xf, t.xoff, cnt, t.esrc, t.edst, &shift);
    ctx->begin();
    if (fixed) {
      t.mode = kFixed;
      t.shift = shift;
      std::vector<int32_t> nu(nd.size()), xu(xf.size());
      for (size_t k = 0; k < nd.size(); ++k) nu[k] = static_cast<int32_t>(std::ldexp(nd[k], shift));
      for (size_t k = 0; k < xf.size(); ++k) xu[k] = static_cast<int32_t>(std::ldexp(xf[k], shift));
      compute_spans_fixed(t, nu, xu);
      t.node32.alloc(nu.size());
      t.xfer32.alloc(xu.size());
      PP_CUDA(cudaMemcpyAsync(t.node32.p, nu.data(), nu.size() * 4, cudaMemcpyHostToDevice, ctx->stream));
      if (!xu.empty())
        PP_CUDA(cudaMemcpyAsync(t.xfer32.p, xu.data(), xu.size() * 4, cudaMemcpyHostToDevice, ctx->stream));
    } else {
      t.mode = kFP64;
      t.node.alloc(nd.size());
      t.xfer64.alloc(xf.size());
      PP_CUDA(cudaMemcpyAsync(t.node.p, nd.data(), nd.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
      if (!xf.empty())
        PP_CUDA(cudaMemcpyAsync(t.xfer64.p, xf.data(), xf.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
    }
    ctx->end_ms();
    *out = tp.release();
  });
}

} // extern "C"

namespace pp {
// Fixed-point tables of C configs per layer whose values (in units of 2^-shift,
// within [0, vmax]) come from a host generator in fill order (node cells by
// layer, then xfer cells by edge id, row-major), streamed to the device
// through a pinned buffer: no host copy of the whole table set.
pp_tables *tables_fixed_streamed(pp_context *ctx, const Graph &g, int32_t C, int shift, int64_t vmax,
                                 const std::function<void(int32_t *, size_t)> &gen) {
  PP_REQUIRE(C >= 1 && C <= 65535, "configs must be in 1..65535");
  auto tp = std::make_unique<pp_tables>();
  Tables &t = tp->impl;
  t.ctx = ctx;
  init_layout(t, g, std::vector<int32_t>(static_cast<size_t>(g.nl), C));
  t.configs.resize(static_cast<size_t>(4 * t.ncells));
  for (int64_t k = 0; k < t.ncells; ++k) {
    t.configs[static_cast<size_t>(4 * k)] = 1, t.configs[static_cast<size_t>(4 * k + 1)] = 1;
    t.configs[static_cast<size_t>(4 * k + 2)] = 1, t.configs[static_cast<size_t>(4 * k + 3)] = k % C + 1;
  }
  t.mode = kFixed;
  t.shift = shift;
  t.node_span.assign(static_cast<size_t>(g.nl), vmax);
  t.absmax_node.assign(static_cast<size_t>(g.nl), vmax);
  t.row_span.assign(static_cast<size_t>(g.ne), vmax);
  t.col_span.assign(static_cast<size_t>(g.ne), vmax);
  t.absmax_edge.assign(static_cast<size_t>(g.ne), vmax);
  PP_REQUIRE(static_cast<double>(vmax) * (g.nl + g.ne) < 2147483647.0, "tables too large for exact fixed point");
  t.node32.alloc(static_cast<size_t>(t.ncells));
  t.xfer32.alloc(static_cast<size_t>(t.xcells));
  constexpr size_t kChunk = size_t(16) << 20; // cells per staging half
  PinnedBuf stage;
  int32_t *h = static_cast<int32_t *>(stage.ensure(2 * kChunk * 4));
  cudaEvent_t done[2];
  PP_CUDA(cudaEventCreateWithFlags(&done[0], cudaEventDisableTiming));
  PP_CUDA(cudaEventCreateWithFlags(&done[1], cudaEventDisableTiming));
  ctx->begin();
  int half = 0;
  auto stream_into = [&](int32_t *dst, int64_t n) {
    for (int64_t o = 0; o < n; o += static_cast<int64_t>(kChunk)) {
      const size_t m = static_cast<size_t>(std::min<int64_t>(static_cast<int64_t>(kChunk), n - o));
      int32_t *hb = h + half * kChunk;
      PP_CUDA(cudaEventSynchronize(done[half])); // the copy that last used this half is done
      gen(hb, m);
      PP_CUDA(cudaMemcpyAsync(dst + o, hb, m * 4, cudaMemcpyHostToDevice, ctx->stream));
      PP_CUDA(cudaEventRecord(done[half], ctx->stream));
      half ^= 1;
    }
  };
  PP_CUDA(cudaEventRecord(done[0], ctx->stream));
  PP_CUDA(cudaEventRecord(done[1], ctx->stream));
  stream_into(t.node32.p, t.ncells);
  stream_into(t.xfer32.p, t.xcells);
  t.build_ms = ctx->end_ms();
  cudaEventDestroy(done[0]);
  cudaEventDestroy(done[1]);
  return tp.release();
}
} // namespace pp

extern "C" {

pp_status pp_tables_synthetic(pp_context *ctx, const pp_graph *gh, int32_t C, uint64_t seed, pp_tables **out) {
  return guard([&] {
    PP_REQUIRE(ctx && gh && out, "pp_tables_synthetic: null argument");
    PP_REQUIRE(C >= 1 && C <= 65535, "configs must be in 1..65535");
    const Graph &g = gh->impl;
    auto tp = std::make_unique<pp_tables>();
    Tables &t = tp->impl;
    t.ctx = ctx;
    init_layout(t, g, std::vector<int32_t>(static_cast<size_t>(g.nl), C));
    t.configs.resize(static_cast<size_t>(4 * t.ncells));
    for (int64_t k = 0; k < t.ncells; ++k) {
      t.configs[static_cast<size_t>(4 * k)] = 1, t.configs[static_cast<size_t>(4 * k + 1)] = 1;
      t.configs[static_cast<size_t>(4 * k + 2)] = 1, t.configs[static_cast<size_t>(4 * k + 3)] = k % C + 1;
    }
    t.mode = kFixed;
    t.shift = 6;
    // values are k/64 with k in [0, 640]: spans and magnitudes are known a priori
    t.node_span.assign(static_cast<size_t>(g.nl), 640);
    t.absmax_node.assign(static_cast<size_t>(g.nl), 640);
    t.row_span.assign(static_cast<size_t>(g.ne), 640);
    t.col_span.assign(static_cast<size_t>(g.ne), 640);
    t.absmax_edge.assign(static_cast<size_t>(g.ne), 640);
    PP_REQUIRE(640.0 * (g.nl + g.ne) < 2147483647.0, "synthetic graph too large for exact fixed point");
    t.node32.alloc(static_cast<size_t>(t.ncells));
    t.xfer32.alloc(static_cast<size_t>(t.xcells));
    ctx->begin();
    const int grid = ctx->sms * 8;
    synth_kernel<<<grid, 256, 0, ctx->stream>>>(t.node32.p, t.ncells, seed, 0x4e4f4445ULL << 32);
    check_launch(ctx);
    if (t.xcells) {
      synth_kernel<<<grid, 256, 0, ctx->stream>>>(t.xfer32.p, t.xcells, seed, 0x58464552ULL << 32);
      check_launch(ctx);
    }
    t.build_ms = ctx->end_ms();
    *out = tp.release();
  });
}

pp_status pp_tables_synthetic64(pp_context *ctx, const pp_graph *gh, int32_t C, uint64_t seed, pp_tables **out) {
  return guard([&] {
    PP_REQUIRE(ctx && gh && out, "pp_tables_synthetic64: null argument");
    PP_REQUIRE(C >= 1 && C <= 65535, "configs must be in 1..65535");
    const Graph &g = gh->impl;
    auto tp = std::make_unique<pp_tables>();
    Tables &t = tp->impl;
    t.ctx = ctx;
    init_layout(t, g, std::vector<int32_t>(static_cast<size_t>(g.nl), C));
    t.configs.resize(static_cast<size_t>(4 * t.ncells));
    for (int64_t k = 0; k < t.ncells; ++k) {
      t.configs[static_cast<size_t>(4 * k)] = 1, t.configs[static_cast<size_t>(4 * k + 1)] = 1;
      t.configs[static_cast<size_t>(4 * k + 2)] = 1, t.configs[static_cast<size_t>(4 * k + 3)] = k % C + 1;
    }
    t.mode = kFP64;
    t.node.alloc(static_cast<size_t>(t.ncells));
    t.xfer64.alloc(static_cast<size_t>(t.xcells));
    ctx->begin();
    const int grid = ctx->sms * 8;
    synth64_kernel<<<grid, 256, 0, ctx->stream>>>(t.node.p, t.ncells, seed, 0x4e4f4445ULL << 32);
    check_launch(ctx);
    if (t.xcells) {
      synth64_kernel<<<grid, 256, 0, ctx->stream>>>(t.xfer64.p, t.xcells, seed, 0x58464552ULL << 32);
      check_launch(ctx);
    }
    t.build_ms = ctx->end_ms();
    *out = tp.release();
  });
}

pp_status pp_tables_destroy(pp_tables *t) {
  if (t && t->impl.ctx) cudaSetDevice(t->impl.ctx->device);
  delete t;
  return PP_OK;
}

pp_status pp_tables_counts(const pp_tables *tp, int32_t *counts, int64_t *xcells) {
  return guard([&] {
    PP_REQUIRE(tp, "null tables");
    if (counts) std::memcpy(counts, tp->impl.counts.data(), tp->impl.counts.size() * sizeof(int32_t));
    if (xcells) *xcells = tp->impl.xcells;
  });
}

pp_status pp_tables_build_ms(const pp_tables *tp, double *ms) {
  return guard([&] {
    PP_REQUIRE(tp && ms, "null argument");
    *ms = tp->impl.build_ms;
  });
}

pp_status pp_tables_download(pp_tables *tp, int64_t *configs, double *node, double *compute, double *sync,
                             double *xfer) {
  return guard([&] {
    PP_REQUIRE(tp, "null tables");
    Tables &t = tp->impl;
    pp_context *ctx = t.ctx;
    ctx->begin();
    if (configs) std::memcpy(configs, t.configs.data(), t.configs.size() * sizeof(int64_t));
    auto widen = [&](const int32_t *src, int64_t n, double *dst) {
      if (!n) return;
      DBuf<double> tmp(static_cast<size_t>(n));
      widen_kernel<<<ctx->sms * 4, 256, 0, ctx->stream>>>(src, tmp.p, n, t.shift);
      check_launch(ctx);
      PP_CUDA(cudaMemcpyAsync(dst, tmp.p, static_cast<size_t>(n) * 8, cudaMemcpyDeviceToHost, ctx->stream));
      PP_CUDA(cudaStreamSynchronize(ctx->stream));
    };
    if (t.mode == kFP64) {
      if (node) PP_CUDA(cudaMemcpyAsync(node, t.node.p, static_cast<size_t>(t.ncells) * 8, cudaMemcpyDeviceToHost, ctx->stream));
      if (xfer && t.xcells)
        PP_CUDA(cudaMemcpyAsync(xfer, t.xfer64.p, static_cast<size_t>(t.xcells) * 8, cudaMemcpyDeviceToHost, ctx->stream));
    } else {
      if (node) widen(t.node32.p, t.ncells, node);
      if (xfer) widen(t.xfer32.p, t.xcells, xfer);
    }
    if (compute) {
      if (t.analytic)
        PP_CUDA(cudaMemcpyAsync(compute, t.compute.p, static_cast<size_t>(t.ncells) * 8, cudaMemcpyDeviceToHost, ctx->stream));
      else
        std::memset(compute, 0, static_cast<size_t>(t.ncells) * 8);
    }
    if (sync) {
      if (t.analytic)
        PP_CUDA(cudaMemcpyAsync(sync, t.sync.p, static_cast<size_t>(t.ncells) * 8, cudaMemcpyDeviceToHost, ctx->stream));
      else
        std::memset(sync, 0, static_cast<size_t>(t.ncells) * 8);
    }
    ctx->end_ms();
  });
}

pp_status pp_tables_total_cost(pp_tables *tp, const int32_t *indices, double *cost) {
  return guard([&] {
    PP_REQUIRE(tp && indices && cost, "null argument");
    Tables &t = tp->impl;
    pp_context *ctx = t.ctx;
    for (int l = 0; l < t.nl; ++l)
      PP_REQUIRE(indices[l] >= 0 && indices[l] < t.counts[static_cast<size_t>(l)], "config index out of range");
    Packer pk;
    std::vector<int32_t> es(t.esrc.begin(), t.esrc.end()), ed(t.edst.begin(), t.edst.end());
    const size_t oc = pk.put(t.cat_off), ox = pk.put(t.xoff), os = pk.put(es), od = pk.put(ed), on = pk.put(t.counts),
                 oi = pk.put(indices, static_cast<size_t>(t.nl)), oo = pk.put(std::vector<double>(1));
    ctx->begin();
    unsigned char *b = ctx->upload(pk);
    auto P = [&](size_t o) { return b + o; };
    if (t.mode == kFP64)
      total_cost_kernel<double><<<1, 1, 0, ctx->stream>>>(
          t.node.p, t.xfer64.p, reinterpret_cast<int64_t *>(P(oc)), reinterpret_cast<int64_t *>(P(ox)),
          reinterpret_cast<int32_t *>(P(os)), reinterpret_cast<int32_t *>(P(od)), reinterpret_cast<int32_t *>(P(on)),
          reinterpret_cast<int32_t *>(P(oi)), t.nl, t.ne, 0, reinterpret_cast<double *>(P(oo)));
    else
      total_cost_kernel<int32_t><<<1, 1, 0, ctx->stream>>>(
          t.node32.p, t.xfer32.p, reinterpret_cast<int64_t *>(P(oc)), reinterpret_cast<int64_t *>(P(ox)),
          reinterpret_cast<int32_t *>(P(os)), reinterpret_cast<int32_t *>(P(od)), reinterpret_cast<int32_t *>(P(on)),
          reinterpret_cast<int32_t *>(P(oi)), t.nl, t.ne, t.shift, reinterpret_cast<double *>(P(oo)));
    check_launch(ctx);
    PP_CUDA(cudaMemcpyAsync(cost, P(oo), 8, cudaMemcpyDeviceToHost, ctx->stream));
    ctx->end_ms();
  });
}

pp_status pp_tables_evaluate_batch(pp_tables *tp, int64_t n, const int32_t *indices, double *cost, double *node_total,
                                   double *xfer_total) {
  return guard([&] {
    PP_REQUIRE(tp && (n == 0 || (indices && cost)) && n >= 0, "pp_tables_evaluate_batch: bad argument");
    Tables &t = tp->impl;
    pp_context *ctx = t.ctx;
    for (int64_t s = 0; s < n; ++s)
      for (int l = 0; l < t.nl; ++l) {
        const int32_t x = indices[s * t.nl + l];
        PP_REQUIRE(x >= 0 && x < t.counts[static_cast<size_t>(l)], "config index out of range");
      }
    if (n == 0) return;
    Packer pk;
    std::vector<int32_t> es(t.esrc.begin(), t.esrc.end()), ed(t.edst.begin(), t.edst.end());
    const size_t oc = pk.put(t.cat_off), ox = pk.put(t.xoff), os = pk.put(es), od = pk.put(ed), on = pk.put(t.counts),
                 oi = pk.put(indices, static_cast<size_t>(n) * static_cast<size_t>(t.nl));
    DBuf<double> out(static_cast<size_t>(n) * 3);
    ctx->begin();
    unsigned char *b = ctx->upload(pk);
    auto P = [&](size_t o) { return b + o; };
    const int grid = static_cast<int>(std::min<int64_t>((n + 255) / 256, int64_t(ctx->sms) * 8));
    double *o0 = out.p, *o1 = node_total ? out.p + n : nullptr, *o2 = xfer_total ? out.p + 2 * n : nullptr;
    auto run = [&](auto *node, auto *xf, int shift) {
      using T = std::remove_const_t<std::remove_pointer_t<decltype(node)>>;
      evaluate_batch_kernel<T><<<grid, 256, 0, ctx->stream>>>(
          node, xf, reinterpret_cast<int64_t *>(P(oc)), reinterpret_cast<int64_t *>(P(ox)),
          reinterpret_cast<int32_t *>(P(os)), reinterpret_cast<int32_t *>(P(od)), reinterpret_cast<int32_t *>(P(on)),
          reinterpret_cast<int32_t *>(P(oi)), n, t.nl, t.ne, shift, o0, o1, o2);
    };
    if (t.mode == kFP64)
      run(static_cast<const double *>(t.node.p), static_cast<const double *>(t.xfer64.p), 0);
    else
      run(static_cast<const int32_t *>(t.node32.p), static_cast<const int32_t *>(t.xfer32.p), t.shift);
    check_launch(ctx);
    PP_CUDA(cudaMemcpyAsync(cost, o0, static_cast<size_t>(n) * 8, cudaMemcpyDeviceToHost, ctx->stream));
    if (node_total) PP_CUDA(cudaMemcpyAsync(node_total, o1, static_cast<size_t>(n) * 8, cudaMemcpyDeviceToHost, ctx->stream));
    if (xfer_total) PP_CUDA(cudaMemcpyAsync(xfer_total, o2, static_cast<size_t>(n) * 8, cudaMemcpyDeviceToHost, ctx->stream));
    ctx->end_ms();
  });
}

} // extern "C"

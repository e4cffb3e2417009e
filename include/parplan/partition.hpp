/* parplan/partition.hpp — configs, regions, config enumeration, placement.
 *
 * Drop-in for /root/reference/proj/include/parplan/partition.hpp:
 *   Config + lexicographic order (:31-69), Strategy (:78), Region (:85-120),
 *   parallelizable_dims (:140-156), enumerate_configs (:174-204),
 *   owned_region (:213-232), required_input_region (:283-350), place (:356-369).
 * The region arithmetic itself lives in geometry.hpp so that the xfer-table
 * kernel evaluates exactly the same formulas.
 */
#pragma once

#include "parplan/geometry.hpp"
#include "parplan/graph.hpp"

#include <array>
#include <tuple>
#include <vector>

namespace parplan {

/// Partition degree per tensor dimension.
struct Config {
  i64 sample = 1;
  i64 channel = 1;
  i64 height = 1;
  i64 width = 1;

  constexpr i64 degree(Dim d) const {
    return d == Dim::Sample ? sample : d == Dim::Channel ? channel : d == Dim::Height ? height : width;
  }
  constexpr i64 &degree(Dim d) {
    return d == Dim::Sample ? sample : d == Dim::Channel ? channel : d == Dim::Height ? height : width;
  }
  constexpr i64 total() const { return sample * channel * height * width; }

  friend constexpr bool operator==(const Config &, const Config &) = default;
  friend constexpr bool operator<(const Config &a, const Config &b) {
    return std::tie(a.sample, a.channel, a.height, a.width) < std::tie(b.sample, b.channel, b.height, b.width);
  }
};

inline std::string to_string(const Config &c) {
  return "{n=" + std::to_string(c.sample) + ", c=" + std::to_string(c.channel) + ", h=" + std::to_string(c.height) +
         ", w=" + std::to_string(c.width) + "}";
}

using Strategy = std::vector<Config>;

/// Half-open box [lo, hi) over (sample, channel, height, width).
struct Region {
  std::array<i64, kDimCount> lo{{0, 0, 0, 0}};
  std::array<i64, kDimCount> hi{{0, 0, 0, 0}};

  i64 length(Dim d) const {
    const auto i = static_cast<size_t>(d);
    return hi[i] > lo[i] ? hi[i] - lo[i] : 0;
  }
  i64 volume() const { return geo::box_volume(lo.data(), hi.data()); }
  bool empty() const { return volume() == 0; }
  friend bool operator==(const Region &, const Region &) = default;
};

inline Region full_region(const TensorShape &s) {
  Region r;
  for (Dim d : kAllDims) r.hi[static_cast<size_t>(d)] = s.extent(d);
  return r;
}

inline Region intersect(const Region &a, const Region &b) {
  Region r;
  for (size_t i = 0; i < kDimCount; ++i) {
    r.lo[i] = std::max(a.lo[i], b.lo[i]);
    r.hi[i] = std::max(r.lo[i], std::min(a.hi[i], b.hi[i]));
  }
  return r;
}

inline std::string to_string(const Region &r) {
  std::string s = "[";
  for (size_t i = 0; i < kDimCount; ++i)
    s += (i ? " x [" : "[") + std::to_string(r.lo[i]) + "," + std::to_string(r.hi[i]) + ")";
  return s + "]";
}

namespace detail {
inline std::array<i64, 4> dims_of(const TensorShape &s) { return {s.sample, s.channel, s.height, s.width}; }
inline std::array<i64, 4> dims_of(const Config &c) { return {c.sample, c.channel, c.height, c.width}; }
} // namespace detail

/// Dimensions a layer's output may be split along.
inline std::array<bool, kDimCount> parallelizable_dims(const LayerKind &kind, const TensorShape &shape) {
  if (is_kind<Conv2D>(kind) || is_kind<Pool2D>(kind)) return {{true, true, true, true}};
  if (is_kind<FullyConnected>(kind) || is_kind<Softmax>(kind)) return {{true, true, false, false}};
  return {{shape.sample > 1, shape.channel > 1, shape.height > 1, shape.width > 1}};
}

namespace detail {
inline std::vector<i64> divisors_up_to(i64 n, i64 cap) {
  std::vector<i64> out;
  for (i64 d = 1, lim = std::min(n, cap); d <= lim; ++d)
    if (n % d == 0) out.push_back(d);
  return out;
}
} // namespace detail

/// Every config whose degrees divide the extents, are 1 on non-parallelizable
/// dimensions and multiply to at most device_count; lexicographic order.
inline std::vector<Config> enumerate_configs(const LayerKind &kind, const TensorShape &shape, int device_count) {
  if (device_count < 1) throw InputError("enumerate_configs: need at least one device");
  const auto par = parallelizable_dims(kind, shape);
  const i64 cap = device_count;
  std::array<std::vector<i64>, kDimCount> ch;
  for (Dim d : kAllDims) {
    const auto i = static_cast<size_t>(d);
    ch[i] = par[i] ? detail::divisors_up_to(shape.extent(d), cap) : std::vector<i64>{1};
  }
  std::vector<Config> out;
  for (i64 n : ch[0])
    for (i64 c : ch[1]) {
      if (n * c > cap) break;
      for (i64 h : ch[2]) {
        if (n * c * h > cap) break;
        for (i64 w : ch[3]) {
          if (n * c * h * w > cap) break;
          out.push_back({n, c, h, w});
        }
      }
    }
  return out;
}

/// Output block of one partition (row-major decode, W fastest).
inline Region owned_region(const TensorShape &shape, const Config &config, i64 part_index) {
  if (part_index < 0 || part_index >= config.total())
    throw InputError("owned_region: partition index " + std::to_string(part_index) + " out of range for " +
                     std::to_string(config.total()) + " partitions");
  const auto s = detail::dims_of(shape), c = detail::dims_of(config);
  Region r;
  geo::owned_box(s.data(), c.data(), part_index, r.lo.data(), r.hi.data());
  return r;
}

namespace detail {
/// Sum of the preceding siblings' extents on a Concat's axis for `edge`.
inline i64 concat_band_offset(const ComputationGraph &graph, const Edge &edge) {
  const auto *cat = std::get_if<Concat>(&graph.layer(edge.dst).kind);
  if (!cat) return 0;
  i64 off = 0;
  for (int eid : graph.in_edges(edge.dst)) {
    const Edge &sib = graph.edge(eid);
    if (sib.dst_input_pos == edge.dst_input_pos) break;
    off += graph.edge_shape(sib).extent(cat->axis);
  }
  return off;
}
} // namespace detail

/// Input block (source coordinates) a destination partition reads over `edge`.
inline Region required_input_region(const ComputationGraph &graph, const Edge &edge, const Config &dst_config,
                                    i64 part_index) {
  const Layer &dst = graph.layer(edge.dst);
  if (part_index < 0 || part_index >= dst_config.total())
    throw InputError("owned_region: partition index " + std::to_string(part_index) + " out of range for " +
                     std::to_string(dst_config.total()) + " partitions");
  i64 params[7];
  detail::kind_params(dst.kind, params);
  const auto ins = detail::dims_of(graph.edge_shape(edge)), outs = detail::dims_of(graph.shape(edge.dst));
  const auto dc = detail::dims_of(dst_config);
  Region r;
  if (!geo::required_box(static_cast<int>(dst.kind.index()), params, ins.data(), outs.data(),
                         detail::concat_band_offset(graph, edge), dc.data(), part_index, r.lo.data(), r.hi.data()))
    throw InputError("layer '" + dst.id + "' does not consume inputs");
  return r;
}

/// Identity placement: partition i runs on device i.
struct Placement {
  i64 partition_count = 0;
  int device(i64 part_index) const { return static_cast<int>(part_index); }
};

inline Placement place(const Config &config, const DeviceGraph &devices) {
  if (config.total() > devices.count())
    throw InputError("config " + to_string(config) + " needs " + std::to_string(config.total()) + " devices, only " +
                     std::to_string(devices.count()) + " available");
  return Placement{config.total()};
}

} // namespace parplan

/* parplan/baselines.hpp — fixed reference strategies (data / model / OWT).
 *
 * Drop-in for /root/reference/proj/include/parplan/baselines.hpp:52-79
 * (BaselineKind, baseline_name, baseline_strategy).  Host code: one config per
 * layer, degree = the largest divisor of the split extent <= device count.
 */
#pragma once

#include "parplan/partition.hpp"

namespace parplan {

enum class BaselineKind { Data, Model, Owt };

inline const char *baseline_name(BaselineKind k) {
  return k == BaselineKind::Data ? "data" : k == BaselineKind::Model ? "model" : "owt";
}

namespace detail {
inline i64 largest_divisor_up_to(i64 n, i64 cap) {
  for (i64 d = std::min(n, cap); d > 1; --d)
    if (n % d == 0) return d;
  return 1;
}
} // namespace detail

/// data: every layer split over samples; model: parameterised layers over
/// output channels; owt: dense/softmax over channels, the rest over samples.
inline Strategy baseline_strategy(BaselineKind kind, const ComputationGraph &graph, const DeviceGraph &devices) {
  const i64 cap = devices.count();
  Strategy s(static_cast<size_t>(graph.layer_count()));
  for (int l = 0; l < graph.layer_count(); ++l) {
    const LayerKind &k = graph.layer(l).kind;
    const bool by_channel = (kind == BaselineKind::Model && has_parameters(k)) ||
                            (kind == BaselineKind::Owt && (is_kind<FullyConnected>(k) || is_kind<Softmax>(k)));
    Config c;
    if (by_channel)
      c.channel = detail::largest_divisor_up_to(graph.shape(l).channel, cap);
    else
      c.sample = detail::largest_divisor_up_to(graph.shape(l).sample, cap);
    s[static_cast<size_t>(l)] = c;
  }
  return s;
}

} // namespace parplan

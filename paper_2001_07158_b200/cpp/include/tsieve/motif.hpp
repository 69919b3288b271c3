// tsieve/motif.hpp -- query types of the B200 drop-in.
//
// Same names and meaning as the reference API
// (/root/reference/proj/core/include/tsieve/motif.hpp:11-74).  Every kind
// is evaluated on the device: size-only / multiset by the temporal sieve,
// timed kinds by the edge-constrained sieve, ordered colors by the
// vertex-ordered sieve (or the exact DP for VC-ColorfulPath).
#pragma once

#include <cstdint>
#include <map>
#include <vector>

namespace tsieve {

using Vertex = std::int32_t;
using Timestamp = std::int32_t;
using Color = std::int32_t;
using EdgeId = std::int32_t;

enum class QueryKind {
  size_only,
  multiset,
  ordered_colors,
  ordered_times_multiset,
  ordered_times_only,
};

struct MotifQuery {
  QueryKind kind = QueryKind::size_only;
  int k = 0;
  std::map<Color, int> multiset;  // ascending color -> multiplicity
  std::vector<Color> order;
  std::vector<Timestamp> times;

  static MotifQuery size_only(int k);
  static MotifQuery from_multiset(const std::vector<Color>& colors);
  static MotifQuery from_order(const std::vector<Color>& order);
  static MotifQuery from_times(const std::vector<Timestamp>& times,
                               const std::vector<Color>& colors);

  bool has_multiset() const {
    return kind == QueryKind::multiset || kind == QueryKind::ordered_times_multiset;
  }
  bool has_times() const {
    return kind == QueryKind::ordered_times_multiset || kind == QueryKind::ordered_times_only;
  }
};

inline MotifQuery MotifQuery::size_only(int k) {
  MotifQuery q;
  q.k = k;
  return q;
}

inline MotifQuery MotifQuery::from_multiset(const std::vector<Color>& colors) {
  MotifQuery q;
  q.kind = QueryKind::multiset;
  q.k = static_cast<int>(colors.size());
  for (Color c : colors) ++q.multiset[c];
  return q;
}

inline MotifQuery MotifQuery::from_order(const std::vector<Color>& order) {
  MotifQuery q = from_multiset(order);
  q.kind = QueryKind::ordered_colors;
  q.order = order;
  return q;
}

inline MotifQuery MotifQuery::from_times(const std::vector<Timestamp>& times,
                                         const std::vector<Color>& colors) {
  MotifQuery q = from_multiset(colors);
  q.kind = colors.empty() ? QueryKind::ordered_times_only : QueryKind::ordered_times_multiset;
  q.k = static_cast<int>(times.size()) + 1;
  q.times = times;
  return q;
}

}  // namespace tsieve

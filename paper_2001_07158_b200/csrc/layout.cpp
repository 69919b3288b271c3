// layout.cpp -- see layout.hpp.  Host C++ (OpenMP where it pays).
#include "layout.hpp"

#include <parallel/algorithm>

#include <algorithm>
#include <numeric>
#include <stdexcept>

namespace tsv {

void canonicalize(int32_t n, int64_t m, const int32_t* u, const int32_t* v,
                  const int32_t* ts, bool directed, int32_t t, HostLayout& L,
                  const int32_t* eps) {
  if (n < 0) throw std::invalid_argument("negative vertex count");
  L.n = n;
  L.directed = directed;
  L.dropped_self_loops = 0;
  struct E {
    int32_t ts, u, v, eps;
  };
  std::vector<E> kept;
  kept.reserve(static_cast<size_t>(m));
  for (int64_t i = 0; i < m; ++i) {
    int32_t a = u[i], b = v[i];
    if (a < 0 || a >= n || b < 0 || b >= n)
      throw std::invalid_argument("edge endpoint out of range");
    if (ts[i] < 1) throw std::invalid_argument("timestamp below 1");
    if (a == b) {
      ++L.dropped_self_loops;
      continue;
    }
    if (!directed && a > b) std::swap(a, b);
    kept.push_back({ts[i], a, b, eps ? eps[i] : 1});
  }
  auto key_less = [](const E& x, const E& y) {
    if (x.ts != y.ts) return x.ts < y.ts;
    if (x.u != y.u) return x.u < y.u;
    return x.v < y.v;
  };
  // multiway-mergesort on all host cores for the 1e8-1e9-edge configs
  // (transition times need std::sort's exact permutation for duplicates)
  if (kept.size() > (1u << 20) && !eps)
    __gnu_parallel::sort(kept.begin(), kept.end(), key_less);
  else
    std::sort(kept.begin(), kept.end(), key_less);
  auto same = [](const E& x, const E& y) {
    return x.ts == y.ts && x.u == y.u && x.v == y.v;
  };
  size_t w = 0;
  for (size_t i = 0; i < kept.size(); ++i)
    if (w == 0 || !same(kept[w - 1], kept[i])) kept[w++] = kept[i];
  L.dropped_duplicates = static_cast<int64_t>(kept.size() - w);
  kept.resize(w);
  if (w >= kEdgeMask)
    throw std::invalid_argument("edge count exceeds the engine's 2^30 edge ids");
  int32_t max_ts = 0;
  L.eu.resize(w);
  L.ev.resize(w);
  L.ets.resize(w);
  L.eeps.assign(eps ? w : 0, 1);
  for (size_t i = 0; i < w; ++i) {
    L.eu[i] = kept[i].u;
    L.ev[i] = kept[i].v;
    L.ets[i] = kept[i].ts;
    if (eps) L.eeps[i] = kept[i].eps;
    max_ts = std::max(max_ts, kept[i].ts);
  }
  L.t = t > 0 ? t : std::max<int32_t>(max_ts, 1);
  if (max_ts > L.t) throw std::invalid_argument("timestamp exceeds t");
}

void adopt_canonical(int32_t n, int64_t m, const int32_t* u, const int32_t* v,
                     const int32_t* ts, bool directed, int32_t t, HostLayout& L) {
  if (n < 0 || m < 0) throw std::invalid_argument("negative size");
  if (m >= static_cast<int64_t>(kEdgeMask))
    throw std::invalid_argument("edge count exceeds the engine's 2^30 edge ids");
  L.n = n;
  L.directed = directed;
  L.dropped_self_loops = L.dropped_duplicates = 0;
  L.eu.assign(u, u + m);
  L.ev.assign(v, v + m);
  L.ets.assign(ts, ts + m);
  int32_t max_ts = 0;
  for (int64_t i = 0; i < m; ++i) {
    if (u[i] < 0 || u[i] >= n || v[i] < 0 || v[i] >= n)
      throw std::invalid_argument("edge endpoint out of range");
    if (ts[i] < 1) throw std::invalid_argument("timestamp below 1");
    if (u[i] == v[i] || (!directed && u[i] > v[i]))
      throw std::invalid_argument("edge list is not canonical");
    if (i > 0) {
      const bool lt = ts[i - 1] != ts[i] ? ts[i - 1] < ts[i]
                      : u[i - 1] != u[i] ? u[i - 1] < u[i]
                                         : v[i - 1] < v[i];
      if (!lt) throw std::invalid_argument("edge list is not canonical");
    }
    max_ts = std::max(max_ts, ts[i]);
  }
  L.t = t > 0 ? t : std::max<int32_t>(max_ts, 1);
  if (max_ts > L.t) throw std::invalid_argument("timestamp exceeds t");
}

void build_layout(HostLayout& L, int64_t chunk_target, int sm_count) {
  const int32_t n = L.n;
  const int64_t m = static_cast<int64_t>(L.eu.size());
  const int64_t A = L.directed ? m : 2 * m;

  // Stable counting sort of arcs by head over edge order gives (head, ts)
  // order, since edges are sorted by ts (graph.cpp:34-36).
  std::vector<int64_t> head_off(static_cast<size_t>(n) + 1, 0);
  for (int64_t i = 0; i < m; ++i) {
    ++head_off[L.ev[i] + 1];
    if (!L.directed) ++head_off[L.eu[i] + 1];
  }
  for (int32_t x = 0; x < n; ++x) head_off[x + 1] += head_off[x];
  std::vector<int64_t> cur(head_off.begin(), head_off.end() - 1);
  std::vector<int32_t> a_tail(static_cast<size_t>(A)), a_edge(static_cast<size_t>(A)),
      a_ts(static_cast<size_t>(A));
  for (int64_t i = 0; i < m; ++i) {
    int64_t p = cur[L.ev[i]]++;
    a_tail[p] = L.eu[i];
    a_edge[p] = static_cast<int32_t>(i);
    a_ts[p] = L.ets[i];
    if (!L.directed) {
      p = cur[L.eu[i]]++;
      a_tail[p] = L.ev[i];
      a_edge[p] = static_cast<int32_t>(i);
      a_ts[p] = L.ets[i];
    }
  }

  // Runs: (head, ts) groups, vertex-major.
  L.run_head.clear();
  L.run_ts.clear();
  L.vtx_run_off.assign(static_cast<size_t>(n) + 1, 0);
  std::vector<int32_t> arc_run(static_cast<size_t>(A));
  for (int32_t x = 0; x < n; ++x) {
    L.vtx_run_off[x] = static_cast<int32_t>(L.run_head.size());
    for (int64_t p = head_off[x]; p < head_off[x + 1]; ++p) {
      if (p == head_off[x] || a_ts[p] != a_ts[p - 1]) {
        L.run_head.push_back(x);
        L.run_ts.push_back(a_ts[p]);
      }
      arc_run[p] = static_cast<int32_t>(L.run_head.size() - 1);
    }
  }
  L.vtx_run_off[n] = static_cast<int32_t>(L.run_head.size());
  if (L.run_head.size() >= (1ull << 31))
    throw std::invalid_argument("run count exceeds int32 indexing");

  // Per-arc predecessor state index and flags.
  L.arc_src.resize(static_cast<size_t>(A));
  L.arc_meta.resize(static_cast<size_t>(A));
  L.arc_tail = a_tail;
#pragma omp parallel for schedule(static)
  for (int64_t p = 0; p < A; ++p) {
    const int32_t x = a_tail[p];
    const int32_t* b = L.run_ts.data() + L.vtx_run_off[x];
    const int32_t* e = L.run_ts.data() + L.vtx_run_off[x + 1];
    const int32_t* it = std::lower_bound(b, e, a_ts[p]);  // first ts >= arc ts
    L.arc_src[p] = (it == b) ? -1 : static_cast<int32_t>((it - 1) - L.run_ts.data());
    uint32_t meta = static_cast<uint32_t>(a_edge[p]);
    const int32_t h = L.run_head[arc_run[p]];
    if (p == head_off[h]) meta |= kVStart;
    if (p + 1 == A || arc_run[p + 1] != arc_run[p]) meta |= kRunEnd;
    L.arc_meta[p] = meta;
  }

  // Chunks: pack whole vertices up to the target; split longer vertices.
  if (chunk_target <= 0) {
    const int64_t want = static_cast<int64_t>(std::max(sm_count, 1)) * 64;
    chunk_target = A / std::max<int64_t>(want, 1);
    chunk_target = std::clamp<int64_t>(chunk_target, 64, 2048);
  }
  L.chunk_arc.clear();
  L.chunk_carry.clear();
  L.chunk_arc.push_back(0);
  int64_t open = 0;  // arcs in the currently open chunk
  for (int32_t x = 0; x < n; ++x) {
    const int64_t deg = head_off[x + 1] - head_off[x];
    if (deg == 0) continue;
    if (deg > chunk_target) {
      if (open > 0) {
        L.chunk_arc.push_back(head_off[x]);
        L.chunk_carry.push_back(0);
        open = 0;
      }
      // pieces of chunk_target arcs; all but the first continue vertex x
      bool first = true;
      for (int64_t s = head_off[x]; s < head_off[x + 1]; s += chunk_target) {
        L.chunk_arc.push_back(std::min(s + chunk_target, head_off[x + 1]));
        L.chunk_carry.push_back(first ? 0 : 1);
        first = false;
      }
      continue;
    }
    if (open > 0 && open + deg > chunk_target) {
      L.chunk_arc.push_back(head_off[x]);
      L.chunk_carry.push_back(0);
      open = 0;
    }
    open += deg;
  }
  if (open > 0) {
    L.chunk_arc.push_back(A);
    L.chunk_carry.push_back(0);
  }
  const size_t C = L.chunk_carry.size();
  L.chunk_run.assign(C + 1, 0);
  for (size_t c = 0; c < C; ++c) {
    int32_t ends = 0;
    for (int64_t p = L.chunk_arc[c]; p < L.chunk_arc[c + 1]; ++p)
      ends += (L.arc_meta[p] & kRunEnd) ? 1 : 0;
    L.chunk_run[c + 1] = L.chunk_run[c] + ends;
  }
  L.carry_list.clear();
  for (size_t c = 0; c < C; ++c)
    if (L.chunk_carry[c]) L.carry_list.push_back(static_cast<int32_t>(c));
}

}  // namespace tsv

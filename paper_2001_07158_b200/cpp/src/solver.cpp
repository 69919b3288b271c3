// solver.cpp -- problem drivers on top of the GPU temporal sieve.
//
// Semantics follow /root/reference/proj/core/src/solver.cpp: effective
// instance (make_effective :42-126), preparation (prepare :499-546, color
// filter of preprocess_mask :458-497), the decision / optimum / extraction
// driver (solve_single :609-703: binary search :641-662, localized reverse
// DFS :314-394, self-reduction shrink_to_core :557-607 + forward DFS
// :398-452).  The rainbow / wildcard loops (:705-784) are out of scope.  Each probe is one
// engine call on the device: the temporal sieve (four problems, all edge
// models), the edge-constrained sieve (EC problems), the vertex-ordered sieve
// (VC-PathMotif) or the exact DP (VC-ColorfulPath).
#include "tsieve/solver.hpp"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <deque>
#include <functional>
#include <map>
#include <stdexcept>

#include "tsv.h"

namespace tsieve {

namespace {

using Clock = std::chrono::steady_clock;

double since(Clock::time_point t0) {
  return std::chrono::duration<double>(Clock::now() - t0).count();
}

struct Prep {
  Problem problem = Problem::path_motif;
  SieveConfig cfg;
  MotifQuery query;
  VertexColoring coloring;
  TemporalGraph graph;
  AnchorSpec anchor;
  ShadeAssignment shades;
  int k = 0;
  bool infeasible = false;
  std::string why;
  int kept = 0;
  double pre_s = 0;
  std::uint64_t peak = 0;
};

bool uses_shades(Problem p) {
  return p != Problem::vc_path_motif && p != Problem::vc_colorful_path;
}

void make_effective(const TemporalGraph& g, const VertexColoring& col, const SolveRequest& req,
                    Prep& p) {
  p.problem = req.problem;
  p.cfg = req.config;
  p.anchor = {};
  switch (req.problem) {
    case Problem::k_temp_path:
      if (req.query.kind != QueryKind::size_only)
        throw std::invalid_argument("k-TempPath takes a size-only query");
      p.query = MotifQuery::from_multiset(std::vector<Color>(static_cast<size_t>(
                                              std::max(req.query.k, 0)), 1));
      p.coloring = VertexColoring::uniform(g.n());
      break;
    case Problem::path_motif:
    case Problem::colorful_path:
      if (req.query.kind != QueryKind::multiset)
        throw std::invalid_argument("expected a color-multiset query");
      p.query = req.query;
      p.coloring = col;
      break;
    case Problem::sd_colorful_path: {
      if (req.query.kind != QueryKind::size_only)
        throw std::invalid_argument("(s,d)-ColorfulPath takes --k (interior size)");
      if (req.source < 0 || req.source >= g.n() || req.dest < 0 || req.dest >= g.n() ||
          req.source == req.dest)
        throw std::invalid_argument("invalid source/dest");
      const int k = req.query.k;
      std::vector<Color> c(static_cast<size_t>(g.n()));
      for (Vertex x = 0; x < g.n(); ++x) {
        const Color o = col.primary(x);
        c[x] = (o >= 1 && o <= k) ? o : k + 3;  // sentinel for off-range colors
      }
      c[req.source] = k + 1;
      c[req.dest] = k + 2;
      p.coloring = VertexColoring(std::move(c), k + 3);
      std::vector<Color> all;
      for (Color x = 1; x <= k + 2; ++x) all.push_back(x);
      p.query = MotifQuery::from_multiset(all);
      p.anchor = {req.source, req.dest};
      break;
    }
    case Problem::ec_temp_path: {
      if (req.query.kind != QueryKind::ordered_times_only)
        throw std::invalid_argument("EC-TempPath takes a timestamp tuple");
      p.query = MotifQuery::from_times(req.query.times,
                                       std::vector<Color>(static_cast<size_t>(req.query.k), 1));
      p.coloring = VertexColoring::uniform(g.n());
      break;
    }
    case Problem::ec_path_motif:
      if (req.query.kind != QueryKind::ordered_times_multiset)
        throw std::invalid_argument(
            "EC-PathMotif takes a timestamp tuple plus a color multiset");
      p.query = req.query;
      p.coloring = col;
      break;
    case Problem::vc_path_motif:
    case Problem::vc_colorful_path:
      if (req.query.kind != QueryKind::ordered_colors)
        throw std::invalid_argument("VC variants take an ordered color tuple");
      if (req.problem == Problem::vc_colorful_path) {
        std::vector<Color> sorted = req.query.order;
        std::sort(sorted.begin(), sorted.end());
        if (std::adjacent_find(sorted.begin(), sorted.end()) != sorted.end())
          throw std::invalid_argument("VC-ColorfulPath needs distinct colors");
      }
      p.query = req.query;
      p.coloring = col;
      break;
    case Problem::rainbow_path:
      throw std::logic_error("rainbow handled by its own driver");
  }
  p.k = p.query.k;
  if (p.k < 1) throw std::invalid_argument("k must be positive");
  if (p.query.has_times()) {
    const auto& ts = p.query.times;
    for (size_t i = 1; i < ts.size(); ++i)
      if (ts[i] <= ts[i - 1])
        throw std::invalid_argument("prescribed timestamps must strictly increase");
  }
}

// Kept-vertex mask (solver.cpp:458-497 of the reference): the exact color
// filter, then the junction sieve on the static projection of what is left
// (whp: flags exactly the vertices on a properly colored static k-path).
// TSIEVE_TRACE=1: phase wall times of solve() on stderr
void solve_mark(const char* what, Clock::time_point t0) {
  static const bool on = std::getenv("TSIEVE_TRACE") != nullptr;
  if (on)
    std::fprintf(stderr, "[solve] %-26s %9.1f ms\n", what,
                 std::chrono::duration<double, std::milli>(Clock::now() - t0).count());
}

std::vector<bool> preprocess_mask(const TemporalGraph& g, const Prep& p, PreprocessLevel level,
                                  std::uint64_t& peak) {
  std::vector<bool> keep(static_cast<size_t>(g.n()), true);
  if (level == PreprocessLevel::color_filter || level == PreprocessLevel::both) {
    for (Vertex x = 0; x < g.n(); ++x) {
      bool hit = false;
      for (const auto& kv : p.query.multiset)
        if (p.coloring.has_color(x, kv.first)) {
          hit = true;
          break;
        }
      keep[x] = hit;
    }
  }
  if ((level == PreprocessLevel::static_sieve || level == PreprocessLevel::both) &&
      !p.query.multiset.empty()) {
    MotifQuery relaxed;
    relaxed.kind = QueryKind::multiset;
    relaxed.k = p.k;
    relaxed.multiset = p.query.multiset;
    const auto jt0 = Clock::now();
    const ShadeAssignment sh = build_shades(relaxed, p.coloring, p.cfg);
    if (!sh.feasible) return std::vector<bool>(static_cast<size_t>(g.n()), false);
    solve_mark("junction: shades", jt0);
    const TemporalGraph filtered = restrict_to(g, keep, g.t());
    solve_mark("junction: color filter", jt0);
    const StaticProjection proj = StaticProjection::project(filtered);
    solve_mark("junction: projection", jt0);
    const SieveOutcome jo = eval_junction_sieve(proj, p.k, sh, p.cfg);
    solve_mark("junction: sieve", jt0);
    peak = std::max(peak, jo.peak_field_words);
    std::vector<bool> flagged(static_cast<size_t>(g.n()), false);
    for (Vertex x : jo.flagged) flagged[x] = true;
    for (Vertex x = 0; x < g.n(); ++x) keep[x] = keep[x] && flagged[x];
  }
  return keep;
}

Prep prepare(const TemporalGraph& g, const VertexColoring& col, const SolveRequest& req) {
  Prep p;
  const auto pt0 = Clock::now();
  make_effective(g, col, req, p);
  solve_mark("make_effective", pt0);
  const auto t0 = Clock::now();
  if (p.k > g.n()) {
    p.infeasible = true;
    p.why = "k exceeds vertex count";
    p.graph = g;
    return p;
  }
  if (p.query.has_times() &&
      (p.query.times.front() < 1 || p.query.times.back() > g.t())) {
    p.infeasible = true;
    p.why = "prescribed timestamp outside [1..t]";
    p.graph = g;
    return p;
  }
  if (uses_shades(p.problem)) {
    p.shades = build_shades(p.query, p.coloring, p.cfg);
    if (!p.shades.feasible) {
      p.infeasible = true;
      p.why = "query color " + std::to_string(p.shades.missing_color) + " absent from the graph";
      p.graph = g;
      return p;
    }
  }
  solve_mark("build_shades", pt0);
  PreprocessLevel level = req.preprocess;
  // the exact DP stays exact: only the lossless filter applies to it
  if (p.problem == Problem::vc_colorful_path &&
      (level == PreprocessLevel::static_sieve || level == PreprocessLevel::both))
    level = PreprocessLevel::color_filter;
  const std::vector<bool> keep = preprocess_mask(g, p, level, p.peak);
  solve_mark("preprocess mask", pt0);
  p.graph = restrict_to(g, keep, g.t());
  solve_mark("restrict_to", pt0);
  p.kept = static_cast<int>(std::count(keep.begin(), keep.end(), true));
  if (p.kept < p.k) {
    p.infeasible = true;
    p.why = "fewer than k vertices remain after preprocessing";
  }
  p.pre_s = since(t0);
  return p;
}

struct Probe {
  SieveOutcome out;
  bool exact = false;  // holds for every seed
};

// One oracle call of the problem's engine (solver.cpp:199-230 of the
// reference); every engine runs on the device.
Probe probe(const Prep& p, const TemporalGraph& graph, Timestamp max_ts) {
  Probe pr;
  switch (p.problem) {
    case Problem::ec_temp_path:
    case Problem::ec_path_motif:
      if (p.query.times.back() > max_ts) {
        pr.out.accumulators.assign(static_cast<size_t>(graph.n()), 0);
        pr.exact = true;
      } else {
        pr.out = eval_edge_constrained_sieve(graph, p.query.times, p.shades, p.cfg);
      }
      break;
    case Problem::vc_path_motif:
      pr.out = eval_vertex_ordered_sieve(graph, p.query.order, p.coloring, max_ts, p.cfg);
      break;
    case Problem::vc_colorful_path: {  // exact indicator DP (dp_probe)
      std::vector<std::uint8_t> f(static_cast<size_t>(graph.n()) + 1, 0);
      const int rc = tsv_vc_colorful_dp(
          graph.device_graph(tsieve::device()), p.k, p.query.order.data(),
          p.coloring.primaries().empty() ? nullptr : p.coloring.primaries().data(),
          p.coloring.wildcard_active() ? p.coloring.wildcard_color() : -1, max_ts, f.data());
      if (rc == TSV_ERR_INVALID) throw std::invalid_argument(tsv_last_error());
      if (rc != TSV_OK) throw std::runtime_error(tsv_last_error());
      pr.exact = true;
      pr.out.accumulators.assign(static_cast<size_t>(graph.n()), 0);
      std::uint64_t h = 1469598103934665603ull;
      for (Vertex u = 0; u < graph.n(); ++u)
        if (f[u]) {
          pr.out.accumulators[u] = 1;
          pr.out.flagged.push_back(u);
          h ^= static_cast<std::uint64_t>(u);
          h *= 1099511628211ull;
        }
      pr.out.global_nonzero = !pr.out.flagged.empty();
      pr.out.fn_bound = 0.0;
      pr.out.checksum = h;
      break;
    }
    default:
      pr.out = eval_temporal_sieve(graph, p.k, max_ts, p.shades, p.cfg, p.anchor);
  }
  return pr;
}

// ---- witness extraction (host DFS over the incidence lists) ---------------

struct Dfs {
  const TemporalGraph& g;
  const VertexColoring& col;
  const MotifQuery& q;
  AnchorSpec anchor;
  Timestamp horizon;
  EdgeModel model = EdgeModel::instant;
  std::map<Color, int> left;
  std::vector<char> used;
  std::vector<Vertex> chain;
  std::vector<TemporalEdge> chain_edges;

  Dfs(const TemporalGraph& g_, const VertexColoring& c_, const MotifQuery& q_, AnchorSpec a_,
      Timestamp h_)
      : g(g_), col(c_), q(q_), anchor(a_), horizon(h_), left(q_.multiset),
        used(static_cast<size_t>(g_.n()), 0) {}

  // Places v at 1-based position pos (consuming one unit of its color, or of
  // the wildcard color; ordered queries need the position's color) and runs
  // fn; undoes the consumption unless fn succeeds.
  template <typename Fn>
  bool place(Vertex v, int pos, Fn&& fn) {
    if (q.kind == QueryKind::ordered_colors)
      return col.has_color(v, q.order[static_cast<size_t>(pos - 1)]) && fn();
    auto attempt = [&](Color c) {
      auto it = left.find(c);
      if (it == left.end() || it->second == 0) return false;
      --it->second;
      const bool ok = fn();
      ++it->second;
      return ok;
    };
    if (attempt(col.primary(v))) return true;
    return col.wildcard_active() && attempt(col.wildcard_color());
  }

  // effective transition time / vertex delay (solver.cpp DfsCtx of the
  // reference): 1 unless the edge model uses them
  std::int32_t eps_eff(const TemporalEdge& e) const {
    return (model == EdgeModel::transition_only || model == EdgeModel::transition_delay) ? e.eps
                                                                                          : 1;
  }
  std::int32_t delta_eff(Vertex v) const {
    return (model == EdgeModel::delay_only || model == EdgeModel::transition_delay) ? g.delay(v)
                                                                                     : 1;
  }

  bool allowed(Vertex v, int pos) const {
    if (anchor.source >= 0 && ((v == anchor.source) != (pos == 1))) return false;
    if (anchor.sink >= 0 && ((v == anchor.sink) != (pos == q.k))) return false;
    return true;
  }

  bool step(Vertex v, const TemporalEdge& e, const std::function<bool()>& next) {
    used[v] = 1;
    chain.push_back(v);
    chain_edges.push_back(e);
    if (next()) return true;
    chain_edges.pop_back();
    chain.pop_back();
    used[v] = 0;
    return false;
  }

  // Reverse temporal DFS: fills position pos from the in-arcs of the current
  // first vertex, descending timestamps, ascending neighbor within a stamp.
  bool backward(int pos) {
    if (pos == 0) return true;
    const Vertex x = chain.back();
    const bool last_step = chain_edges.empty();
    Timestamp hi = last_step ? horizon : chain_edges.back().ts - delta_eff(x);
    const bool timed = q.has_times();
    if (timed) hi = std::min(hi, q.times[static_cast<size_t>(pos - 1)]);
    auto arcs = g.in_arcs(x);
    auto end = std::upper_bound(arcs.begin(), arcs.end(), hi,
                                [](Timestamp t, const Incidence& a) { return t < a.ts; });
    while (end != arcs.begin()) {
      const Timestamp ts = std::prev(end)->ts;
      auto beg = end;
      while (beg != arcs.begin() && std::prev(beg)->ts == ts) --beg;
      for (auto it = beg; it != end; ++it) {
        const Vertex v = it->other;
        if (used[v]) continue;
        const TemporalEdge& e = g.edge(it->edge);
        if (timed && it->ts != q.times[static_cast<size_t>(pos - 1)]) continue;
        if (last_step ? it->ts + eps_eff(e) - 1 > horizon
                      : chain_edges.back().ts - it->ts < eps_eff(e) + delta_eff(x) - 1)
          continue;
        if (!allowed(v, pos)) continue;
        if (place(v, pos, [&] { return step(v, e, [&] { return backward(pos - 1); }); }))
          return true;
      }
      end = beg;
    }
    return false;
  }

  // Forward temporal DFS: ascending timestamps, ascending neighbor.
  bool forward(int pos) {
    if (pos > q.k) return true;
    const Vertex x = chain.back();
    const Timestamp lo =
        chain_edges.empty()
            ? 1
            : chain_edges.back().ts +
                  std::max<std::int32_t>(0, eps_eff(chain_edges.back()) + delta_eff(x) - 1);
    auto arcs = g.out_arcs(x);
    auto it = std::lower_bound(arcs.begin(), arcs.end(), lo,
                               [](const Incidence& a, Timestamp t) { return a.ts < t; });
    for (; it != arcs.end(); ++it) {
      const Vertex v = it->other;
      if (used[v]) continue;
      const TemporalEdge& e = g.edge(it->edge);
      if (q.has_times() && it->ts != q.times[static_cast<size_t>(pos - 2)]) continue;
      if (it->ts + eps_eff(e) - 1 > horizon || !allowed(v, pos)) continue;
      if (place(v, pos, [&] { return step(v, e, [&] { return forward(pos + 1); }); }))
        return true;
    }
    return false;
  }
};

std::optional<TemporalPath> extract_backward(const Prep& p, Vertex end, Timestamp horizon) {
  Dfs d(p.graph, p.coloring, p.query, p.anchor, horizon);
  d.model = p.cfg.edge_model;
  if (!d.allowed(end, p.query.k)) return std::nullopt;
  const bool ok = d.place(end, p.query.k, [&] {
    d.used[end] = 1;
    d.chain.push_back(end);
    if (d.backward(p.query.k - 1)) return true;
    d.chain.pop_back();
    d.used[end] = 0;
    return false;
  });
  if (!ok) return std::nullopt;
  TemporalPath path;
  path.vertices.assign(d.chain.rbegin(), d.chain.rend());
  path.edges.assign(d.chain_edges.rbegin(), d.chain_edges.rend());
  return path;
}

std::optional<TemporalPath> extract_forward(const Prep& p, const TemporalGraph& core,
                                            Vertex start, Timestamp horizon) {
  Dfs d(core, p.coloring, p.query, p.anchor, horizon);
  d.model = p.cfg.edge_model;
  if (!d.allowed(start, 1)) return std::nullopt;
  const bool ok = d.place(start, 1, [&] {
    d.used[start] = 1;
    d.chain.push_back(start);
    if (d.forward(2)) return true;
    d.chain.pop_back();
    d.used[start] = 0;
    return false;
  });
  if (!ok) return std::nullopt;
  TemporalPath path;
  path.vertices = d.chain;
  path.edges = d.chain_edges;
  return path;
}

// Self-reduction, phase 1: shrink the vertex set with deletion probes on
// restricted graphs (block halving, then a linear cleanup).
std::vector<bool> shrink_to_core(const Prep& p, Timestamp horizon, int& calls,
                                 std::uint64_t& peak) {
  std::vector<bool> keep(static_cast<size_t>(p.graph.n()), false);
  for (const TemporalEdge& e : p.graph.edges()) keep[e.u] = keep[e.v] = true;
  std::vector<Vertex> cand;
  for (Vertex x = 0; x < p.graph.n(); ++x)
    if (keep[x]) cand.push_back(x);

  // Each deletion probe restricts the graph ON THE DEVICE (order-preserving
  // filter + rebuild, tsv_graph_restrict) and evaluates there; no host graph
  // is rebuilt per probe.
  const int model = static_cast<int>(p.cfg.edge_model);
  // the temporal sieve under the instant model restricts on the device; the
  // other engines / models restrict on the host and probe the result
  const bool temporal = p.problem == Problem::k_temp_path || p.problem == Problem::path_motif ||
                        p.problem == Problem::colorful_path ||
                        p.problem == Problem::sd_colorful_path;
  const bool on_device = temporal && model == 0;
  const tsv_graph* base = on_device ? p.graph.device_graph(tsieve::device()) : nullptr;
  tsv_config cfg{};
  cfg.seed = p.cfg.seed;
  cfg.field_bits = p.cfg.field_bits;
  cfg.lane_width = p.cfg.lane_width;
  cfg.edge_model = model;
  cfg.memory_cap_words = p.cfg.memory_cap_words;
  std::vector<std::uint8_t> mask8(static_cast<size_t>(p.graph.n()));
  std::vector<std::uint64_t> acc(static_cast<size_t>(p.graph.n()) + 1);
  static const std::int32_t kNoShade = 0;
  auto still_yes_without = [&](const std::vector<Vertex>& block) {
    for (Vertex x = 0; x < p.graph.n(); ++x) mask8[x] = keep[x] ? 1 : 0;
    for (Vertex x : block) mask8[x] = 0;
    if (!temporal) {
      std::vector<bool> kb(mask8.begin(), mask8.end());
      const TemporalGraph sub = restrict_to(p.graph, kb, horizon);
      const Probe pr = probe(p, sub, horizon);
      ++calls;
      peak = std::max(peak, pr.out.peak_field_words);
      return pr.out.global_nonzero;
    }
    tsv_graph* sub = nullptr;
    std::optional<TemporalGraph> host_sub;
    const tsv_graph* probe_graph = nullptr;
    if (model == 0) {
      if (tsv_graph_restrict(base, mask8.data(), horizon, &sub) != TSV_OK)
        throw std::runtime_error(tsv_last_error());
      probe_graph = sub;
    } else {  // delay models: restrict on the host, mirror for the model
      std::vector<bool> kb(mask8.begin(), mask8.end());
      host_sub.emplace(restrict_to(p.graph, kb, horizon));
      probe_graph = host_sub->device_graph(tsieve::device(), model);
    }
    tsv_outcome o{};
    const int rc = tsv_eval_temporal_sieve(
        probe_graph, p.k, horizon, p.shades.vertex_off.data(),
        p.shades.vertex_shades.empty() ? &kNoShade : p.shades.vertex_shades.data(), &cfg,
        p.anchor.source, p.anchor.sink, acc.data(), &o);
    if (sub) tsv_graph_free(sub);
    if (rc == TSV_ERR_INVALID) throw std::invalid_argument(tsv_last_error());
    if (rc != TSV_OK) throw std::runtime_error(tsv_last_error());
    ++calls;
    peak = std::max(peak, o.peak_field_words);
    if (p.cfg.localize) return o.global_nonzero != 0;
    std::uint64_t total = 0;
    for (Vertex x = 0; x < p.graph.n(); ++x) total ^= acc[x];
    return total != 0;
  };

  std::deque<std::vector<Vertex>> work{cand};
  std::vector<Vertex> survivors;
  while (!work.empty()) {
    std::vector<Vertex> block = std::move(work.front());
    work.pop_front();
    if (block.empty()) continue;
    if (still_yes_without(block)) {
      for (Vertex x : block) keep[x] = false;
    } else if (block.size() == 1) {
      survivors.push_back(block[0]);
    } else {
      const size_t half = block.size() / 2;
      work.emplace_back(block.begin(), block.begin() + half);
      work.emplace_back(block.begin() + half, block.end());
    }
  }
  for (Vertex x : survivors)
    if (keep[x] && still_yes_without({x})) keep[x] = false;
  return keep;
}

SolveReport solve_single(const TemporalGraph& g, const VertexColoring& col,
                         const SolveRequest& req, SolveMode mode) {
  SolveReport r;
  const Prep p = prepare(g, col, req);
  r.preprocessed_n = p.kept;
  r.preprocessed_m = p.graph.m();
  r.timings.preprocess_s = p.pre_s;
  r.peak_field_words = p.peak;
  if (p.infeasible) {
    r.certain = true;
    r.note = p.why;
    return r;
  }

  const auto t0 = Clock::now();
  const Timestamp full = p.graph.t();
  const Probe whole_probe = probe(p, p.graph, full);
  solve_mark("probe at t", t0);
  const SieveOutcome& whole = whole_probe.out;
  r.oracle_calls = 1;
  r.decision = whole.global_nonzero;
  // a nonzero accumulator certifies a match; NO is exact only for the
  // deterministic paths
  r.certain = whole_probe.exact || r.decision;
  r.flagged = whole.flagged;
  r.checksum = whole.checksum;
  r.peak_field_words = std::max(r.peak_field_words, whole.peak_field_words);
  r.timings.sieve_s = since(t0);
  if (!r.decision || mode == SolveMode::decide) {
    r.fn_bound = whole.fn_bound * r.oracle_calls;
    return r;
  }

  Timestamp horizon = full;
  SieveOutcome at = whole;
  if (mode == SolveMode::optimum || mode == SolveMode::extract_optimum) {
    const auto ts0 = Clock::now();
    Timestamp lo = 1, hi = full;
    while (lo < hi) {
      const Timestamp mid = lo + (hi - lo) / 2;
      const auto tp = Clock::now();
      SieveOutcome o = probe(p, p.graph, mid).out;
      if (std::getenv("TSIEVE_TRACE"))
        std::fprintf(stderr, "probe max_ts=%d %s %.3f ms\n", mid,
                     o.global_nonzero ? "YES" : "NO", 1e3 * since(tp));
      ++r.oracle_calls;
      r.peak_field_words = std::max(r.peak_field_words, o.peak_field_words);
      if (o.global_nonzero) {
        hi = mid;
        at = std::move(o);
      } else {
        lo = mid + 1;
      }
    }
    horizon = lo;
    r.optimum_ts = horizon;
    if (horizon == full) at = whole;
    r.timings.sieve_s += since(ts0);
  }

  if (mode == SolveMode::extract || mode == SolveMode::extract_optimum) {
    const auto te = Clock::now();
    auto accept = [&](std::optional<TemporalPath> w) {
      if (!w) return false;
      if (!validate_path(p.graph, p.coloring, *w, p.query, p.cfg.edge_model, p.anchor.source,
                         p.anchor.sink))
        return false;
      r.witness = std::move(*w);
      return true;
    };
    if (req.extraction == ExtractionStrategy::localized) {
      for (Vertex u : at.flagged)
        if (accept(extract_backward(p, u, horizon))) break;
    } else {
      int calls = 0;
      const std::vector<bool> core = shrink_to_core(p, horizon, calls, r.peak_field_words);
      r.oracle_calls += calls;
      const TemporalGraph cg = restrict_to(p.graph, core, horizon);
      for (Vertex u = 0; u < cg.n() && !r.witness; ++u)
        if (core[u]) accept(extract_forward(p, cg, u, horizon));
    }
    r.extraction_failed = !r.witness;
    r.timings.extract_s = since(te);
  }
  r.fn_bound = whole.fn_bound * r.oracle_calls;
  return r;
}

}  // namespace

const char* problem_name(Problem p) {
  switch (p) {
    case Problem::k_temp_path: return "ktemppath";
    case Problem::path_motif: return "pathmotif";
    case Problem::colorful_path: return "colorfulpath";
    case Problem::sd_colorful_path: return "sdcolorful";
    case Problem::rainbow_path: return "rainbow";
    case Problem::ec_temp_path: return "ectemppath";
    case Problem::ec_path_motif: return "ecpathmotif";
    case Problem::vc_path_motif: return "vcpathmotif";
    case Problem::vc_colorful_path: return "vccolorfulpath";
  }
  return "?";
}

std::optional<Problem> problem_from_name(const std::string& name) {
  for (int i = 0; i <= static_cast<int>(Problem::vc_colorful_path); ++i) {
    const auto p = static_cast<Problem>(i);
    if (name == problem_name(p)) return p;
  }
  return std::nullopt;
}

EffectiveInstance effective_instance(const TemporalGraph& g, const VertexColoring& coloring,
                                     const SolveRequest& req) {
  Prep p;
  make_effective(g, coloring, req, p);
  return {std::move(p.query), std::move(p.coloring), p.anchor, p.k};
}

SolveReport solve(const TemporalGraph& g, const VertexColoring& coloring,
                  const SolveRequest& req, SolveMode mode) {
  // The RainbowPath subset loop and the wildcard loop (solver.cpp:705-784 of
  // the reference) are outer drivers off the temporal-sieve path (SURVEY.md
  // section 2, out of scope): not provided by this engine.
  if (req.wildcard_max > 0)
    throw std::invalid_argument("--wildcards-max is not supported by the B200 engine");
  if (req.problem == Problem::rainbow_path)
    throw std::invalid_argument("RainbowPath is not supported by the B200 engine");
  return solve_single(g, coloring, req, mode);
}

SolveReport decide(const TemporalGraph& g, const VertexColoring& coloring,
                   const SolveRequest& req) {
  return solve(g, coloring, req, SolveMode::decide);
}

SolveReport find_optimum_timestamp(const TemporalGraph& g, const VertexColoring& coloring,
                                   const SolveRequest& req) {
  return solve(g, coloring, req, SolveMode::optimum);
}

SolveReport extract_localized(const TemporalGraph& g, const VertexColoring& coloring,
                              const SolveRequest& req, bool optimize) {
  SolveRequest r = req;
  r.extraction = ExtractionStrategy::localized;
  return solve(g, coloring, r, optimize ? SolveMode::extract_optimum : SolveMode::extract);
}

SolveReport extract_self_reducible(const TemporalGraph& g, const VertexColoring& coloring,
                                   const SolveRequest& req, bool optimize) {
  SolveRequest r = req;
  r.extraction = ExtractionStrategy::self_reducible;
  return solve(g, coloring, r, optimize ? SolveMode::extract_optimum : SolveMode::extract);
}

SolveReport decide_sd_colorful(const TemporalGraph& g, const VertexColoring& coloring,
                               Vertex source, Vertex dest, int k, const SieveConfig& config) {
  SolveRequest req;
  req.problem = Problem::sd_colorful_path;
  req.query = MotifQuery::size_only(k);
  req.source = source;
  req.dest = dest;
  req.config = config;
  return decide(g, coloring, req);
}

SolveReport decide_rainbow(const TemporalGraph& g, const VertexColoring& coloring, int k,
                           const SieveConfig& config) {
  SolveRequest req;
  req.problem = Problem::rainbow_path;
  req.query = MotifQuery::size_only(k);
  req.config = config;
  return decide(g, coloring, req);
}

SolveReport solve_with_wildcards(const TemporalGraph& g, const VertexColoring& coloring,
                                 const SolveRequest& req, int k_max) {
  SolveRequest r = req;
  r.wildcard_max = k_max;
  return solve(g, coloring, r, SolveMode::decide);
}

PreprocessResult preprocess(const TemporalGraph& g, const VertexColoring& coloring,
                            const SolveRequest& req, PreprocessLevel level) {
  SolveRequest sub = req;
  sub.preprocess = level;
  Prep p;
  make_effective(g, coloring, sub, p);
  PreprocessResult out;
  out.kept = preprocess_mask(g, p, level, out.peak_field_words);
  out.graph = restrict_to(g, out.kept, g.t());
  out.kept_count = static_cast<int>(std::count(out.kept.begin(), out.kept.end(), true));
  return out;
}

}  // namespace tsieve

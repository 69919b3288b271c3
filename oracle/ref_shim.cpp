// ref_shim.cpp -- own-code C entry points over the UNMODIFIED reference core.
//
// TEST INFRASTRUCTURE ONLY (see oracle/tsv_oracle.c header).  oracle/Makefile
// compiles this file together with /root/reference/proj/core/src/*.cpp (in
// place, never copied) into oracle/_ref/libtsieve_ref.so.  Python reaches it
// through oracle/oracle.py (ctypes) to pin the CPU restatement, to generate
// golden vectors, and as bench.py's reference CPU arm.
//
// Reference interfaces driven here (file:line under /root/reference/proj):
//   TemporalGraph::build        core/src/graph.cpp:14-109
//   load_graph                  core/src/graph.cpp:376-448
//   build_shades                core/src/sieve.cpp:658-718
//   eval_temporal_sieve         core/src/sieve.cpp:720-732
//   solve / SolveMode           core/src/solver.cpp:821-827
//   effective_instance          core/src/solver.cpp (make_effective :42-126)
//   validate_path               core/src/graph.cpp:238-333

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <sstream>
#include <string>
#include <vector>

#include "tsieve/gf.hpp"
#include "tsieve/graph.hpp"
#include "tsieve/sieve.hpp"
#include "tsieve/solver.hpp"

using namespace tsieve;

namespace {

std::string g_err;

// Edge-model overrides for the next ref_solve (ref_set_model; test driver
// state, cleared by ref_set_model(NULL, NULL, 0, 0)).
std::vector<std::int32_t> g_eps, g_delays;
int g_model = 0;
std::vector<std::int32_t> g_times, g_order;  // ref_set_query

TemporalGraph make_graph(int32_t n, int64_t m, const int32_t* u,
                         const int32_t* v, const int32_t* ts, int directed,
                         int32_t t) {
  std::vector<TemporalEdge> edges(static_cast<size_t>(m));
  const bool eps = static_cast<int64_t>(g_eps.size()) == m;
  for (int64_t i = 0; i < m; ++i) edges[i] = {u[i], v[i], ts[i], eps ? g_eps[i] : 1};
  TemporalGraph g = TemporalGraph::build(n, std::move(edges), directed != 0, t);
  if (static_cast<int32_t>(g_delays.size()) == n && n > 0) g.set_delays(g_delays);
  return g;
}

VertexColoring make_coloring(int32_t n, const int32_t* colors) {
  std::vector<Color> c(static_cast<size_t>(n), 1);
  Color q = 1;
  if (colors)
    for (int32_t i = 0; i < n; ++i) {
      c[i] = colors[i];
      q = std::max(q, c[i]);
    }
  return VertexColoring(std::move(c), q);
}

size_t put(char* buf, size_t cap, const std::string& s) {
  if (buf && cap) {
    size_t w = std::min(cap - 1, s.size());
    std::memcpy(buf, s.data(), w);
    buf[w] = 0;
  }
  return s.size();
}

}  // namespace

// field width of ref_eval_temporal / ref_solve (the reference's GF(2^b)
// dispatch, sieve.cpp:637-649); 64 unless set
static int g_field_bits = 64;

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_set_query(const int32_t* times, int32_t ntimes, const int32_t* order,
                   int32_t norder) {
  g_times.assign(times ? times : nullptr, times ? times + ntimes : nullptr);
  g_order.assign(order ? order : nullptr, order ? order + norder : nullptr);
}

void ref_set_model(const int32_t* eps, int64_t m, const int32_t* delays, int32_t n,
                   int32_t edge_model) {
  g_eps.assign(eps ? eps : nullptr, eps ? eps + m : nullptr);
  g_delays.assign(delays ? delays : nullptr, delays ? delays + n : nullptr);
  g_model = edge_model;
}

// gf::mul<uint64_t> (gf.hpp:85-106) and gf::draw_nonzero (gf.hpp:147-153).
uint64_t ref_gf_mul(uint64_t a, uint64_t b) { return gf::mul<std::uint64_t>(a, b); }
uint64_t ref_draw_nonzero(uint64_t seed, uint64_t role, uint64_t a, uint64_t b,
                          uint64_t c) {
  return gf::draw_nonzero<std::uint64_t>(seed, static_cast<gf::Role>(role), a, b, c);
}

// Canonical edge list of TemporalGraph::build; returns the kept count.
// eval_temporal_sieve of the reference under an edge model: edges carry
// transition times eps (NULL = 1), delays (NULL = none) are set on the
// graph, edge_model 0..3 = instant / transition / delay / both.
int64_t ref_eval_temporal_model(int32_t n, int64_t m, const int32_t* u, const int32_t* v,
                                const int32_t* ts, const int32_t* eps, const int32_t* delays,
                                int directed, int32_t t, const int32_t* colors,
                                const int32_t* motif, int32_t motif_len, int32_t max_ts,
                                uint64_t seed, int32_t lanes, int32_t edge_model,
                                int32_t anchor_source, int32_t anchor_sink, uint64_t* acc_out,
                                uint64_t* checksum_out, int32_t* out_u, int32_t* out_v,
                                int32_t* out_ts, int32_t* out_eps) {
  try {
    std::vector<TemporalEdge> edges(static_cast<size_t>(m));
    for (int64_t i = 0; i < m; ++i) edges[i] = {u[i], v[i], ts[i], eps ? eps[i] : 1};
    TemporalGraph g = TemporalGraph::build(n, std::move(edges), directed != 0, t);
    if (delays) g.set_delays(std::vector<std::int32_t>(delays, delays + n));
    for (int64_t i = 0; i < g.m(); ++i) {
      const TemporalEdge& e = g.edge(static_cast<EdgeId>(i));
      if (out_u) out_u[i] = e.u;
      if (out_v) out_v[i] = e.v;
      if (out_ts) out_ts[i] = e.ts;
      if (out_eps) out_eps[i] = e.eps;
    }
    VertexColoring col = make_coloring(n, colors);
    MotifQuery q = MotifQuery::from_multiset(std::vector<Color>(motif, motif + motif_len));
    SieveConfig cfg;
    cfg.seed = seed;
    cfg.lane_width = lanes;
    cfg.threads = 1;
    cfg.memory_cap_words = ~std::uint64_t{0};
    static const EdgeModel models[] = {EdgeModel::instant, EdgeModel::transition_only,
                                       EdgeModel::delay_only, EdgeModel::transition_delay};
    cfg.edge_model = models[edge_model & 3];
    ShadeAssignment sh = build_shades(q, col, cfg);
    if (!sh.feasible) return -2;
    if (max_ts <= 0) max_ts = g.t();
    SieveOutcome out = eval_temporal_sieve(g, motif_len, max_ts, sh, cfg,
                                           AnchorSpec{anchor_source, anchor_sink});
    for (int32_t i = 0; i < n; ++i) acc_out[i] = out.accumulators[i];
    *checksum_out = out.checksum;
    return g.m();
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

int64_t ref_canonical_edges(int32_t n, int64_t m, const int32_t* u,
                            const int32_t* v, const int32_t* ts, int directed,
                            int32_t* out_u, int32_t* out_v, int32_t* out_ts) {
  try {
    TemporalGraph g = make_graph(n, m, u, v, ts, directed, 0);
    for (int64_t i = 0; i < g.m(); ++i) {
      out_u[i] = g.edge(static_cast<EdgeId>(i)).u;
      out_v[i] = g.edge(static_cast<EdgeId>(i)).v;
      out_ts[i] = g.edge(static_cast<EdgeId>(i)).ts;
    }
    return g.m();
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// Shade CSR of build_shades for a color multiset query.  Returns the number
// of vertex_shades entries (vertex_off has n+1 entries), -1 on error, -2 if
// the query is infeasible (missing color).
int64_t ref_build_shades(int32_t n, const int32_t* colors, const int32_t* motif,
                         int32_t motif_len, uint64_t seed, int32_t* vertex_off,
                         int32_t* vertex_shades, int64_t cap) {
  try {
    VertexColoring col = make_coloring(n, colors);
    MotifQuery q = MotifQuery::from_multiset(
        std::vector<Color>(motif, motif + motif_len));
    SieveConfig cfg;
    cfg.seed = seed;
    ShadeAssignment sh = build_shades(q, col, cfg);
    if (!sh.feasible) return -2;
    for (int32_t i = 0; i <= n; ++i) vertex_off[i] = sh.vertex_off[i];
    int64_t cnt = static_cast<int64_t>(sh.vertex_shades.size());
    for (int64_t i = 0; i < cnt && i < cap; ++i)
      vertex_shades[i] = sh.vertex_shades[i];
    return cnt;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// eval_temporal_sieve on a graph built from raw edges with a color-multiset
// query.  acc_out receives the n accumulators.  Returns the seconds spent in
// eval_temporal_sieve (>= 0), -1 on error, -2 if the query is infeasible.
void ref_set_field_bits(int32_t b) { g_field_bits = b; }

double ref_eval_temporal(int32_t n, int64_t m, const int32_t* u,
                         const int32_t* v, const int32_t* ts, int directed,
                         int32_t t, const int32_t* colors,
                         const int32_t* motif, int32_t motif_len,
                         int32_t max_ts, uint64_t seed, int32_t lanes,
                         int32_t threads, int32_t anchor_source,
                         int32_t anchor_sink, int32_t repeats,
                         uint64_t* acc_out, uint64_t* checksum_out,
                         int64_t* nflagged_out, int32_t* global_out) {
  try {
    TemporalGraph g = make_graph(n, m, u, v, ts, directed, t);
    VertexColoring col = make_coloring(n, colors);
    MotifQuery q = MotifQuery::from_multiset(
        std::vector<Color>(motif, motif + motif_len));
    SieveConfig cfg;
    cfg.seed = seed;
    cfg.lane_width = lanes;
    cfg.threads = threads;
    cfg.field_bits = g_field_bits;
    cfg.memory_cap_words = ~std::uint64_t{0};
    ShadeAssignment sh = build_shades(q, col, cfg);
    if (!sh.feasible) return -2;
    AnchorSpec anchor{anchor_source, anchor_sink};
    if (max_ts <= 0) max_ts = g.t();
    SieveOutcome out;
    double best = -1;
    for (int r = 0; r < std::max(1, repeats); ++r) {
      auto t0 = std::chrono::steady_clock::now();
      out = eval_temporal_sieve(g, q.k, max_ts, sh, cfg, anchor);
      double s = std::chrono::duration<double>(
                     std::chrono::steady_clock::now() - t0)
                     .count();
      if (best < 0 || s < best) best = s;
    }
    for (int32_t i = 0; i < n; ++i) acc_out[i] = out.accumulators[i];
    *checksum_out = out.checksum;
    *nflagged_out = static_cast<int64_t>(out.flagged.size());
    *global_out = out.global_nonzero ? 1 : 0;
    return best;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// Full solver run (decide / optimum / extract) through solve().  problem is
// the CLI name (ktemppath, pathmotif, colorfulpath, sdcolorful); mode is
// 0 decide, 1 optimum, 2 extract, 3 extract_optimum; extraction 0 localized,
// 1 self-reducible; preprocess 0 none, 1 colors, 2 static, 3 both.  Writes a
// compact JSON record into buf and returns its length, or -1 on error.
int64_t ref_solve(int32_t n, int64_t m, const int32_t* u, const int32_t* v,
                  const int32_t* ts, int directed, int32_t t,
                  const int32_t* colors, const char* problem,
                  const int32_t* motif, int32_t motif_len, int32_t k,
                  int32_t source, int32_t dest, uint64_t seed, int32_t mode,
                  int32_t extraction, int32_t preprocess, char* buf,
                  int64_t cap) {
  try {
    TemporalGraph g = make_graph(n, m, u, v, ts, directed, t);
    VertexColoring col = make_coloring(n, colors);
    SolveRequest req;
    auto p = problem_from_name(problem);
    if (!p) throw std::invalid_argument("unknown problem");
    req.problem = *p;
    if (!g_order.empty())
      req.query = MotifQuery::from_order(std::vector<Color>(g_order.begin(), g_order.end()));
    else if (!g_times.empty())
      req.query = MotifQuery::from_times(
          std::vector<Timestamp>(g_times.begin(), g_times.end()),
          std::vector<Color>(motif, motif + std::max(motif_len, 0)));
    else if (motif_len > 0)
      req.query = MotifQuery::from_multiset(
          std::vector<Color>(motif, motif + motif_len));
    else
      req.query = MotifQuery::size_only(k);
    req.source = source;
    req.dest = dest;
    req.config.seed = seed;
    req.config.threads = 1;
    req.config.field_bits = g_field_bits;
    static const EdgeModel models[] = {EdgeModel::instant, EdgeModel::transition_only,
                                       EdgeModel::delay_only, EdgeModel::transition_delay};
    req.config.edge_model = models[g_model & 3];
    static const PreprocessLevel levels[] = {
        PreprocessLevel::none, PreprocessLevel::color_filter,
        PreprocessLevel::static_sieve, PreprocessLevel::both};
    req.preprocess = levels[preprocess & 3];
    req.extraction = extraction ? ExtractionStrategy::self_reducible
                                : ExtractionStrategy::localized;
    static const SolveMode modes[] = {SolveMode::decide, SolveMode::optimum,
                                      SolveMode::extract,
                                      SolveMode::extract_optimum};
    SolveReport r = solve(g, col, req, modes[mode & 3]);
    std::ostringstream os;
    char cs[32];
    std::snprintf(cs, sizeof cs, "%016llx",
                  static_cast<unsigned long long>(r.checksum));
    os << "{\"decision\":" << (r.decision ? "true" : "false")
       << ",\"certain\":" << (r.certain ? "true" : "false")
       << ",\"optimum_ts\":" << r.optimum_ts
       << ",\"oracle_calls\":" << r.oracle_calls << ",\"checksum\":\"" << cs
       << "\",\"extraction_failed\":"
       << (r.extraction_failed ? "true" : "false") << ",\"flagged\":[";
    for (size_t i = 0; i < r.flagged.size(); ++i)
      os << (i ? "," : "") << r.flagged[i];
    os << "],\"witness\":";
    if (r.witness) {
      os << "{\"vertices\":[";
      for (size_t i = 0; i < r.witness->vertices.size(); ++i)
        os << (i ? "," : "") << r.witness->vertices[i];
      os << "],\"edges\":[";
      for (size_t i = 0; i < r.witness->edges.size(); ++i) {
        const TemporalEdge& e = r.witness->edges[i];
        os << (i ? "," : "") << "[" << e.u << "," << e.v << "," << e.ts << "]";
      }
      os << "]}";
    } else {
      os << "null";
    }
    os << ",\"preprocessed_n\":" << r.preprocessed_n
       << ",\"preprocessed_m\":" << r.preprocessed_m << "}";
    return static_cast<int64_t>(put(buf, static_cast<size_t>(cap), os.str()));
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// load_graph on in-memory text; writes canonical edges (dense ids, rank
// timestamps), colors and t.  Returns m or -1.  names (may be null) receives
// the '\n'-joined vertex tokens.
int64_t ref_load_graph(const char* edge_text, const char* color_text,
                       int directed, int32_t* n_out, int32_t* t_out,
                       int32_t* out_u, int32_t* out_v, int32_t* out_ts,
                       int64_t cap, int32_t* colors_out, int32_t ncap,
                       char* names, int64_t names_cap) {
  try {
    std::istringstream es(edge_text);
    std::istringstream cs(color_text ? color_text : "");
    LoadResult lr = load_graph(es, color_text ? &cs : nullptr, directed != 0);
    *n_out = lr.graph.n();
    *t_out = lr.graph.t();
    for (int64_t i = 0; i < lr.graph.m() && i < cap; ++i) {
      out_u[i] = lr.graph.edge(static_cast<EdgeId>(i)).u;
      out_v[i] = lr.graph.edge(static_cast<EdgeId>(i)).v;
      out_ts[i] = lr.graph.edge(static_cast<EdgeId>(i)).ts;
    }
    for (int32_t i = 0; i < lr.graph.n() && i < ncap; ++i)
      colors_out[i] = lr.coloring.primary(i);
    std::string joined;
    for (size_t i = 0; i < lr.vertex_names.size(); ++i)
      joined += (i ? "\n" : "") + lr.vertex_names[i];
    put(names, static_cast<size_t>(names_cap), joined);
    return lr.graph.m();
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

}  // extern "C"

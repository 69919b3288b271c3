// sieve.cpp -- shade assignment (host) and the GPU-backed temporal sieve.
// build_shades follows /root/reference/proj/core/src/sieve.cpp:658-718;
// eval_temporal_sieve replaces sieve.cpp:720-732 by the C-ABI call.
#include <cstdlib>
#include "tsieve/sieve.hpp"
#include "tsieve/prefault.hpp"

#include <algorithm>
#include <bit>
#include <cmath>
#include <stdexcept>
#include <string>

#include "tsv.h"

namespace tsieve {

namespace {

void check_config(const SieveConfig& cfg) {
  if (cfg.field_bits != 8 && cfg.field_bits != 16 && cfg.field_bits != 32 &&
      cfg.field_bits != 64)
    throw std::invalid_argument("field_bits must be 8, 16, 32 or 64");
  if (cfg.lane_width < 1 || cfg.lane_width > 256 ||
      !std::has_single_bit(static_cast<unsigned>(cfg.lane_width)))
    throw std::invalid_argument("lane_width must be a power of two in [1,256]");
  if (cfg.threads < 1) throw std::invalid_argument("threads must be >= 1");
}

}  // namespace

double false_negative_bound(int k, int field_bits) {
  return (2.0 * k - 1.0) / std::pow(2.0, field_bits);
}

// Shades (sieve.cpp:658-718): the query's colors in ascending order get
// consecutive shade ids 1..k, multiplicity many each; a vertex carries the
// shades of its primary color (plus those of the wildcard color when one is
// active).  Every vertex's list is a run of consecutive ids, so the CSR is a
// prefix sum of per-vertex counts, computed on all host threads (n = 1e8 at
// C5).
ShadeAssignment build_shades(const MotifQuery& query, const VertexColoring& coloring,
                             const SieveConfig& config) {
  check_config(config);
  if (query.multiset.empty()) throw std::invalid_argument("build_shades needs a color multiset");
  int total = 0;
  for (const auto& kv : query.multiset) total += kv.second;
  if (total != query.k) throw std::invalid_argument("multiset multiplicities do not sum to k");

  ShadeAssignment sh;
  sh.k = query.k;
  sh.seed = config.seed;
  const std::int64_t n = coloring.n();
  const Color q = coloring.q();
  // colors present among the primaries (every color when a wildcard is active)
  std::vector<char> present(static_cast<size_t>(q) + 2, 0);
  if (coloring.wildcard_active()) {
    const Color w = coloring.wildcard_color();
    if (w >= 0 && w < static_cast<Color>(present.size())) present[w] = 1;
  }
#pragma omp parallel for schedule(static) if (n > (1 << 20))
  for (std::int64_t x = 0; x < n; ++x) {
    const Color c = coloring.primary(static_cast<Vertex>(x));
    if (c >= 0 && c < static_cast<Color>(present.size()) && !present[c]) present[c] = 1;
  }
  // per color: first shade id and how many (0: not in the query)
  std::vector<std::int32_t> first(static_cast<size_t>(q) + 2, 0), many(first.size(), 0);
  int next = 1;
  for (const auto& [c, mu] : query.multiset) {  // std::map: ascending colors
    sh.colors.push_back(c);
    std::vector<int> ids(static_cast<size_t>(mu));
    for (int i = 0; i < mu; ++i) ids[i] = next + i;
    sh.shade_sets.push_back(std::move(ids));
    if (c >= 0 && c < static_cast<Color>(first.size())) {
      first[c] = next;
      many[c] = mu;
    }
    next += mu;
    const bool here = c >= 1 && c < static_cast<Color>(present.size()) && present[c];
    if (!here && sh.feasible) {
      sh.feasible = false;
      sh.missing_color = c;
    }
  }
  const Color wild = coloring.wildcard_active() ? coloring.wildcard_color() : -1;
  const std::int32_t wf = wild >= 0 && wild < static_cast<Color>(first.size()) ? first[wild] : 0;
  const std::int32_t wm = wild >= 0 && wild < static_cast<Color>(first.size()) ? many[wild] : 0;
  auto own = [&](std::int64_t x, std::int32_t& f, std::int32_t& c) {
    const Color col = coloring.primary(static_cast<Vertex>(x));
    const bool in = col >= 0 && col < static_cast<Color>(first.size());
    f = in ? first[col] : 0;
    c = in ? many[col] : 0;
  };
  detail::reserve_prefaulted(sh.vertex_off, static_cast<size_t>(n) + 1);
  sh.vertex_off.assign(static_cast<size_t>(n) + 1, 0);
  const std::int64_t block = std::int64_t{1} << 16;
  const std::int64_t nb = (n + block - 1) / block;
  std::vector<std::int64_t> part(static_cast<size_t>(nb) + 1, 0);
#pragma omp parallel for schedule(static) if (n > (1 << 20))
  for (std::int64_t b = 0; b < nb; ++b) {
    std::int64_t acc = 0;
    for (std::int64_t x = b * block; x < std::min(n, (b + 1) * block); ++x) {
      std::int32_t f, c;
      own(x, f, c);
      acc += c + wm;
      sh.vertex_off[x + 1] = static_cast<std::int32_t>(acc);  // block-local for now
    }
    part[b + 1] = acc;
  }
  for (std::int64_t b = 0; b < nb; ++b) part[b + 1] += part[b];
  detail::reserve_prefaulted(sh.vertex_shades, static_cast<size_t>(part[nb]));
  sh.vertex_shades.resize(static_cast<size_t>(part[nb]));
#pragma omp parallel for schedule(static) if (n > (1 << 20))
  for (std::int64_t b = 0; b < nb; ++b) {
    for (std::int64_t x = b * block; x < std::min(n, (b + 1) * block); ++x) {
      sh.vertex_off[x + 1] += static_cast<std::int32_t>(part[b]);
      std::int32_t f, c;
      own(x, f, c);
      std::int32_t at = sh.vertex_off[x + 1] - c - wm;
      for (std::int32_t i = 0; i < c; ++i) sh.vertex_shades[at++] = f + i;
      for (std::int32_t i = 0; i < wm; ++i) sh.vertex_shades[at++] = wf + i;
    }
  }
  return sh;
}

namespace {
// The reference's default cap (2^31 words) bounds ITS dense layers (host
// RAM, sieve.cpp:161-166); the engine's sparse state lives in HBM and is
// bounded by the device itself, so the default means "no cap" here (C4 /
// C5 would otherwise fall back to the slower engines under 16 GB).  Any
// other value is the bound on the engine's working set (CapError beyond).
std::uint64_t engine_cap(const SieveConfig& config) {
  return config.memory_cap_words == SieveConfig{}.memory_cap_words ? ~std::uint64_t{0}
                                                                    : config.memory_cap_words;
}
int default_device() {
  const char* e = std::getenv("TSV_DEVICE");
  return e ? std::atoi(e) : 0;
}
thread_local int t_device = default_device();
void finish(SieveOutcome& out, int k, const SieveConfig& config, const tsv_outcome& o);
}  // namespace

void set_device(int d) { t_device = d; }
int device() { return t_device; }

SieveOutcome eval_temporal_sieve(const TemporalGraph& g, int k, Timestamp max_ts,
                                 const ShadeAssignment& shades, const SieveConfig& config,
                                 const AnchorSpec& anchor) {
  check_config(config);
  if (max_ts < 1 || max_ts > g.t()) throw std::invalid_argument("max_ts outside [1..t]");
  if (static_cast<int>(shades.vertex_off.size()) != g.n() + 1)
    throw std::invalid_argument("shade assignment built for a different graph");
  const int model = static_cast<int>(config.edge_model);  // enum order = tsv.h codes

  tsv_config c{};
  c.seed = config.seed;
  c.field_bits = config.field_bits;
  c.lane_width = config.lane_width;
  c.edge_model = model;
  c.points_per_batch = 0;
  c.memory_cap_words = engine_cap(config);

  SieveOutcome out;
  detail::reserve_prefaulted(out.accumulators, static_cast<size_t>(g.n()));
  out.accumulators.assign(static_cast<size_t>(g.n()), 0);
  std::uint64_t scratch = 0;
  tsv_outcome o{};
  static const std::int32_t kNoShade = 0;
  const int rc = tsv_eval_temporal_sieve(
      g.device_graph(tsieve::device(), model), k, max_ts, shades.vertex_off.data(),
      shades.vertex_shades.empty() ? &kNoShade : shades.vertex_shades.data(), &c,
      anchor.source, anchor.sink, g.n() ? out.accumulators.data() : &scratch, &o);
  if (rc == TSV_ERR_INVALID) throw std::invalid_argument(tsv_last_error());
  if (rc != TSV_OK) throw std::runtime_error(tsv_last_error());

  finish(out, k, config, o);
  return out;
}

namespace {

// Decision rule, fn bound and checksum of finalize (sieve.cpp:136-159).
// The flagged list (ascending nonzero accumulators) is gathered on all host
// threads: per-block counts, a scan, then an ordered fill.
void finish(SieveOutcome& out, int k, const SieveConfig& config, const tsv_outcome& o) {
  const auto& acc = out.accumulators;
  const int64_t n = static_cast<int64_t>(acc.size());
  const int64_t block = int64_t{1} << 16;
  const int64_t nb = (n + block - 1) / block;
  std::vector<int64_t> cnt(static_cast<size_t>(nb) + 1, 0);
  std::uint64_t total = 0;
#pragma omp parallel for schedule(static) reduction(^ : total) if (n > (1 << 20))
  for (int64_t b = 0; b < nb; ++b) {
    int64_t c = 0;
    for (int64_t x = b * block; x < std::min(n, (b + 1) * block); ++x) {
      c += acc[static_cast<size_t>(x)] != 0;
      total ^= acc[static_cast<size_t>(x)];
    }
    cnt[static_cast<size_t>(b) + 1] = c;
  }
  for (int64_t b = 0; b < nb; ++b) cnt[b + 1] += cnt[b];
  detail::reserve_prefaulted(out.flagged, static_cast<size_t>(cnt[nb]));
  out.flagged.resize(static_cast<size_t>(cnt[nb]));
#pragma omp parallel for schedule(static) if (n > (1 << 20))
  for (int64_t b = 0; b < nb; ++b) {
    int64_t w = cnt[b];
    for (int64_t x = b * block; x < std::min(n, (b + 1) * block); ++x)
      if (acc[static_cast<size_t>(x)]) out.flagged[static_cast<size_t>(w++)] = static_cast<Vertex>(x);
  }
  if (config.localize) {
    out.global_nonzero = !out.flagged.empty();
  } else {
    out.global_nonzero = total != 0;
  }
  out.fn_bound = false_negative_bound(k, config.field_bits);
  out.peak_field_words = o.peak_field_words;
  out.checksum = o.checksum;
}

tsv_config to_abi(const SieveConfig& config) {
  tsv_config c{};
  c.seed = config.seed;
  c.field_bits = config.field_bits;
  c.lane_width = config.lane_width;
  c.edge_model = 0;
  c.memory_cap_words = engine_cap(config);
  return c;
}

}  // namespace

SieveOutcome eval_delay_sieve(const TemporalGraph& g, int k, Timestamp max_ts,
                              const ShadeAssignment& shades, const SieveConfig& config) {
  if (config.edge_model == EdgeModel::instant)
    throw std::invalid_argument("eval_delay_sieve requires a delay edge model");
  return eval_temporal_sieve(g, k, max_ts, shades, config);
}

SieveOutcome eval_edge_constrained_sieve(const TemporalGraph& g,
                                         const std::vector<Timestamp>& times,
                                         const ShadeAssignment& shades,
                                         const SieveConfig& config) {
  check_config(config);
  if (times.empty()) throw std::invalid_argument("times must be nonempty");
  for (std::size_t i = 0; i < times.size(); ++i) {
    if (times[i] < 1 || times[i] > g.t())
      throw std::invalid_argument("prescribed timestamp outside [1..t]");
    if (i > 0 && times[i] <= times[i - 1])
      throw std::invalid_argument("prescribed timestamps must strictly increase");
  }
  const int k = static_cast<int>(times.size()) + 1;
  SieveOutcome out;
  detail::reserve_prefaulted(out.accumulators, static_cast<size_t>(g.n()));
  out.accumulators.assign(static_cast<size_t>(g.n()), 0);
  // a prescribed timestamp with no edge is a certain NO (sieve.cpp:767-774)
  for (Timestamp ts : times)
    if (g.runs_at(ts).empty()) {
      out.fn_bound = 0.0;
      out.checksum = 1469598103934665603ull;  // FNV-1a basis: no nonzero entries
      return out;
    }
  if (static_cast<int>(shades.vertex_off.size()) != g.n() + 1)
    throw std::invalid_argument("shade assignment built for a different graph");
  const tsv_config c = to_abi(config);
  std::uint64_t scratch = 0;
  static const std::int32_t kNoShade = 0;
  tsv_outcome o{};
  const int rc = tsv_eval_edge_constrained(
      g.device_graph(tsieve::device()), k, times.data(), shades.vertex_off.data(),
      shades.vertex_shades.empty() ? &kNoShade : shades.vertex_shades.data(), &c,
      g.n() ? out.accumulators.data() : &scratch, &o);
  if (rc == TSV_ERR_INVALID) throw std::invalid_argument(tsv_last_error());
  if (rc != TSV_OK) throw std::runtime_error(tsv_last_error());
  finish(out, k, config, o);
  return out;
}

SieveOutcome eval_vertex_ordered_sieve(const TemporalGraph& g, const std::vector<Color>& order,
                                       const VertexColoring& coloring, Timestamp max_ts,
                                       const SieveConfig& config) {
  check_config(config);
  if (order.empty()) throw std::invalid_argument("order must be nonempty");
  if (max_ts < 1 || max_ts > g.t()) throw std::invalid_argument("max_ts outside [1..t]");
  const int k = static_cast<int>(order.size());
  const tsv_config c = to_abi(config);
  SieveOutcome out;
  detail::reserve_prefaulted(out.accumulators, static_cast<size_t>(g.n()));
  out.accumulators.assign(static_cast<size_t>(g.n()), 0);
  std::uint64_t scratch = 0;
  static const std::int32_t kNoColor = 0;
  tsv_outcome o{};
  const int rc = tsv_eval_vertex_ordered(
      g.device_graph(tsieve::device()), k, order.data(),
      coloring.primaries().empty() ? &kNoColor : coloring.primaries().data(),
      coloring.wildcard_active() ? coloring.wildcard_color() : -1, max_ts, &c,
      g.n() ? out.accumulators.data() : &scratch, &o);
  if (rc == TSV_ERR_INVALID) throw std::invalid_argument(tsv_last_error());
  if (rc != TSV_OK) throw std::runtime_error(tsv_last_error());
  finish(out, k, config, o);
  return out;
}

namespace {

SieveOutcome eval_projection(const StaticProjection& gs, int k, const ShadeAssignment& shades,
                             const SieveConfig& config, bool junction) {
  check_config(config);
  if (static_cast<int>(shades.vertex_off.size()) != gs.n() + 1)
    throw std::invalid_argument("shade assignment built for a different graph");
  std::vector<std::int32_t> a(static_cast<size_t>(gs.m()) + 1), b(a.size());
  for (std::int64_t i = 0; i < gs.m(); ++i) {
    a[i] = gs.edges()[i].first;
    b[i] = gs.edges()[i].second;
  }
  tsv_config c{};
  c.seed = config.seed;
  c.field_bits = config.field_bits;
  c.lane_width = config.lane_width;
  c.memory_cap_words = engine_cap(config);
  SieveOutcome out;
  out.accumulators.assign(static_cast<size_t>(gs.n()), 0);
  std::uint64_t scratch = 0;
  static const std::int32_t kNoShade = 0;
  tsv_outcome o{};
  const int rc = tsv_eval_static_projection(
      gs.n(), gs.m(), a.data(), b.data(), gs.directed() ? 1 : 0, junction ? 1 : 0, k,
      shades.vertex_off.data(),
      shades.vertex_shades.empty() ? &kNoShade : shades.vertex_shades.data(), &c, tsieve::device(),
      gs.n() ? out.accumulators.data() : &scratch, &o);
  if (rc == TSV_ERR_INVALID) throw std::invalid_argument(tsv_last_error());
  if (rc != TSV_OK) throw std::runtime_error(tsv_last_error());
  for (Vertex x = 0; x < gs.n(); ++x)
    if (out.accumulators[x]) out.flagged.push_back(x);
  if (config.localize) {
    out.global_nonzero = !out.flagged.empty();
  } else {
    std::uint64_t total = 0;
    for (std::uint64_t v : out.accumulators) total ^= v;
    out.global_nonzero = total != 0;
  }
  out.fn_bound = false_negative_bound(k, config.field_bits);
  out.peak_field_words = o.peak_field_words;
  out.checksum = o.checksum;
  return out;
}

}  // namespace

SieveOutcome eval_static_sieve(const StaticProjection& gs, int k, const ShadeAssignment& shades,
                               const SieveConfig& config) {
  return eval_projection(gs, k, shades, config, false);
}

SieveOutcome eval_junction_sieve(const StaticProjection& gs, int k,
                                 const ShadeAssignment& shades, const SieveConfig& config) {
  return eval_projection(gs, k, shades, config, true);
}

}  // namespace tsieve

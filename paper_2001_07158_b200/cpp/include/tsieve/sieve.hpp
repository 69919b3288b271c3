// tsieve/sieve.hpp -- the temporal sieve entry point of the B200 drop-in.
//
// Same declarations as /root/reference/proj/core/include/tsieve/sieve.hpp
// for the temporal path (SieveConfig :24-32, ShadeAssignment :39-56,
// build_shades :61-63, SieveOutcome :65-72, AnchorSpec :76-79,
// eval_temporal_sieve :84-87, false_negative_bound).  eval_temporal_sieve
// runs on the GPU through tsv_eval_temporal_sieve (include/tsv.h); there is
// no host evaluation.  Field widths other than 64 and non-instant edge
// models are rejected with std::invalid_argument.  The static, junction,
// edge-constrained and vertex-ordered engines are not part of this path.
#pragma once

#include <cstdint>
#include <span>
#include <vector>

#include "tsieve/graph.hpp"
#include "tsieve/motif.hpp"

namespace tsieve {

struct SieveConfig {
  std::uint64_t seed = 1;
  int field_bits = 64;
  int lane_width = 8;  // accepted for compatibility; results never depend on it
  int threads = 1;     // accepted for compatibility; the GPU grid replaces it
  bool localize = true;
  EdgeModel edge_model = EdgeModel::instant;
  std::uint64_t memory_cap_words = std::uint64_t{1} << 31;
};

// CUDA device that the calling thread's evaluations run on (engine extension,
// kept out of SieveConfig so its layout is the reference's).  Default: the
// TSV_DEVICE environment variable, else 0.
void set_device(int device);
int device();

struct ShadeAssignment {
  int k = 0;
  std::uint64_t seed = 0;
  bool feasible = true;
  Color missing_color = 0;
  std::vector<Color> colors;
  std::vector<std::vector<int>> shade_sets;
  std::vector<std::int32_t> vertex_off;
  std::vector<std::int32_t> vertex_shades;

  std::span<const std::int32_t> shades_of(Vertex u) const {
    return {vertex_shades.data() + vertex_off[u], vertex_shades.data() + vertex_off[u + 1]};
  }
};

ShadeAssignment build_shades(const MotifQuery& query, const VertexColoring& coloring,
                             const SieveConfig& config);

struct SieveOutcome {
  bool global_nonzero = false;
  std::vector<std::uint64_t> accumulators;
  std::vector<Vertex> flagged;
  double fn_bound = 0.0;
  std::uint64_t peak_field_words = 0;
  std::uint64_t checksum = 0;
};

struct AnchorSpec {
  Vertex source = -1;
  Vertex sink = -1;
};

SieveOutcome eval_temporal_sieve(const TemporalGraph& g, int k, Timestamp max_ts,
                                 const ShadeAssignment& shades, const SieveConfig& config,
                                 const AnchorSpec& anchor = {});

// Static-projection engines (sieve.hpp:90-102 of the reference), also on
// the GPU: the junction sieve is the default preprocessing pass.
SieveOutcome eval_static_sieve(const StaticProjection& gs, int k, const ShadeAssignment& shades,
                               const SieveConfig& config);
SieveOutcome eval_junction_sieve(const StaticProjection& gs, int k,
                                 const ShadeAssignment& shades, const SieveConfig& config);

// Delay-model entry (sieve.hpp of the reference): eval_temporal_sieve under
// a non-instant config.edge_model.
SieveOutcome eval_delay_sieve(const TemporalGraph& g, int k, Timestamp max_ts,
                              const ShadeAssignment& shades, const SieveConfig& config);

// Edge-constrained sieve: the l-th edge of the path must carry timestamp
// times[l-2] (sieve.cpp:477-536, 758-780 of the reference); on the GPU.
SieveOutcome eval_edge_constrained_sieve(const TemporalGraph& g,
                                         const std::vector<Timestamp>& times,
                                         const ShadeAssignment& shades,
                                         const SieveConfig& config);

// Vertex-ordered sieve: position l must carry color order[l-1]
// (sieve.cpp:540-635, 782-794); on the GPU.
SieveOutcome eval_vertex_ordered_sieve(const TemporalGraph& g, const std::vector<Color>& order,
                                       const VertexColoring& coloring, Timestamp max_ts,
                                       const SieveConfig& config);

double false_negative_bound(int k, int field_bits);

}  // namespace tsieve

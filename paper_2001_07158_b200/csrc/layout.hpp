// layout.hpp -- host-side construction of the engine's HBM layout.
//
// From raw temporal edges this builds exactly the canonical edge ids of
// TemporalGraph::build (/root/reference/proj/core/src/graph.cpp:14-43) and
// then, instead of the reference's time-major ArcRun table (graph.cpp:50-79),
// a VERTEX-MAJOR event layout:
//
//   runs   = distinct (head, ts) pairs, ordered by (head, ts)      -> R entries
//   arcs   = grouped by run in that order; per arc:
//              src  = index of the tail's last run with ts' < ts (or -1):
//                     the state P[l-1][tail][ts-1] of sieve.cpp:249-250
//              meta = edge id | VSTART (first arc of its head's segment)
//                             | RUNEND (last arc of its run)
//              tail (level-2 base case and the (s,d) anchor only)
//   chunks = contiguous arc ranges, one per warp; whole vertices except
//            vertices longer than the chunk target, which are split into
//            pieces that need a carry fix-up of the per-vertex prefix.
//
// Field arithmetic is exact, so the per-vertex prefix XOR over runs in time
// order is the reference's stay term (sieve.cpp:229-230) made event-driven.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace tsv {

constexpr uint32_t kVStart = 1u << 31;
constexpr uint32_t kRunEnd = 1u << 30;
constexpr uint32_t kEdgeMask = kRunEnd - 1;

struct HostLayout {
  int32_t n = 0, t = 0;
  bool directed = false;
  int64_t dropped_self_loops = 0, dropped_duplicates = 0;
  // canonical edges (edge id = index); eeps only when transition times given
  std::vector<int32_t> eu, ev, ets, eeps;
  // vertex-major runs
  std::vector<int32_t> run_head, run_ts;
  std::vector<int32_t> vtx_run_off;  // n+1
  // arcs in run order
  std::vector<int32_t> arc_src, arc_tail;
  std::vector<uint32_t> arc_meta;
  // chunks
  std::vector<int64_t> chunk_arc;   // C+1
  std::vector<int32_t> chunk_run;   // C+1: run-ends before the chunk
  std::vector<uint8_t> chunk_carry; // C: first arc continues a vertex
  std::vector<int32_t> carry_list;  // chunks with chunk_carry set
};

// Canonical edges per graph.cpp:14-43.  Throws std::invalid_argument with the
// reference's messages on range errors.  t == 0 takes the max timestamp.
// eps (nullable): per-edge transition times carried to L.eeps; among
// duplicate (ts,u,v) edges the one std::sort leaves first is kept, as in
// the reference (same comparator and input sequence => same permutation).
void canonicalize(int32_t n, int64_t m, const int32_t* u, const int32_t* v,
                  const int32_t* ts, bool directed, int32_t t, HostLayout& L,
                  const int32_t* eps = nullptr);

// Adopts an edge list that must already be canonical (strictly increasing
// (ts,u,v), u != v, u < v when undirected); throws std::invalid_argument
// otherwise.
void adopt_canonical(int32_t n, int64_t m, const int32_t* u, const int32_t* v,
                     const int32_t* ts, bool directed, int32_t t, HostLayout& L);

// Builds runs/arcs/chunks from L's canonical edges.  chunk_target = arcs per
// chunk (0 = choose from the arc count and the SM count).
void build_layout(HostLayout& L, int64_t chunk_target, int sm_count);

}  // namespace tsv

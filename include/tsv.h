/*
 * tsv.h -- C-ABI of the B200 temporal-sieve engine (libtsv.so).
 *
 * Plain pointers and sizes only.  This is the boundary the host side of the
 * reference would bind: the C++ drop-in (paper_2001_07158_b200/cpp, same API
 * as /root/reference/proj/core/include/tsieve/{graph,sieve}.hpp) and the
 * Python mirror (paper_2001_07158_b200 package, ctypes) both call it.  There is
 * no CPU fallback: every compute entry point runs CUDA kernels for sm_100a or
 * returns TSV_ERR_CUDA.
 *
 * Status codes: 0 ok; TSV_ERR_INVALID maps to the reference's
 * std::invalid_argument, TSV_ERR_CAP to std::runtime_error (memory cap,
 * sieve.cpp:161-166), TSV_ERR_CUDA to a device failure.  tsv_last_error()
 * returns the message of the last failure on the calling thread.
 */
#ifndef TSV_H_
#define TSV_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TSV_OK 0
#define TSV_ERR_INVALID 1
#define TSV_ERR_CAP 2
#define TSV_ERR_CUDA 3

/* Opaque device-resident temporal graph: runs (head, ts) in vertex-major
 * order, arcs grouped by run with their predecessor-state index, chunk table.
 * Immutable after creation, so binary-search probes reuse it. */
typedef struct tsv_graph tsv_graph;
/* Opaque device-resident shade CSR (ShadeAssignment, sieve.hpp:39-56). */
typedef struct tsv_shades tsv_shades;

typedef struct {
  int32_t n;          /* vertices */
  int32_t t;          /* timestamp range [1..t] */
  int32_t directed;
  int32_t device;     /* CUDA ordinal the graph lives on */
  int64_t m;          /* canonical edges (edge id = index) */
  int64_t arcs;       /* m directed, 2m undirected */
  int64_t runs;       /* distinct (ts, head) pairs */
  int64_t chunks;     /* work chunks of the level kernel */
  int64_t split_chunks; /* chunks that continue a vertex (carry fix-up) */
  int64_t dropped_self_loops;
  int64_t dropped_duplicates;
  int64_t device_bytes; /* bytes of graph structure resident in HBM */
  int64_t arcs_with_src;   /* arcs with a predecessor run (gathers per level) */
  int64_t runs_referenced; /* runs some arc reads (stores per level < k) */
} tsv_graph_info;

/* Replaces TemporalGraph::build (graph.cpp:14-109) for the engine: drops
 * self-loops, orients undirected edges u<v, sorts by (ts,u,v), removes
 * duplicates (edge id = index), groups arcs into (ts, head) runs and uploads
 * the layout to `device`.  t = 0 takes the max timestamp.  Errors: endpoint
 * out of range, timestamp < 1 or > t (TSV_ERR_INVALID). */
int tsv_graph_build(int32_t n, int64_t m, const int32_t* u, const int32_t* v,
                    const int32_t* ts, int directed, int32_t t, int device,
                    tsv_graph** out);

/* Same, for an edge list that is ALREADY canonical (what a host-side
 * TemporalGraph holds): validated in O(m) instead of re-sorted. */
int tsv_graph_build_canonical(int32_t n, int64_t m, const int32_t* u,
                              const int32_t* v, const int32_t* ts,
                              int directed, int32_t t, int device,
                              tsv_graph** out);

/* Device mirror of an ALREADY canonical edge list under an edge model
 * (EdgeModel, graph.hpp:179; sieve.cpp:179-186, 257-291): 0 instant,
 * 1 transition times eps[m] (NULL = all 1), 2 vertex delays delays[n]
 * (NULL = all 0), 3 both.  An arc departing at ts lands in slot
 * ts + eps - 1 of its head and reads its tail's state at ts - delta(tail)
 * (delta = delay, or 1 without a delay model).  Evaluations must use the
 * same config edge_model.  Errors: eps < 1, negative delays, as for
 * tsv_graph_build_canonical. */
int tsv_graph_build_model(int32_t n, int64_t m, const int32_t* u, const int32_t* v,
                          const int32_t* ts, const int32_t* eps, const int32_t* delays,
                          int directed, int32_t t, int edge_model, int device,
                          tsv_graph** out);

/* Host-only canonicalization (no device): the edge list TemporalGraph::build
 * keeps, in edge-id order.  Returns the kept count (<= m) or -1 on error. */
int64_t tsv_canonical_edges(int32_t n, int64_t m, const int32_t* u,
                            const int32_t* v, const int32_t* ts, int directed,
                            int32_t* out_u, int32_t* out_v, int32_t* out_ts);

/* Same, carrying per-edge transition times (eps may be NULL; out_eps may be
 * NULL).  Among duplicate (ts,u,v) edges the survivor is the reference's
 * (same std::sort permutation, graph.cpp:34-41). */
int64_t tsv_canonical_edges_eps(int32_t n, int64_t m, const int32_t* u,
                                const int32_t* v, const int32_t* ts,
                                const int32_t* eps, int directed, int32_t* out_u,
                                int32_t* out_v, int32_t* out_ts, int32_t* out_eps);

/* Induced subgraph on the device (restrict_to, graph.cpp:483-494): edges with
 * ts <= max_ts whose endpoints are both kept (keep_vertex: n host bytes);
 * kept edges keep their relative order, so the rebuild's edge ids are their
 * ranks, exactly as the reference renumbers.  t = min(max_ts, t).  Used by
 * the self-reduction extraction probes. */
int tsv_graph_restrict(const tsv_graph* g, const uint8_t* keep_vertex,
                       int32_t max_ts, tsv_graph** out);

void tsv_graph_free(tsv_graph* g);
int tsv_graph_get_info(const tsv_graph* g, tsv_graph_info* out);

/* Copies the canonical edge list (m entries each) back to the host. */
int tsv_graph_edges(const tsv_graph* g, int32_t* u, int32_t* v, int32_t* ts);

/* The graph's static projection, computed on its device (replaces the host
 * grouping of StaticProjection::project, graph.cpp:148-199 of the
 * reference): *ms distinct (a, b) pairs in ascending order (a < b for
 * undirected graphs) into a[], b[] (capacity m each), back_off[ms + 1] and
 * back[m] = the temporal edge ids of each pair, increasing within a pair.
 * Host arrays. */
int tsv_graph_static_edges(const tsv_graph* g, int64_t* ms, int32_t* a, int32_t* b,
                           int32_t* back_off, int32_t* back);

/* Uploads a shade CSR: vertex_off[n+1], vertex_shades[vertex_off[n]] with
 * 1-based shade ids in [1..k] (build_shades, sieve.cpp:658-718). */
int tsv_shades_upload(const tsv_graph* g, int k, const int32_t* vertex_off,
                      const int32_t* vertex_shades, tsv_shades** out);
void tsv_shades_free(tsv_shades* s);

typedef struct {
  uint64_t seed;             /* SieveConfig::seed */
  int32_t field_bits;        /* must be 64 */
  int32_t lane_width;        /* accepted, results independent of it */
  int32_t edge_model;        /* 0 instant, 1 transition, 2 delay, 3 both (the
                                graph must be built for it) */
  int32_t points_per_batch;  /* 0 = engine choice; else power of two <= 128 */
  uint64_t memory_cap_words; /* SieveConfig::memory_cap_words */
} tsv_config;

typedef struct {
  int32_t global_nonzero;    /* decision (localize rule, sieve.cpp:149-150) */
  int32_t pad;
  int64_t flagged;           /* number of nonzero accumulators */
  uint64_t checksum;         /* FNV-1a fold, sieve.cpp:35-49 */
  uint64_t peak_field_words; /* field words resident during the evaluation */
  double fn_bound;           /* (2k-1)/2^64 */
} tsv_outcome;

/* Replaces eval_temporal_sieve (sieve.hpp:84-87, sieve.cpp:720-732) for the
 * instant edge model over GF(2^64).  accumulators: host buffer of n words
 * (zero-extended, sink-only when anchor_sink >= 0).  Synchronous. */
int tsv_eval_temporal_sieve(const tsv_graph* g, int k, int32_t max_ts,
                            const int32_t* vertex_off,
                            const int32_t* vertex_shades,
                            const tsv_config* cfg, int32_t anchor_source,
                            int32_t anchor_sink, uint64_t* accumulators,
                            tsv_outcome* out);

/* Sharded / device-resident form: XORs the contributions of sieve points
 * A in [p_begin, p_end) into the DEVICE buffer d_acc (n words, caller-owned,
 * not cleared) on `stream` (cudaStream_t, 0 = legacy default).  No finalize,
 * no host copies.  Used for multi-GPU sieve-point sharding and timing. */
int tsv_eval_points_device(const tsv_graph* g, const tsv_shades* s, int k,
                           int32_t max_ts, const tsv_config* cfg,
                           int32_t anchor_source, uint64_t p_begin,
                           uint64_t p_end, uint64_t* d_acc, void* stream);

/* Edge-constrained sieve (eval_edge_constrained_sieve, sieve.cpp:477-536,
 * 758-780): level l uses only the edges with timestamp times[l-2]
 * (times: k-1 strictly increasing stamps in [1..t]); per-vertex state, no
 * anchor.  Instant model only. */
int tsv_eval_edge_constrained(const tsv_graph* g, int k, const int32_t* times,
                              const int32_t* vertex_off, const int32_t* vertex_shades,
                              const tsv_config* cfg, uint64_t* accumulators,
                              tsv_outcome* out);

/* Vertex-ordered sieve (eval_vertex_ordered_sieve, sieve.cpp:540-635,
 * 782-794): positional z (Role::label_z) and, at level l, only arcs whose
 * tail has color order[l-2] and head order[l-1] (colors: n primary colors;
 * wildcard_color matches every vertex, -1 = none). */
int tsv_eval_vertex_ordered(const tsv_graph* g, int k, const int32_t* order,
                            const int32_t* colors, int32_t wildcard_color,
                            int32_t max_ts, const tsv_config* cfg,
                            uint64_t* accumulators, tsv_outcome* out);

/* VC-ColorfulPath's exact indicator DP (dp_probe, solver.cpp:146-191) in
 * earliest-arrival form on the device; flagged[n] = 1 where a path realizing
 * the order ends by max_ts. */
int tsv_vc_colorful_dp(const tsv_graph* g, int k, const int32_t* order,
                       const int32_t* colors, int32_t wildcard_color, int32_t max_ts,
                       uint8_t* flagged);

/* Static-projection engines over the projection's edge list (a[i], b[i]),
 * i = static edge id (StaticProjection::project, graph.cpp:148-199):
 * junction != 0 replaces eval_junction_sieve (sieve.cpp:376-473, the
 * default `--preprocess both` pass), junction == 0 eval_static_sieve
 * (sieve.cpp:311-369).  Synchronous; accumulators = n host words. */
int tsv_eval_static_projection(int32_t n, int64_t ms, const int32_t* a,
                               const int32_t* b, int directed, int junction,
                               int k, const int32_t* vertex_off,
                               const int32_t* vertex_shades,
                               const tsv_config* cfg, int device,
                               uint64_t* accumulators, tsv_outcome* out);

/* d_out[i] = XOR_{p < nparts} d_parts[p*n + i] (multi-GPU combine). */
int tsv_xor_combine_device(const uint64_t* d_parts, int nparts, int64_t n,
                           uint64_t* d_out, void* stream);

/* Host finalize of accumulators (sieve.cpp:136-159): sink restriction,
 * flagged count, checksum.  Modifies acc in place when anchor_sink >= 0. */
int tsv_finalize(int32_t n, uint64_t* acc, int32_t anchor_sink,
                 tsv_outcome* out);

/* Device finalize (finalize.cu): zeroes all but the sink of the DEVICE
 * accumulators when anchor_sink >= 0, then the flagged count and the FNV-1a
 * checksum (out->flagged, checksum, global_nonzero), computed in parallel
 * on the device.  Synchronizes `stream`. */
int tsv_finalize_device(uint64_t* d_acc, int64_t n, int32_t anchor_sink, void* stream,
                        tsv_outcome* out);

/* ---- Vertex-partitioned evaluation (multi-GPU) ----
 * One full evaluation (all 2^k points, coefficient form) split by HEAD
 * VERTEX: rank r of `world` owns the vertices [n r/world, n (r+1)/world)
 * and computes their state rows level by level (vertex-lane engine,
 * coef_vertex.cu: every shaded vertex multi-shade, k <= 5, no hubs).
 * Between levels the caller makes every rank's rows visible to all ranks:
 * rows of level l live at [slot_lo, slot_hi) x row_words[l] in each rank's
 * full-size state buffer (an all-gather of those ranges; shard.py).  At
 * level k every rank XORs the readout of its own vertices into d_acc. */
typedef struct {
  int32_t applicable;        /* 0: hub vertices or k out of range: use point sharding */
  int32_t pad;
  int64_t slot_lo, slot_hi;  /* this rank's state rows */
  int64_t slots;             /* all state rows */
  int64_t state_words;       /* words of each of the two state buffers */
  int32_t row_words[32];     /* row stride of level l: C(k, l) */
} tsv_partition;

int tsv_vertex_partition(const tsv_graph* g, const tsv_shades* s, int k, int rank,
                         int world, tsv_partition* out);
/* Level `level` (2..k) of rank's share: reads level-1 rows from d_prev
 * (unused at level 2), writes its level rows into d_cur (level < k) or XORs
 * its vertices' readout into d_acc (level k).  Asynchronous on `stream`. */
int tsv_eval_vertex_level(const tsv_graph* g, const tsv_shades* s, int k, int level,
                          int32_t max_ts, const tsv_config* cfg, int32_t anchor_source,
                          int rank, int world, const uint64_t* d_prev, uint64_t* d_cur,
                          uint64_t* d_acc, void* stream);

/* The same level with the row exchange inside the kernel: a
 * row is stored into d_cur and, as it is formed, into peer_cur[q] of every
 * OTHER rank q that reads it (its reader byte, fixed per graph) --
 * peer_cur[0..world) are the ranks' level buffers as mapped on THIS device
 * (NVLink peer memory, e.g. torch symmetric memory; peer_cur[rank] is
 * ignored, a null entry is skipped), world <= 8.  After a barrier across
 * the ranks every buffer holds the rows its rank reads; no pack / all-to-all
 * / unpack.  Replaces the reference's per-block loop over one machine's
 * lanes (sieve.cpp:199-304) across GPUs.  Asynchronous on `stream`. */
int tsv_eval_vertex_level_peer(const tsv_graph* g, const tsv_shades* s, int k, int level,
                               int32_t max_ts, const tsv_config* cfg, int32_t anchor_source,
                               int rank, int world, const uint64_t* d_prev, uint64_t* d_cur,
                               uint64_t* d_acc, uint64_t* const* peer_cur, void* stream);

/* Targeted row exchange between levels (instead of an all-gather): rank
 * sends to peer q exactly its rows some arc of q reads, receives likewise;
 * the lists are fixed per graph.  plan: row counts per peer (world <= 8);
 * pack: this rank's outgoing rows of level-l buffer d_rows (row_words =
 * C(k, l)) into d_sendbuf, peers in rank order; unpack: d_recvbuf (peers in
 * rank order) into d_rows.  The bytes in between move with one all-to-all
 * (shard.py).  Asynchronous on `stream`. */
typedef struct {
  int64_t send_rows[32], recv_rows[32];
  int64_t send_total, recv_total;
} tsv_exchange;
int tsv_vertex_exchange_plan(const tsv_graph* g, const tsv_shades* s, int k, int rank,
                             int world, tsv_exchange* out);
int tsv_vertex_exchange_pack(const tsv_graph* g, int rank, int world, int row_words,
                             const uint64_t* d_rows, uint64_t* d_sendbuf, void* stream);
int tsv_vertex_exchange_unpack(const tsv_graph* g, int rank, int world, int row_words,
                               const uint64_t* d_recvbuf, uint64_t* d_rows, void* stream);

/* Ascending indices of the nonzero words of acc[0..n) (the flagged list of
 * finalize, sieve.cpp:136-159) into idx (capacity n), on all host threads.
 * Returns the count. */
int64_t tsv_nonzero_index(const uint64_t* acc, int64_t n, int32_t* idx);

/* Per-kernel device-time profile (CUDA events on the launching stream).
 * names: "level", "level_first", "fixup", "readout", "zj" ... */
int tsv_profile_enable(int on);
int tsv_profile_get(const char* kernel, int64_t* launches, double* total_ms);
int tsv_profile_reset(void);
/* Number of engine kernels launched since the last reset. */
int64_t tsv_kernel_launches(void);

/* GF(2^64) on device (replaces gf::mul<uint64_t>, gf.hpp:85-106): self-test
 * of n products (a[i]*b[i] -> out[i], host buffers) with the production
 * general multiply (variant 0) or another form: 1 bit-serial, 2 holes +
 * Karatsuba, 3 holes + schoolbook, 4-6 warp-uniform shared-memory tables, 9
 * period-5 holes, 10 the per-lane shared-memory table of the vertex-lane
 * engine's arc products (tsv_gf_bench: 10 / 11 / 12 = 1 / 5 / 10 products
 * per table build). */
int tsv_gf_mul_device(int variant, int64_t n, const uint64_t* a,
                      const uint64_t* b, uint64_t* out);
/* Throughput microbenchmark: products/s of a variant (device only). */
int tsv_gf_bench(int variant, int64_t iters_per_thread, double* products_per_s);
/* y draws on device (draw_nonzero(seed, role=3, edge, level-1, 0)). */
int tsv_draw_edge_y_device(uint64_t seed, int32_t level, int64_t n,
                           const int32_t* edges, uint64_t* out);

const char* tsv_last_error(void);
const char* tsv_version(void);

#ifdef __cplusplus
}
#endif
#endif /* TSV_H_ */

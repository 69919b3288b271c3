// engine.hpp -- device-side views and kernel launchers (internal).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <functional>

namespace tsv {

// Device pointers of a resident graph (layout.hpp describes the arrays).
struct DevGraph {
  int32_t n = 0;
  int64_t A = 0, R = 0, C = 0;
  const int32_t* arc_src = nullptr;
  const uint32_t* arc_meta = nullptr;
  const int32_t* arc_tail = nullptr;
  const int32_t* run_head = nullptr;
  const int32_t* run_ts = nullptr;
  const int32_t* vtx_run_off = nullptr;
  const int64_t* chunk_arc = nullptr;
  const int32_t* chunk_run = nullptr;
  const uint8_t* chunk_carry = nullptr;
  const int32_t* carry_list = nullptr;
  int32_t ncarry = 0;
  // State slots: S_l of run r is read at level l+1 only through some arc's
  // src, so only such runs get S_l, stored at row run_slot[r] (their rank in
  // run order; -1 = never read).  arc_src holds SLOTS, not run indices.
  const int32_t* run_slot = nullptr;
  int64_t S = 0;  // state rows = referenced runs
};

// One sieve-point batch [pb, pe) of W = lanes * ppt consecutive points.
struct Batch {
  uint64_t pb = 0, pe = 0;
  int lanes = 32, ppt = 1;
#ifdef __CUDACC__
  __host__ __device__
#endif
  int W() const { return lanes * ppt; }
};

struct LevelParams {
  DevGraph g;
  const uint64_t* zj = nullptr;  // n x k
  const uint64_t* zb = nullptr;  // n x W: z_u^A of the batch (wide kernel, optional)
  int k = 0;
  int ell = 2;                   // level being produced
  uint64_t seed = 1;
  int32_t anchor_source = -1;
  Batch b;
  const uint64_t* s_prev = nullptr;  // S x W (level ell-1), unused at ell=2
  uint64_t* s_cur = nullptr;         // S x W (level ell)
  uint64_t* agg = nullptr;           // C x W chunk tail aggregates
  // y-multiply path of the wide kernel: 0 = smem tables (default), 1 = holes
  // general product.  Set from TSV_YMUL=holes for measurements.
  int ymul = 0;
  // Level k fused with the readout (wide kernel only): no S_k is stored;
  // acc[u] ^= XOR_w z_u * (XOR of u's arc products with ts <= max_ts).
  bool last = false;
  int32_t max_ts = 0;
  uint64_t* acc = nullptr;
  // Vertex-ordered sieve (vc_impl, sieve.cpp:540-635): an arc is live at
  // this level only when its tail has color vc_tail and its head vc_head
  // (has_color: primary color, or any color when it is the wildcard).
  const int32_t* vc_color = nullptr;  // n primary colors, nullptr = not VC
  int32_t vc_head = 0, vc_tail = 0, vc_wild = -1;
};

// One level of a static-projection engine (static_kernels.cu).
struct StaticLevel {
  int64_t C = 0;                      // chunks
  const int64_t* chunk_arc = nullptr; // C+1
  const int32_t* arc_head = nullptr;  // head-sorted arcs
  const int32_t* arc_tail = nullptr;
  const int32_t* arc_edge = nullptr;  // static edge id
  const uint64_t* zj = nullptr;
  int k = 0;
  uint64_t seed = 1;
  uint64_t role = 3;                  // edge_y (ending) or edge_y2 (starting)
  int level = 1;                      // second draw index
  bool tail_times_z = false;          // walks-starting family
  bool head_times_z = false;          // walks-ending family
  const uint64_t* src = nullptr;      // n x W, nullptr = all-ones layer
  uint64_t* out = nullptr;            // n x W, zeroed, XOR-accumulated
  uint64_t pb = 0, pe = 0;
  int ppt = 1;                        // W = 32 * ppt
  int bits = 64;                      // field width (small_field.cuh for 8/16/32)
};

void launch_static_level(const StaticLevel& p, cudaStream_t st);
void launch_static_base(int32_t n, const uint64_t* zj, int k, uint64_t pb, uint64_t pe, int ppt,
                        uint64_t* out, cudaStream_t st);
void launch_static_readout(int32_t n, const uint64_t* a, const uint64_t* b, int ppt,
                           uint64_t* acc, cudaStream_t st, int bits = 64);

// ---- on-device graph build (build_kernels.cu) ------------------------------

struct BuildStatus {
  long long first_bad_endpoint;  // smallest input index with an endpoint out of range
  long long first_bad_ts;        // smallest input index with ts < 1
  long long self_loops;
  int max_ts;
  int not_canonical;
};

struct DeviceLayout {
  int64_t m = 0, A = 0, R = 0, C = 0;
  int32_t ncarry = 0;
  int64_t dropped_duplicates = 0;
  int32_t *eu = nullptr, *ev = nullptr, *ets = nullptr;  // canonical edges
  int32_t* arc_src = nullptr;
  uint32_t* arc_meta = nullptr;
  int32_t* arc_tail = nullptr;
  int32_t *run_head = nullptr, *run_ts = nullptr, *vtx_run_off = nullptr;
  int64_t* chunk_arc = nullptr;
  int32_t* chunk_run = nullptr;
  uint8_t* chunk_carry = nullptr;
  int32_t* carry_list = nullptr;
};

// Builds the layout of layout.hpp on the device from device edge arrays.
// canonical = the input is already canonical (validated, not re-sorted).
// alloc/release manage device memory (stream-ordered); buffers still live at
// return belong to `out`.  Errors are reported through *d_status.
// d_eps (m, canonical input only) / d_delay (n): transition times and vertex
// delays of a non-instant edge model, or nullptr.
void device_build(const int32_t* d_u, const int32_t* d_v, const int32_t* d_ts, int64_t m,
                  int32_t n, bool directed, bool canonical, DeviceLayout& out,
                  BuildStatus* d_status, int sm_count, cudaStream_t st,
                  const std::function<void*(size_t)>& alloc,
                  const std::function<void(void*)>& release, const int32_t* d_eps = nullptr,
                  const int32_t* d_delay = nullptr);

// Order-preserving filter of a canonical edge list (restrict_to): keeps
// edges with ts <= max_ts and both endpoints kept; returns the kept count.
// oid (optional): the kept edges' indices in the input list.
int64_t device_restrict(const int32_t* eu, const int32_t* ev, const int32_t* ets, int64_t m,
                        const uint8_t* d_keep, int32_t max_ts, int32_t* ou, int32_t* ov,
                        int32_t* ots, cudaStream_t st,
                        const std::function<void*(size_t)>& alloc,
                        const std::function<void(void*)>& release, int32_t* oid = nullptr);
// keep[u] = vertex u has at least one shade (shade CSR offsets, device)
void launch_shaded_mask(int32_t n, const int32_t* off, uint8_t* keep, cudaStream_t st);
// arc_meta edge ids of a layout built from a filtered list -> the ids of the
// unfiltered list (oid[filtered id])
void launch_remap_edge_ids(int64_t A, uint32_t* meta, const int32_t* oid, cudaStream_t st);

// Kernel launchers (kernels.cu).  All are asynchronous on `st`.
// w_{d,j} table (k x k) of the constrained substitution, on the device
void launch_wtab(int k, uint64_t seed, uint64_t* wtab, cudaStream_t st);
void launch_zj(int32_t n, int k, uint64_t seed, const int32_t* vertex_off,
               const int32_t* vertex_shades, const uint64_t* wtab, uint64_t* zj,
               cudaStream_t st);
void launch_level(const LevelParams& p, cudaStream_t st);
void launch_fixup(const LevelParams& p, cudaStream_t st);
void launch_zbatch(int32_t n, const uint64_t* zj, int k, const Batch& b, uint64_t* zb,
                   cudaStream_t st);
void launch_k1(int32_t n, const uint64_t* zj, Batch b, int32_t anchor_source,
               uint64_t* acc, cudaStream_t st, const int32_t* colors = nullptr,
               int32_t color = -1, int32_t wild = -1);
// positional z_{u,j} = draw(seed, label_z, u, j+1) (build_zj_positional, sieve.cpp:103-113)
// launch_zj with w = identity (the coefficient engine's shade basis)
// the shade CSR of a table where every vertex has the same list `pattern` (c entries)
void launch_uniform_csr(int32_t n, int c, const int32_t* pattern, int32_t* off, int32_t* shades,
                        cudaStream_t st);
void launch_zj_ident(int32_t n, int k, uint64_t seed, const int32_t* vertex_off,
                     const int32_t* vertex_shades, uint64_t* zj, cudaStream_t st);
void launch_zj_positional(int32_t n, int k, uint64_t seed, uint64_t* zj, cudaStream_t st);
// Edge-constrained level (ec_impl, sieve.cpp:477-536): the arcs of edges
// [e0, e1) (one timestamp) add z_head * y(e, l-1) * prev[tail] into cur[head]
// (n x W rows, W = 32*ppt; prev of level 1 = the batch z table).
void launch_ec_level(int64_t e0, int64_t e1, int directed, const int32_t* eu,
                     const int32_t* ev, const uint64_t* zb, int W, uint64_t seed, int ell,
                     const uint64_t* prev, uint64_t* cur, cudaStream_t st);
// acc[u] ^= XOR_w rows[u][w]
void launch_row_xor(int32_t n, int W, const uint64_t* rows, uint64_t* acc, cudaStream_t st);
// VC-ColorfulPath exact DP (dp_probe, solver.cpp:146-191) in earliest-arrival
// form: e_next[head] = min(ts + 1) over edges ts <= max_ts whose tail/head
// colors match the order step and with e_prev[tail] <= ts.
void launch_vc_dp_level(int64_t m, int directed, const int32_t* eu, const int32_t* ev,
                        const int32_t* ets, int32_t max_ts, const int32_t* colors,
                        int32_t tail_color, int32_t head_color, int32_t wild,
                        const int32_t* e_prev, int32_t* e_next, cudaStream_t st);
// Canonical edges (edge id order) rebuilt from an instant-model layout: the
// arc carrying edge id e knows its tail, its run's head and timestamp
// (build_kernels.cu).  Outputs are device arrays of m entries.
void edges_from_layout(const DevGraph& g, bool directed, int32_t* eu, int32_t* ev, int32_t* ets,
                       cudaStream_t st);

// Static projection of canonical edges (graph.cpp:148-199): writes the ms
// distinct (a, b) pairs ascending (a < b when undirected) to a, b, the first
// index of each into off (ms + 1 entries, off[ms] = m) and the temporal
// edge ids grouped by pair, increasing within a pair, into back (m).  All
// device arrays; returns ms (synchronizes st).
int64_t static_projection(const int32_t* u, const int32_t* v, int64_t m, int32_t n, bool directed,
                          int32_t* a, int32_t* b, int32_t* off, int32_t* back, cudaStream_t st,
                          const std::function<void*(size_t)>& alloc,
                          const std::function<void(void*)>& release);

// State slots (build_kernels.cu): run_slot[r] = rank of r among the runs
// some arc reads (else -1) and arc_src rewritten from run indices to slots.
// Returns {arcs with a src, referenced runs}; synchronizes `st`.
// vtx_run_off (n+1, optional): also give every vertex's last run a slot
// (time windows of the coefficient engine read each vertex's final state).
struct SlotCounts {
  int64_t arcs_with_src = 0, slots = 0;
};
SlotCounts build_run_slots(int64_t A, int64_t R, int32_t* arc_src, int32_t* run_slot,
                           cudaStream_t st, const int32_t* vtx_run_off = nullptr,
                           int32_t n = 0);
void launch_xor_combine(const uint64_t* parts, int nparts, int64_t n,
                        uint64_t* out, cudaStream_t st);
void launch_gf_mul(int variant, int64_t n, const uint64_t* a, const uint64_t* b,
                   uint64_t* out, cudaStream_t st);
double launch_gf_bench(int variant, int64_t iters, uint64_t* sink, int blocks,
                       int threads, cudaStream_t st);
void launch_draw_y(uint64_t seed, int32_t level, int64_t n, const int32_t* edges,
                   uint64_t* out, cudaStream_t st);

// Profiling hooks (tsv_abi.cu).
// finalize (sieve.cpp:136-159) of device accumulators (finalize.cu): zeroes
// all but the sink when sink >= 0; flagged count and FNV-1a checksum.
// Synchronizes `st`.
void device_finalize(uint64_t* d_acc, int64_t n, int64_t sink, cudaStream_t st,
                     uint64_t* checksum, int64_t* flagged);

// Temporal sieve over GF(2^8 / 2^16 / 2^32) (small_field.cu): points
// [pb, pe) in batches of W, XORed (zero-extended) into acc; the vertex list
// (head, start, count, nv) is build_vertex_list's.
struct SmallFieldArgs {
  int bits = 32;
  DevGraph g;
  const int32_t* head = nullptr;
  const int64_t* start = nullptr;
  const int32_t* count = nullptr;
  int64_t nv = 0;
  const int32_t* off = nullptr;     // shade CSR (device)
  const int32_t* shades = nullptr;
  int k = 0;
  uint64_t seed = 1;
  int32_t anchor = -1;
  int32_t max_ts = 0;
  uint64_t pb = 0, pe = 0;
  int W = 1;
  uint64_t* acc = nullptr;
  std::function<void*(size_t)> alloc;
  std::function<void(void*)> release;
};
void launch_small_field(const SmallFieldArgs& a, cudaStream_t st);
// n x k shade table z_{u,j} over GF(2^bits), bits 8/16/32, zero-extended
void launch_small_zj64(int bits, int32_t n, int k, uint64_t seed, const int32_t* off,
                       const int32_t* shades, uint64_t* zj, cudaStream_t st);

void prof_begin(const char* name, cudaStream_t st);
void prof_end(cudaStream_t st);

}  // namespace tsv

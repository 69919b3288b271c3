// coef.hpp -- the coefficient (top-degree) form of the temporal sieve
// (coef_kernels.cu; the derivation is at the top of that file).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <functional>
#include <vector>

#include "engine.hpp"

namespace tsv {

// One level l of the coefficient engine (kernel k_coef_arcs).
struct CoefParams {
  DevGraph g;
  const uint64_t* zj = nullptr;  // n x k: S_1 rows (v_{u,d} in the shade basis)
  int k = 0;
  int ell = 2;                   // level being produced
  bool last = false;             // ell == k: flush vertex pieces into ulast
  uint64_t seed = 1;
  int32_t anchor_source = -1;
  int E = 0;                     // input entries C(k, ell-1)
  int e0 = 0, ne = 0;            // entry slice of this launch
  const uint64_t* s_prev = nullptr;  // S rows of level ell-1 (ell > 2), stride rs_in
  uint64_t* ubuf = nullptr;          // S rows of level ell, stride rs_out (see below)
  int rs_in = 0, rs_out = 0;
  uint64_t* agg = nullptr;           // C x E: chunk tail prefixes
  uint64_t* ulast = nullptr;         // n x k: level-k vertex sums (zeroed)
  int32_t max_ts = 0;
  // some arc may land past max_ts (a binary-search probe below t, or an edge
  // model with transition times): the vertex-lane engine then stops a
  // vertex at its first arc past the horizon at every level (false: no arc
  // is past it, no timestamp is read)
  bool below_t = true;
  // per vertex: -1 no shade (S = 0), d = its only shade, -2 several
  // (nullptr: no zero skipping, no single-shade form)
  const int8_t* vsh = nullptr;
  const uint64_t* vsv = nullptr;   // n: v_{u,d} of a single-shade vertex, else 1
  const uint8_t* sflag = nullptr;  // S: row of level ell-1 is nonzero (ell > 2)
  uint8_t* sflag_out = nullptr;    // S: row of level ell is nonzero (cleared)
  // A single-shade vertex's rows keep U_l (the S_l entries are
  // S_l[T] = v_h * U_l[T - {d}] for T containing its shade d, else 0; v_h
  // rides on the next arc's y): for a source with shade d the level-ell arcs
  // read entry e (an (ell-1)-subset) at smap[d * E + e] of its U row (-1: zero).
  const int32_t* smap = nullptr;
  // item-stream kernel (coef_items.cu): compact frames, per (tail class,
  // head class) item lists of (input index, output index); class = the
  // vertex's shade, or k for several shades
  const int2* items = nullptr;
  const int32_t* item_off = nullptr;  // (k+1) x (k+1)
  const int32_t* item_cnt = nullptr;
  const uint64_t* item_omask = nullptr;  // (k+1) x (k+1): outputs < 64 an item list reaches
  int32_t* chunk_ctr = nullptr;  // zeroed: persistent warps take chunks from it (nullptr: one per warp)
  int sms = 148;
  int frame_single = 0;  // C(k-1, ell-1) (0: full frames everywhere)
  int frame_multi = 0;   // C(k, ell-1)
  int frame_max = 0;     // accumulator words (frame_multi, or frame_single without multi-shade vertices)
  int warp_words = 0;    // shared words per warp (table + frame accumulator)
  const int32_t* vc_color = nullptr;  // vertex-ordered sieve filter (as LevelParams)
  int32_t vc_head = 0, vc_tail = 0, vc_wild = -1;
  // time windows (coef_window.cu, item-stream kernels): a vertex's prefix
  // starts from its carried U row (carry_in[h * carry_cs], when carry_nz[h])
  // instead of zero, so every window row already holds the carry
  const uint64_t* carry_in = nullptr;
  const uint8_t* carry_nz = nullptr;
  int carry_cs = 0;
};

// Lanes per arc group for an entry slice of ne entries (4, 8, 16 or 32).
int coef_group_lanes(int ne);
// Entries one k_coef_arcs launch covers at most (larger levels are sliced).
constexpr int kCoefSlice = 128;

void launch_coef_arcs(const CoefParams& p, cudaStream_t st);
void launch_coef_fixup(const CoefParams& p, cudaStream_t st);
void launch_coef_items(const CoefParams& p, cudaStream_t st);
// Item lists of level l (2..k) for CoefParams::items: per (tail class tc,
// head class hc), tc/hc = shade d or k (several shades).
struct CoefItems {
  std::vector<int2> items;
  std::vector<int32_t> off, cnt;  // (k+1) x (k+1)
};
CoefItems coef_items(int k, int l);
// Multi-shade heads: S_l[slot] from the U row stored at the same place
// (in place, row stride rs).  F = C(k, l) <= kZAcc.
void launch_coef_ztrans(int64_t S, int F, int l, const int32_t* slot_head, const uint64_t* zj,
                        int k, int E, uint64_t* rows, int rs, const int2* jpairs,
                        const int8_t* vsh, uint8_t* sflag, int sm_count, cudaStream_t st);
// Direct form (k_coef_ztrans_direct): one thread per (listed row, T),
// general products, over the (slot, head) list of k_multi_slots.
void launch_multi_slots(int64_t R, const int32_t* run_slot, const int32_t* run_head,
                        const int8_t* vsh, int2* list, int32_t* count, cudaStream_t st);
void launch_coef_ztrans_direct(int64_t S, int F, int l, const int2* list, const int32_t* count,
                               const uint64_t* zj, int k, uint64_t* rows, int rs,
                               const int2* pairs, const uint8_t* sflag, int sm_count,
                               int64_t rows_hint, cudaStream_t st);
constexpr int kZAcc = 1024;  // largest F the in-place z map handles (k <= 12)
// vsh / vsv of the rows of the n x k shade table (CoefParams)
void launch_vshade(int32_t n, int k, const uint64_t* rows, int8_t* vsh, uint64_t* vsv,
                   cudaStream_t st);
// vsh / vsv non-null: single-shade vertices hold their one compact level-k
// entry in ulast[h * k] (item-stream kernel)
void launch_coef_readout(int32_t n, const uint64_t* zj, int k, const uint64_t* ulast,
                         const int2* pairs, uint64_t scale, const int8_t* vsh,
                         const uint64_t* vsv, uint64_t* acc, cudaStream_t st);
void launch_slot_head(int64_t R, const int32_t* run_slot, const int32_t* run_head,
                      int32_t* slot_head, cudaStream_t st);

// Vertex-lane form of the coefficient engine (coef_vertex.cu): every vertex
// multi-shade, k <= kVertexMaxK.  Work list = the vertices with arcs sorted
// by arc count (descending), built once per graph.
constexpr int kVertexMaxK = 5;
struct VertList {
  int64_t nv = 0;
  int32_t* head = nullptr;   // vertex
  int64_t* start = nullptr;  // its first arc (vertex-major arc order)
  int32_t* count = nullptr;  // its arcs
};
bool vertex_engine_supports(int k);
// row stride (words) of the vertex-lane engine's level-l state rows
int vertex_row_words(int k, int l);
// The list of the vertices in [v_lo, v_hi) (v_hi < 0: all).
void build_vertex_list(const DevGraph& g, VertList& out, cudaStream_t st,
                       const std::function<void*(size_t)>& alloc,
                       const std::function<void(void*)>& release, int32_t v_lo = 0,
                       int32_t v_hi = -1);
// Targeted row exchange of the vertex-partitioned engine: the state slots
// this rank sends to / receives from every peer (rows some arc of the
// receiving rank reads), peers in rank order; fixed per graph (the arcs
// reading a slot are the same at every level).
struct ExchangeLists {
  std::vector<int64_t> send_count, recv_count;  // rows per peer
  int64_t send_total = 0, recv_total = 0;
  int32_t* send_slots = nullptr;  // device, send_total
  int32_t* recv_slots = nullptr;  // device, recv_total
  // one byte per state slot (packed four to a word): bit q = an arc whose
  // head rank q owns reads the slot (kept for the peer-store level kernel)
  const unsigned int* reader_mask = nullptr;
};
// Peer-store form of a level (coef_vertex.cu): every row is also stored
// into the level buffer of each OTHER rank whose bit is set in its reader
// byte -- peer[q] is rank q's buffer as mapped on this device (NVLink peer
// memory) -- so the row exchange rides inside the level kernel.
struct VertPeers {
  const unsigned int* reader_mask = nullptr;
  uint64_t* peer[8] = {};
  int rank = 0;
};
void build_exchange_lists(const DevGraph& g, const std::vector<const VertList*>& lists,
                          const std::vector<int64_t>& slot_lo, const std::vector<int64_t>& slot_hi,
                          int rank, ExchangeLists& out, cudaStream_t st,
                          const std::function<void*(size_t)>& alloc,
                          const std::function<void(void*)>& release);
// rows (F words) of `slots` <-> a packed buffer
void launch_rows_pack(const int32_t* slots, int64_t count, int F, const uint64_t* rows,
                      uint64_t* buf, cudaStream_t st);
void launch_rows_unpack(const int32_t* slots, int64_t count, int F, const uint64_t* buf,
                        uint64_t* rows, cudaStream_t st);
// State slots of the runs before run r (= the first slot of runs >= r).
int64_t count_slots_before(const DevGraph& g, int64_t r, cudaStream_t st,
                           const std::function<void*(size_t)>& alloc,
                           const std::function<void(void*)>& release);
// One level l of the vertex-lane engine: S_l rows (stride C(k, l)) at the
// referenced slots into p.ubuf from p.s_prev (stride C(k, l-1)) or zj (l = 2);
// at l = k the readout acc[h] ^= det * ... (no ulast).
void launch_coef_vertex(const CoefParams& p, const VertList& vl, uint64_t det, uint64_t* acc,
                        cudaStream_t st, const VertPeers* peers = nullptr);

// Time windows (coef_window.cu): arcs without a source in the window read
// the tail's carry slot base + tail; window edge ids -> the original graph's
// (oid[base + local], or base + local when oid is null).
void launch_win_src(int64_t A, int32_t* arc_src, const int32_t* arc_tail, int64_t base,
                    cudaStream_t st);
void launch_win_edge_ids(int64_t A, uint32_t* meta, const int32_t* oid, int64_t base,
                         cudaStream_t st);
// One level of one window, after the arc pass and the chunk fix-up, before
// the z map: carry slots from the carry (the state at the window start),
// then the carry from each vertex's last window row.
struct WinCarryArgs {
  const int32_t* run_slot = nullptr;
  const int32_t* vro = nullptr;  // window vtx_run_off (n+1)
  int32_t n = 0;
  int64_t Sw = 0;                // window slots (carry slots follow)
  const int8_t* vsh = nullptr;
  int frs = 0, frm = 0;          // U-row entries of single- / multi-shade vertices
  uint64_t* rows = nullptr;      // level rows, stride rs
  int rs = 0;
  uint8_t* sflag = nullptr;
  uint64_t* carry = nullptr;     // n x cs
  int cs = 0;
  uint8_t* cnz = nullptr;        // n: carry row nonzero
};
void launch_win_carry(const WinCarryArgs& a, cudaStream_t st);
void launch_win_multi_list(int32_t n, int64_t Sw, const int8_t* vsh, int2* list, int32_t* count,
                           cudaStream_t st);
void launch_ts_group_start(const int32_t* ts, const int64_t* pos, int nb, int64_t* out,
                           cudaStream_t st);

// Static-projection sieves in coefficient form (coef_static.cu): the
// junction sieve (junction = true) or the plain static sieve over the
// projection's head-grouped in-arcs (tail -> head) and out-arcs (head =
// the walk's current vertex, tail = the next one), both with per-head
// offsets (n + 1); zj = the n x k shade-basis table (k_zj_ident), det =
// det(W); XORs the accumulators into acc.
struct StaticCoefInputs {
  int32_t n = 0;
  int k = 0;
  bool junction = true;
  uint64_t seed = 1;
  const int64_t* in_off = nullptr;
  const int32_t* in_tail = nullptr;
  const int32_t* in_edge = nullptr;
  const int64_t* out_off = nullptr;
  const int32_t* out_tail = nullptr;
  const int32_t* out_edge = nullptr;
  const std::vector<int64_t>* h_in_off = nullptr;   // host copies of the offsets (tasks)
  const std::vector<int64_t>* h_out_off = nullptr;
  const uint64_t* zj = nullptr;
  uint64_t det = 1;
  uint64_t* acc = nullptr;
  const struct CoefTables* tables = nullptr;
};
bool static_coef_supported(int k);
uint64_t static_coef_words(int32_t n, int k, bool junction);  // device words it allocates
void eval_static_coef(const StaticCoefInputs& in, cudaStream_t st,
                      const std::function<void*(size_t)>& alloc,
                      const std::function<void(void*)>& release);

// Host tables (colex order = increasing bit mask within a level).
struct CoefTables {
  int k = 0;
  std::vector<int64_t> count;  // count[l] = C(k, l), l = 0..k
  // pairs of level l (2..k): for output o (an l-subset T) and c < l,
  // (rank of T minus its c-th element among the (l-1)-subsets, that element)
  std::vector<std::vector<int2>> pairs;
  // smap of level l: smap[d * C(k,l) + o] = rank of T_o - {d} among the
  // (l-1)-subsets, -1 if d is not in T_o
  std::vector<std::vector<int32_t>> smap;
  // jpairs of level l: for each j < k, the C(k-1, l-1) pairs (rank of an
  // (l-1)-subset T' without j, rank of T' + {j}) in increasing T' order
  std::vector<std::vector<int2>> jpairs;
};
CoefTables coef_tables(int k);

}  // namespace tsv

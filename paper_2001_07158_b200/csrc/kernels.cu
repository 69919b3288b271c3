// kernels.cu -- sm_100a kernels of the temporal sieve (instant edge model).
//
// The reference evaluates Eq. 3 time-major over dense n*W*(t+1) layers
// (/root/reference/proj/core/src/sieve.cpp:170-307).  Here each level l is
// ONE pass over the vertex-major arc stream (layout.hpp):
//
//   prod_a   = y(e_a, l-1) * S_{l-1}[src_a]            (gather, GF multiply)
//   U_a      = XOR of prod over the head's arcs up to a  (segmented scan)
//   S_l[run] = z_head^A * U_{last arc of run}           (at run ends)
//
// S_l[run] is P[l][head][ts(run)] of the reference: its stay term
// (sieve.cpp:229-230) is the prefix over the head's earlier runs, and the
// z_u multiply of sieve.cpp:255 commutes with that prefix because z_u is
// constant along u's runs.  A warp owns one chunk of arcs; G = 32/LANES
// arcs are in flight per step, each processed by LANES threads that hold
// PPT sieve points apiece (W = LANES*PPT points per batch, contiguous in
// HBM so every state gather/store is one coalesced W*8-byte segment).
// Arc metadata and the y draws of 32 arcs are produced cooperatively (one
// arc per thread) and staged in shared memory, so each draw costs one
// thread, not W.
#include <cuda_runtime.h>

#include "engine.hpp"
#include "gf_device.cuh"
#include "layout.hpp"

namespace tsv {
namespace {

constexpr int kWarpsPerBlock = 8;
constexpr int kWideWarps = 4;  // wide kernel: 4 warps per block (shared tables)
constexpr unsigned kFull = 0xffffffffu;
// staged per-arc flags of the wide kernel (kVStart / kRunEnd kept from meta)
constexpr uint32_t kRef = 1u;   // run end whose S_l is read at level l+1
constexpr uint32_t kLive = 2u;  // the arc's product can be nonzero

template <int PPT>
__device__ __forceinline__ void z_of(const uint64_t* __restrict__ zj, int k,
                                     int32_t u, const uint32_t (&pt)[PPT],
                                     const bool (&pv)[PPT],
                                     uint64_t (&z)[PPT]) {
#pragma unroll
  for (int p = 0; p < PPT; ++p) z[p] = 0;
  const uint64_t* row = zj + static_cast<int64_t>(u) * k;
  for (int j = 0; j < k; ++j) {
    const uint64_t r = __ldg(row + j);
#pragma unroll
    for (int p = 0; p < PPT; ++p)
      if ((pt[p] >> j) & 1u) z[p] ^= r;
  }
#pragma unroll
  for (int p = 0; p < PPT; ++p)
    if (!pv[p]) z[p] = 0;
}

// has_color of the reference (graph.hpp:129-131) on the device
__device__ __forceinline__ bool has_color(const int32_t* __restrict__ colors, int32_t x,
                                          int32_t c, int32_t wild) {
  return c == wild || __ldg(colors + x) == c;
}

__device__ __forceinline__ uint64_t z_single(const uint64_t* __restrict__ zj,
                                             int k, int32_t u, uint64_t A) {
  uint64_t z = 0;
  const uint64_t* row = zj + static_cast<int64_t>(u) * k;
  for (int j = 0; j < k; ++j)
    if ((A >> j) & 1ull) z ^= __ldg(row + j);
  return z;
}

// Grouped variant (W = LANES < 32 points per batch): G = 32/LANES arcs are
// in flight per warp step, one per group of LANES lanes (one point per lane);
// y is split once per arc into shared memory and each group multiplies its
// gathered states by its own arc's y (general product).  The per-vertex
// prefix is a segmented XOR-scan across the groups (shuffles) plus a carry
// across steps.  The z_head products at run ends are where the groups
// diverge, so they go through a per-warp work queue: a group whose arc ends a
// run that is needed (kPush) enqueues (run, head, prefix) and whenever G
// entries are pending every group pops one, so each round of general
// products runs with all 32 lanes busy.  Level k (LAST) enqueues one entry per
// vertex piece (its last arc within max_ts) and the pop XORs the group's
// z_head * prefix into acc[head] (fused readout, like flush_vertex).
// Window w of a GfTable (the 16 multiples c * x^(4w) * y) written by one
// lane: 16 lanes build a whole table (the half-warp variant of
// GfTable::build).  With the 136-byte window stride the 16 lanes' stores of
// one entry hit 16 distinct bank pairs.
__device__ __forceinline__ void build_window16(uint64_t* tab, uint64_t y, int w) {
  const uint32_t s = 4u * static_cast<uint32_t>(w);
  uint64_t h, lo;
  asm("shr.b64 %0, %1, %2;" : "=l"(h) : "l"(y), "r"(64u - s));  // 0 when s == 0
  asm("shl.b64 %0, %1, %2;" : "=l"(lo) : "l"(y), "r"(s));
  const uint64_t B0 = lo ^ h ^ (h << 1) ^ (h << 3) ^ (h << 4);
  const uint64_t B1 = gf_mulx(B0), B2 = gf_mulx(B1), B3 = gf_mulx(B2);
  const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(tab)) +
                     GfTable::kWinBytes * static_cast<uint32_t>(w);
  const uint64_t v3 = B1 ^ B0, v5 = B2 ^ B0, v6 = B2 ^ B1, v7 = v6 ^ B0;
  GfTable::sts<0>(a, 0ull);
  GfTable::sts<8>(a, B0);
  GfTable::sts<16>(a, B1);
  GfTable::sts<24>(a, v3);
  GfTable::sts<32>(a, B2);
  GfTable::sts<40>(a, v5);
  GfTable::sts<48>(a, v6);
  GfTable::sts<56>(a, v7);
  GfTable::sts<64>(a, B3);
  GfTable::sts<72>(a, B3 ^ B0);
  GfTable::sts<80>(a, B3 ^ B1);
  GfTable::sts<88>(a, B3 ^ v3);
  GfTable::sts<96>(a, B3 ^ B2);
  GfTable::sts<104>(a, B3 ^ v5);
  GfTable::sts<112>(a, B3 ^ v6);
  GfTable::sts<120>(a, B3 ^ v7);
}

template <int LANES, bool FIRST, bool LAST>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, 3)
    k_level(const LevelParams P) {
  constexpr int G = 32 / LANES;
  constexpr int W = LANES;
  constexpr uint32_t kPush = 4u;  // staged: enqueue this arc's prefix
  __shared__ uint32_t s_ys[kWarpsPerBlock][12][32];  // Karatsuba split of each arc's y
  __shared__ int32_t s_src[kWarpsPerBlock][32];
  __shared__ uint32_t s_meta[kWarpsPerBlock][32];
  __shared__ int32_t s_run[kWarpsPerBlock][32];
  __shared__ int32_t s_head[kWarpsPerBlock][32];
  __shared__ int32_t q_run[kWarpsPerBlock][2 * G];
  __shared__ int32_t q_head[kWarpsPerBlock][2 * G];
  __shared__ uint64_t q_val[kWarpsPerBlock][2 * G][LANES];
  // LANES == 16: each half-warp multiplies by its own arc's y through a
  // shared-memory table it builds (16 lanes x one window each) instead of
  // the general product
  constexpr bool kHalfTab = LANES == 16;
  __shared__ __align__(256) uint64_t s_gtab[kHalfTab ? kWarpsPerBlock : 1][kHalfTab ? 2 : 1]
                                           [GfTable::kWords];
  __shared__ uint64_t s_yraw[kHalfTab ? kWarpsPerBlock : 1][32];

  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t c = static_cast<int64_t>(blockIdx.x) * kWarpsPerBlock + wib;
  if (c >= P.g.C) return;  // warp-uniform
  const int g = lane / LANES, li = lane % LANES;

  const uint64_t A = P.b.pb + li;
  const bool pv = A < P.b.pe;
  const uint64_t pre = draw_prefix(P.seed, kRoleEdgeY);
  const uint64_t yb = static_cast<uint64_t>(P.ell - 1) + 0x165667b19e3779f9ull;
  const int64_t a0 = P.g.chunk_arc[c], a1 = P.g.chunk_arc[c + 1];
  int32_t run_ctr = P.g.chunk_run[c];
  const int last_lane = (G - 1) * LANES + li;
  uint64_t carry = 0;
  int qn = 0;  // pending queue entries (warp-uniform)

  // z_head^A for this lane's point
  auto zval = [&](int32_t h) -> uint64_t {
    if (P.zb) return __ldg(P.zb + static_cast<int64_t>(h) * W + li);
    return pv ? z_single(P.zj, P.k, h, A) : 0ull;
  };
  // group gi pops entry e (all lanes of the warp call this together)
  auto pop = [&](int e, bool on) {
    uint64_t prod = 0;
    int32_t h = -1;
    if (on) {
      h = q_head[wib][e];
      prod = gf_mul(zval(h), q_val[wib][e][li]);
    }
    if (LAST) {  // XOR over the group's points (converged shuffles), one atomic
      uint64_t r = prod;
#pragma unroll
      for (int d = LANES / 2; d >= 1; d >>= 1) r ^= __shfl_xor_sync(kFull, r, d, LANES);
      if (on && li == 0 && r)
        atomicXor(reinterpret_cast<unsigned long long*>(P.acc + h),
                  static_cast<unsigned long long>(r));
    } else if (on) {
      P.s_cur[static_cast<int64_t>(q_run[wib][e]) * W + li] = prod;
    }
  };

  for (int64_t base = a0; base < a1; base += 32) {
    const int nb = static_cast<int>(a1 - base < 32 ? a1 - base : 32);
    uint32_t meta = 0;
    int32_t sidx = -1, head = -1;
    uint64_t y = 0;
    if (lane < nb) {
      meta = __ldg(P.g.arc_meta + base + lane);
      sidx = FIRST ? __ldg(P.g.arc_tail + base + lane) : __ldg(P.g.arc_src + base + lane);
      y = draw_edge_y(pre, yb, meta & kEdgeMask);
    }
    const unsigned ends = __ballot_sync(kFull, lane < nb && (meta & kRunEnd));
    const int32_t myrun = run_ctr + __popc(ends & ((1u << lane) - 1u));
    if (lane < nb) head = __ldg(P.g.run_head + myrun);
    if (kHalfTab) {
      s_yraw[kHalfTab ? wib : 0][lane] = y;
    } else {
      const KSplit ks = ksplit(y);  // once per arc, not once per lane of its group
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        s_ys[wib][j][lane] = ks.l.c[j];
        s_ys[wib][4 + j][lane] = ks.h.c[j];
        s_ys[wib][8 + j][lane] = ks.m.c[j];
      }
    }
    bool live = lane < nb && sidx >= 0;
    if (FIRST) live = live && (P.anchor_source < 0 || sidx == P.anchor_source);
    if (P.vc_color && live) {
      const int32_t tl = FIRST ? sidx : __ldg(P.g.arc_tail + base + lane);
      live = tl >= 0 && has_color(P.vc_color, tl, P.vc_tail, P.vc_wild) &&
             has_color(P.vc_color, head, P.vc_head, P.vc_wild);
    }
    bool push;
    int32_t slot = -1;
    if (LAST) {
      // last arc of its vertex (within this chunk) with ts <= max_ts
      const int32_t myts = lane < nb ? __ldg(P.g.run_ts + myrun) : 0;
      const bool chunk_end = base + lane + 1 >= a1;
      uint32_t nmeta = __shfl_down_sync(kFull, meta, 1);
      int32_t nts = __shfl_down_sync(kFull, myts, 1);
      if (lane == 31 && !chunk_end) {
        nmeta = __ldg(P.g.arc_meta + base + 32);
        nts = __ldg(P.g.run_ts + myrun + ((meta & kRunEnd) ? 1 : 0));
      }
      live = live && myts <= P.max_ts;
      push = lane < nb && myts <= P.max_ts && (chunk_end || (nmeta & kVStart) || nts > P.max_ts);
    } else {
      slot = (lane < nb && (meta & kRunEnd)) ? __ldg(P.g.run_slot + myrun) : -1;
      push = slot >= 0;
    }
    s_src[wib][lane] = sidx;
    s_meta[wib][lane] = (meta & (kVStart | kRunEnd)) | (live ? kLive : 0u) | (push ? kPush : 0u);
    s_run[wib][lane] = slot;
    s_head[wib][lane] = head;
    run_ctr += __popc(ends);
    __syncwarp();

    auto fetch = [&](int i, uint64_t& out) {
      out = 0;
      if (i < nb && (s_meta[wib][i] & kLive)) {
        const int32_t src = s_src[wib][i];
        if (FIRST) {
          out = zval(src);
        } else {
          out = __ldg(P.s_prev + static_cast<int64_t>(src) * W + li);
        }
      }
    };
    uint64_t nxt;
    fetch(g, nxt);
    const int steps = (nb + G - 1) / G;
#pragma unroll 1
    for (int s = 0; s < steps; ++s) {
      const uint64_t val = nxt;
      if (s + 1 < steps) fetch((s + 1) * G + g, nxt);
      const int i = s * G + g;
      const bool act = i < nb;
      const uint32_t mt = act ? s_meta[wib][i] : 0u;
      uint64_t v = 0;
      if (__any_sync(kFull, mt & kLive)) {
        const int ia = act ? i : 0;
        if (kHalfTab) {
          uint64_t* tab = s_gtab[kHalfTab ? wib : 0][kHalfTab ? g : 0];
          __syncwarp();
          build_window16(tab, s_yraw[kHalfTab ? wib : 0][ia], li);
          __syncwarp();
          v = (mt & kLive) ? GfTable{tab}.mul(val) : 0ull;
        } else {
          KSplit ys;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            ys.l.c[j] = s_ys[wib][j][ia];
            ys.h.c[j] = s_ys[wib][4 + j][ia];
            ys.m.c[j] = s_ys[wib][8 + j][ia];
          }
          v = (mt & kLive) ? gf_mul_presplit(ys, val) : 0ull;
        }
      }
      // segmented inclusive XOR-scan over the G groups (vertex starts cut it)
      bool f = (mt & kVStart) != 0;
      if (G > 1) {
#pragma unroll
        for (int d = 1; d < G; d <<= 1) {
          const bool fo = __shfl_up_sync(kFull, f, d * LANES);
          const uint64_t vo = __shfl_up_sync(kFull, v, d * LANES);
          if (g >= d && !f) v ^= vo;
          if (g >= d) f = f || fo;
        }
      }
      if (!f) v ^= carry;
      carry = (G > 1) ? __shfl_sync(kFull, v, last_lane) : v;
      // enqueue the needed prefixes, pop whenever a full round is pending
      const bool push = (mt & kPush) != 0;
      const unsigned pm = __ballot_sync(kFull, push && li == 0);
      if (pm) {
        if (push) {
          const int slot = qn + __popc(pm & ((1u << (g * LANES)) - 1u));
          q_val[wib][slot][li] = v;
          if (li == 0) {
            q_run[wib][slot] = s_run[wib][i];
            q_head[wib][slot] = s_head[wib][i];
          }
        }
        qn += __popc(pm);
        __syncwarp();
        if (qn >= G) {
          pop(qn - G + g, true);
          qn -= G;
        }
        __syncwarp();
      }
    }
    __syncwarp();
  }
  if (qn > 0) pop(g, g < qn);
  if (!LAST && g == 0) P.agg[c * W + li] = carry;
}

// The value multiplied by y(e, l-1) for one arc: the predecessor state
// S_{l-1}[src] (gather), or z_tail^A at level 2 (only from the anchor
// source in the (s,d) variant, sieve.cpp:241-242).
template <int PPT, bool FIRST>
__device__ __forceinline__ void fetch_src(const LevelParams& P, int32_t src,
                                          const uint32_t (&pt)[PPT], const bool (&pv)[PPT],
                                          uint64_t (&out)[PPT]) {
  const int lane = threadIdx.x & 31;
  if (FIRST) {
    if (src >= 0 && (P.anchor_source < 0 || src == P.anchor_source)) {
      if (P.zb) {  // batch z table materialized: one coalesced row per tail
#pragma unroll
        for (int p = 0; p < PPT; ++p)
          out[p] = __ldg(P.zb + static_cast<int64_t>(src) * (32 * PPT) + lane + 32 * p);
      } else {
        z_of<PPT>(P.zj, P.k, src, pt, pv, out);
      }
    } else {
#pragma unroll
      for (int p = 0; p < PPT; ++p) out[p] = 0;
    }
  } else {
#pragma unroll
    for (int p = 0; p < PPT; ++p)
      out[p] = src >= 0 ? __ldg(P.s_prev + static_cast<int64_t>(src) * (32 * PPT) + lane + 32 * p)
                        : 0ull;
  }
}

// Level k fused with the readout: the XOR over the batch's points of
// z_h^A * V, V = h's arc products with ts <= max_ts seen by this warp.  The
// map V -> z*V is linear, so a vertex split across chunks simply contributes
// once per piece (no fix-up), and only one general product per vertex piece
// is needed instead of one per run.
template <int PPT>
__device__ __forceinline__ void flush_vertex(const LevelParams& P, int32_t h,
                                             const uint32_t (&pt)[PPT], const bool (&pv)[PPT],
                                             const uint64_t (&V)[PPT]) {
  const int lane = threadIdx.x & 31;
  uint64_t z[PPT];
  if (P.zb) {
#pragma unroll
    for (int p = 0; p < PPT; ++p)
      z[p] = __ldg(P.zb + static_cast<int64_t>(h) * (32 * PPT) + lane + 32 * p);
  } else {
    z_of<PPT>(P.zj, P.k, h, pt, pv, z);
  }
  uint64_t r = 0;
#pragma unroll
  for (int p = 0; p < PPT; ++p) r ^= gf_mul(z[p], V[p]);
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) r ^= __shfl_xor_sync(kFull, r, d);
  if (lane == 0 && r) atomicXor(reinterpret_cast<unsigned long long*>(P.acc + h),
                                static_cast<unsigned long long>(r));
}

// Wide variant (W = 32*PPT >= 32): one arc per step for the whole warp, so
// y is warp-uniform and its product with the gathered states goes through
// the shared-memory multiple tables (GfTable) when YTAB; z_head^A is cached
// across the consecutive runs of one head.  LAST = level k fused with the
// readout (flush_vertex).
template <int PPT, bool FIRST, bool YTAB, bool LAST>
// Resident blocks per SM (register cap 65536 / (128 * minB)), measured per
// batch shape: PPT 1 -> 6 (80 regs), PPT 2 -> 5 (96 regs), PPT 4 -> 4.
#ifndef TSV_WIDE_MINB
#define TSV_WIDE_MINB(PPT) ((PPT) >= 4 ? 4 : (PPT) == 2 ? 5 : 6)
#endif
__global__ void __launch_bounds__(kWideWarps * 32, TSV_WIDE_MINB(PPT))
    k_level_wide(const LevelParams P) {
  constexpr int W = 32 * PPT;
  __shared__ uint64_t s_y[kWideWarps][32];
  __shared__ int32_t s_src[kWideWarps][32];
  __shared__ uint32_t s_meta[kWideWarps][32];
  __shared__ int32_t s_run[kWideWarps][32];  // state slot of the arc's run
  __shared__ int32_t s_head[kWideWarps][32];
  __shared__ __align__(256) uint64_t s_tab[YTAB ? kWideWarps : 1][GfTable::kWords];
  __shared__ uint32_t s_zs[LAST ? 1 : kWideWarps][PPT][12][32];  // split z_head^A per lane

  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t c = static_cast<int64_t>(blockIdx.x) * kWideWarps + wib;
  if (c >= P.g.C) return;  // warp-uniform

  uint32_t pt[PPT];
  bool pv[PPT];
#pragma unroll
  for (int p = 0; p < PPT; ++p) {
    const uint64_t A = P.b.pb + lane + 32 * p;
    pt[p] = static_cast<uint32_t>(A);
    pv[p] = A < P.b.pe;
  }
  GfTable T{s_tab[YTAB ? wib : 0]};
  const uint64_t pre = draw_prefix(P.seed, kRoleEdgeY);
  const uint64_t yb = static_cast<uint64_t>(P.ell - 1) + 0x165667b19e3779f9ull;
  const int64_t a0 = P.g.chunk_arc[c], a1 = P.g.chunk_arc[c + 1];
  int32_t run_ctr = P.g.chunk_run[c];
  uint64_t U[PPT], z[PPT];
#pragma unroll
  for (int p = 0; p < PPT; ++p) U[p] = z[p] = 0;
  int32_t zhead = -1;  // LAST: the vertex whose products U holds

  for (int64_t base = a0; base < a1; base += 32) {
    const int nb = static_cast<int>(a1 - base < 32 ? a1 - base : 32);
    uint32_t meta = 0;
    int32_t sidx = -1, head = -1;
    uint64_t y = 0;
    if (lane < nb) {
      meta = __ldg(P.g.arc_meta + base + lane);
      sidx = FIRST ? __ldg(P.g.arc_tail + base + lane) : __ldg(P.g.arc_src + base + lane);
      y = draw_edge_y(pre, yb, meta & kEdgeMask);
    }
    const unsigned ends = __ballot_sync(kFull, lane < nb && (meta & kRunEnd));
    const int32_t myrun = run_ctr + __popc(ends & ((1u << lane) - 1u));
    if (lane < nb) head = __ldg(P.g.run_head + myrun);
    s_y[wib][lane] = y;
    s_src[wib][lane] = sidx;
    // The edge id is consumed by the draw above; the staged meta keeps the
    // flags plus kRef = "this run's S is read by the next level" and kLive =
    // "this arc's product can be nonzero" (it has a predecessor state, comes
    // from the anchor source at level 2, and at level k lies within max_ts).
    const int32_t slot = (!LAST && lane < nb && (meta & kRunEnd)) ? __ldg(P.g.run_slot + myrun)
                                                                  : -1;
    const uint32_t ref = slot >= 0 ? kRef : 0u;
    bool live = lane < nb && sidx >= 0;
    if (FIRST) live = live && (P.anchor_source < 0 || sidx == P.anchor_source);
    if (LAST) live = live && __ldg(P.g.run_ts + myrun) <= P.max_ts;
    if (P.vc_color && live) {  // vertex-ordered sieve: per-level color filter
      const int32_t tl = FIRST ? sidx : __ldg(P.g.arc_tail + base + lane);
      live = tl >= 0 && has_color(P.vc_color, tl, P.vc_tail, P.vc_wild) &&
             has_color(P.vc_color, head, P.vc_head, P.vc_wild);
    }
    s_meta[wib][lane] = (meta & (kVStart | kRunEnd)) | ref | (live ? kLive : 0u);
    s_run[wib][lane] = slot;  // state row of this run's S (run ends only)
    s_head[wib][lane] = head;
    run_ctr += __popc(ends);
    __syncwarp();

    // One step per arc; the predecessor states of the next arc are in flight
    // while this one is multiplied (a step is thousands of cycles, so one
    // step of look-ahead covers the HBM latency).  The loop is deliberately
    // not unrolled: the step body is large and must stay in the I-cache.
    uint64_t nxt[PPT];
#pragma unroll
    for (int p = 0; p < PPT; ++p) nxt[p] = 0;
    if (s_meta[wib][0] & kLive) fetch_src<PPT, FIRST>(P, s_src[wib][0], pt, pv, nxt);
#pragma unroll 1
    for (int i = 0; i < nb; ++i) {
      uint64_t val[PPT];
#pragma unroll
      for (int p = 0; p < PPT; ++p) val[p] = nxt[p];
      if (i + 1 < nb && (s_meta[wib][i + 1] & kLive))
        fetch_src<PPT, FIRST>(P, s_src[wib][i + 1], pt, pv, nxt);
      {
        const uint32_t mt = s_meta[wib][i];
        if (LAST) {
          const int32_t h = s_head[wib][i];
          if (h != zhead) {  // vertex boundary (warp-uniform)
            if (zhead >= 0) flush_vertex<PPT>(P, zhead, pt, pv, U);
            zhead = h;
#pragma unroll
            for (int p = 0; p < PPT; ++p) U[p] = 0;
          }
        }
        if (mt & kLive) {  // warp-uniform: dead arcs contribute 0
          const uint64_t yy = s_y[wib][i];
          uint64_t prod[PPT];
          if (YTAB) {
            __syncwarp();
            T.build(yy, lane);
            __syncwarp();
#pragma unroll
            for (int p = 0; p < PPT; ++p) prod[p] = T.mul(val[p]);
          } else {
#pragma unroll
            for (int p = 0; p < PPT; ++p) prod[p] = gf_mul(yy, val[p]);
          }
          if (!LAST && (mt & kVStart)) {
#pragma unroll
            for (int p = 0; p < PPT; ++p) U[p] = prod[p];
          } else {
#pragma unroll
            for (int p = 0; p < PPT; ++p) U[p] ^= prod[p];
          }
        } else if (!LAST && (mt & kVStart)) {
#pragma unroll
          for (int p = 0; p < PPT; ++p) U[p] = 0;
        }
        if (!LAST && (mt & kRef)) {  // run end whose S is needed
          const int32_t h = s_head[wib][i];
          if (h != zhead) {  // new head: z_head^A and its Karatsuba split, cached
            if (P.zb) {
#pragma unroll
              for (int p = 0; p < PPT; ++p)
                z[p] = __ldg(P.zb + static_cast<int64_t>(h) * W + lane + 32 * p);
            } else {
              z_of<PPT>(P.zj, P.k, h, pt, pv, z);
            }
            zhead = h;
#pragma unroll
            for (int p = 0; p < PPT; ++p) {
              const KSplit ks = ksplit(z[p]);
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                s_zs[wib][p][j][lane] = ks.l.c[j];
                s_zs[wib][p][4 + j][lane] = ks.h.c[j];
                s_zs[wib][p][8 + j][lane] = ks.m.c[j];
              }
            }
          }
          const int64_t run = s_run[wib][i];
#pragma unroll
          for (int p = 0; p < PPT; ++p) {
            KSplit ks;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              ks.l.c[j] = s_zs[wib][p][j][lane];
              ks.h.c[j] = s_zs[wib][p][4 + j][lane];
              ks.m.c[j] = s_zs[wib][p][8 + j][lane];
            }
            P.s_cur[run * W + lane + 32 * p] = gf_mul_presplit(ks, U[p]);
          }
        }
      }
    }
    __syncwarp();
  }
  if (LAST) {
    if (zhead >= 0) flush_vertex<PPT>(P, zhead, pt, pv, U);
    return;
  }
#pragma unroll
  for (int p = 0; p < PPT; ++p) P.agg[c * W + lane + 32 * p] = U[p];
}

// A chunk whose first arc continues vertex h (split across chunk
// boundaries) computed h's prefix from zero; its runs of h receive the XOR
// of the tail aggregates of the preceding chunks back to the one where h
// starts, multiplied by z_h (the map U -> z*U is linear).
__global__ void k_fixup(const LevelParams P) {
  const int W = P.b.W();
  const int32_t c = P.g.carry_list[blockIdx.x];
  const int32_t r0 = P.g.chunk_run[c];  // run of the chunk's first arc
  if (r0 >= P.g.R) return;
  const int32_t head = P.g.run_head[r0];
  const int32_t r1 = min(P.g.chunk_run[c + 1], P.g.vtx_run_off[head + 1]);
  if (r0 >= r1) return;  // no run of h ends in this chunk
  for (int w = threadIdx.x; w < W; w += blockDim.x) {
    const uint64_t A = P.b.pb + static_cast<uint64_t>(w);
    if (A >= P.b.pe) continue;
    uint64_t carry = 0;
    for (int64_t cc = c - 1;; --cc) {
      carry ^= P.agg[cc * W + w];
      if (!P.g.chunk_carry[cc] || P.g.run_head[P.g.chunk_run[cc]] != head) break;
    }
    const uint64_t t = gf_mul(z_single(P.zj, P.k, head, A), carry);
    for (int32_t r = r0; r < r1; ++r) {
      const int32_t slot = P.g.run_slot[r];
      if (slot >= 0) P.s_cur[static_cast<int64_t>(slot) * W + w] ^= t;
    }
  }
}

// zb[u][w] = z_u^{pb+w} for one batch (a warp per vertex row, W = 32*ppt)
__global__ void k_zbatch(int32_t n, const uint64_t* __restrict__ zj, int k, Batch b,
                         uint64_t* __restrict__ zb) {
  const int64_t u = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (u >= n) return;
  const int lane = threadIdx.x & 31;
  const int W = b.W();
  for (int w = lane; w < W; w += 32) {
    const uint64_t A = b.pb + static_cast<uint64_t>(w);
    zb[u * W + w] = A < b.pe ? z_single(zj, k, static_cast<int32_t>(u), A) : 0ull;
  }
}

// k = 1: P_{u,1} = z_u^A, readout is the subset sum (sieve.cpp:203-213).
__global__ void k_k1(int32_t n, const uint64_t* __restrict__ zj, Batch b,
                     int32_t anchor_source, uint64_t* __restrict__ acc,
                     const int32_t* __restrict__ colors, int32_t color, int32_t wild) {
  const int64_t u = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (u >= n) return;
  if (anchor_source >= 0 && u != anchor_source) return;
  if (colors && !has_color(colors, static_cast<int32_t>(u), color, wild)) return;
  uint64_t x = 0;
  for (uint64_t A = b.pb; A < b.pe; ++A) x ^= z_single(zj, 1, static_cast<int32_t>(u), A);
  acc[u] ^= x;
}

// w_{d,j} = draw(seed, shade_w, d, j) for d, j in [1..k] (sieve.cpp:85-89),
// drawn on the device so no pageable host copy stalls the stream
__global__ void k_wtab(int k, uint64_t seed, uint64_t* __restrict__ wtab) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= k * k) return;
  const uint64_t pre = draw_prefix(seed, kRoleShadeW);
  wtab[i] = draw_nonzero_from(pre, static_cast<uint64_t>(i / k + 1),
                              static_cast<uint64_t>(i % k + 1), 0);
}

// z_{u,j} = XOR_{d in S(u)} v_{u,d} * w_{d,j}  (sieve.cpp:83-101)
__global__ void k_zj(int32_t n, int k, uint64_t seed,
                     const int32_t* __restrict__ vertex_off,
                     const int32_t* __restrict__ vertex_shades,
                     const uint64_t* __restrict__ wtab, uint64_t* __restrict__ zj) {
  const int64_t u = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (u >= n) return;
  const uint64_t pre = draw_prefix(seed, kRoleShadeV);
  uint64_t row[32];
  for (int j = 0; j < k; ++j) row[j] = 0;
  for (int32_t s = vertex_off[u]; s < vertex_off[u + 1]; ++s) {
    const int d = vertex_shades[s];
    const uint64_t v = draw_nonzero_from(pre, static_cast<uint64_t>(u),
                                         static_cast<uint64_t>(d), 0);
    for (int j = 0; j < k; ++j) row[j] ^= gf_mul(v, wtab[(d - 1) * k + j]);
  }
  for (int j = 0; j < k; ++j) zj[u * k + j] = row[j];
}

// The shade basis (coefficient engine): w = identity, so z_{u,d} = v_{u,d}
// for d in S(u) and 0 otherwise -- no products, no per-thread row array.
__global__ void k_zj_ident(int32_t n, int k, uint64_t seed,
                           const int32_t* __restrict__ vertex_off,
                           const int32_t* __restrict__ vertex_shades, uint64_t* __restrict__ zj) {
  const int64_t u = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (u >= n) return;
  const uint64_t pre = draw_prefix(seed, kRoleShadeV);
  const int32_t s0 = vertex_off[u], s1 = vertex_off[u + 1];
  uint32_t have = 0;
  for (int32_t s = s0; s < s1; ++s) have |= 1u << (vertex_shades[s] - 1);
  for (int j = 0; j < k; ++j)
    if (!((have >> j) & 1u)) zj[u * k + j] = 0;
  for (int32_t s = s0; s < s1; ++s) {
    const int d = vertex_shades[s];
    zj[u * k + d - 1] = draw_nonzero_from(pre, static_cast<uint64_t>(u), static_cast<uint64_t>(d), 0);
  }
}

__global__ void k_zj_positional(int32_t n, int k, uint64_t seed, uint64_t* __restrict__ zj) {
  const int64_t u = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (u >= n) return;
  const uint64_t pre = draw_prefix(seed, 5);  // Role::label_z (gf.hpp:116)
  for (int j = 0; j < k; ++j)
    zj[u * k + j] = draw_nonzero_from(pre, static_cast<uint64_t>(u), static_cast<uint64_t>(j + 1), 0);
}

// One warp per arc of the timestamp's edges; each lane owns W/32 points.
__global__ void k_ec_level(int64_t e0, int64_t e1, int directed, const int32_t* __restrict__ eu,
                           const int32_t* __restrict__ ev, const uint64_t* __restrict__ zb,
                           int W, uint64_t seed, int ell, const uint64_t* __restrict__ prev,
                           uint64_t* __restrict__ cur) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t arcs = (e1 - e0) * (directed ? 1 : 2);
  if (warp >= arcs) return;
  const int64_t e = e0 + (directed ? warp : (warp >> 1));
  const bool rev = !directed && (warp & 1);
  const int32_t tail = rev ? ev[e] : eu[e], head = rev ? eu[e] : ev[e];
  const uint64_t pre = draw_prefix(seed, kRoleEdgeY);
  const uint64_t y = draw_edge_y(pre, static_cast<uint64_t>(ell - 1) + 0x165667b19e3779f9ull,
                                 static_cast<uint32_t>(e));
  for (int w = lane; w < W; w += 32) {
    const uint64_t s = __ldg(prev + static_cast<int64_t>(tail) * W + w);
    const uint64_t v = gf_mul(__ldg(zb + static_cast<int64_t>(head) * W + w), gf_mul(y, s));
    if (v)
      atomicXor(reinterpret_cast<unsigned long long*>(cur + static_cast<int64_t>(head) * W + w),
                static_cast<unsigned long long>(v));
  }
}

__global__ void k_row_xor(int32_t n, int W, const uint64_t* __restrict__ rows,
                          uint64_t* __restrict__ acc) {
  const int64_t u = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (u >= n) return;
  uint64_t x = 0;
  for (int w = 0; w < W; ++w) x ^= rows[u * W + w];
  acc[u] ^= x;
}

__global__ void k_vc_dp_level(int64_t m, int directed, const int32_t* __restrict__ eu,
                              const int32_t* __restrict__ ev, const int32_t* __restrict__ ets,
                              int32_t max_ts, const int32_t* __restrict__ colors,
                              int32_t tail_c, int32_t head_c, int32_t wild,
                              const int32_t* __restrict__ e_prev, int32_t* __restrict__ e_next) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const int32_t t = ets[i];
  if (t > max_ts) return;
  auto relax = [&](int32_t head, int32_t tail) {
    if (!has_color(colors, head, head_c, wild) || !has_color(colors, tail, tail_c, wild)) return;
    if (e_prev[tail] <= t) atomicMin(e_next + head, t + 1);
  };
  relax(ev[i], eu[i]);
  if (!directed) relax(eu[i], ev[i]);
}

__global__ void k_xor_combine(const uint64_t* __restrict__ parts, int nparts,
                              int64_t n, uint64_t* __restrict__ out) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
       i < n; i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    uint64_t x = 0;
    for (int p = 0; p < nparts; ++p) x ^= parts[p * n + i];
    out[i] = x;
  }
}

__global__ void k_draw_y(uint64_t seed, int32_t level, int64_t n,
                         const int32_t* edges, uint64_t* out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t pre = draw_prefix(seed, kRoleEdgeY);
  out[i] = draw_edge_y(pre, static_cast<uint64_t>(level - 1) + 0x165667b19e3779f9ull,
                       static_cast<uint32_t>(edges[i]));
}

template <int LANES, int PPT>
void level_dispatch(const LevelParams& p, cudaStream_t st) {
  const dim3 grid(static_cast<unsigned>((p.g.C + kWarpsPerBlock - 1) / kWarpsPerBlock));
  const dim3 block(kWarpsPerBlock * 32);
  if (LANES == 32) {
    const dim3 wgrid(static_cast<unsigned>((p.g.C + kWideWarps - 1) / kWideWarps));
    const dim3 wblock(kWideWarps * 32);
    const bool first = p.ell == 2;
#define TSV_WIDE(Y, L)                                                      \
  do {                                                                      \
    if (first) k_level_wide<PPT, true, Y, L><<<wgrid, wblock, 0, st>>>(p);  \
    else k_level_wide<PPT, false, Y, L><<<wgrid, wblock, 0, st>>>(p);       \
  } while (0)
    if (p.ymul == 1) {
      if (p.last) TSV_WIDE(false, true);
      else TSV_WIDE(false, false);
    } else {
      if (p.last) TSV_WIDE(true, true);
      else TSV_WIDE(true, false);
    }
#undef TSV_WIDE
    return;
  }
  if (LANES < 32 && PPT == 1) {
    constexpr int L = LANES < 32 ? LANES : 16;  // (instantiated for LANES < 32 only)
    if (p.ell == 2) {
      if (p.last) k_level<L, true, true><<<grid, block, 0, st>>>(p);
      else k_level<L, true, false><<<grid, block, 0, st>>>(p);
    } else {
      if (p.last) k_level<L, false, true><<<grid, block, 0, st>>>(p);
      else k_level<L, false, false><<<grid, block, 0, st>>>(p);
    }
  }
}

unsigned blocks_for(int64_t n, int threads) {
  return static_cast<unsigned>((n + threads - 1) / threads);
}


// Shade CSR in which every vertex carries the same shade list (k-TempPath:
// all k shades; C5): off[i] = i * c, shades[i * c + j] = pattern[j].
__global__ void k_uniform_csr(int32_t n, int c, const int32_t* __restrict__ pattern,
                              int32_t* __restrict__ off, int32_t* __restrict__ shades) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i > n) return;
  off[i] = static_cast<int32_t>(i * c);
  if (i < n)
    for (int j = 0; j < c; ++j) shades[i * c + j] = pattern[j];
}

}  // namespace

void launch_level(const LevelParams& p, cudaStream_t st) {
  if (p.g.C == 0) return;
  // profile names: the wide kernel's middle levels are "level"; the grouped
  // kernel (W < 32) reports as "level_grouped[_first]"
  const bool wide = p.b.lanes == 32;
  prof_begin(p.last ? "level_last"
             : p.ell == 2 ? (wide ? "level_first" : "level_grouped_first")
                          : (wide ? "level" : "level_grouped"),
             st);
  switch (p.b.lanes * 8 + p.b.ppt) {
    case 1 * 8 + 1: level_dispatch<1, 1>(p, st); break;
    case 2 * 8 + 1: level_dispatch<2, 1>(p, st); break;
    case 4 * 8 + 1: level_dispatch<4, 1>(p, st); break;
    case 8 * 8 + 1: level_dispatch<8, 1>(p, st); break;
    case 16 * 8 + 1: level_dispatch<16, 1>(p, st); break;
    case 32 * 8 + 1: level_dispatch<32, 1>(p, st); break;
    case 32 * 8 + 2: level_dispatch<32, 2>(p, st); break;
    case 32 * 8 + 4: level_dispatch<32, 4>(p, st); break;
    default: break;
  }
  prof_end(st);
}

void launch_fixup(const LevelParams& p, cudaStream_t st) {
  if (p.g.ncarry == 0) return;
  prof_begin("fixup", st);
  const int threads = p.b.W() < 128 ? ((p.b.W() + 31) / 32) * 32 : 128;
  k_fixup<<<p.g.ncarry, threads, 0, st>>>(p);
  prof_end(st);
}

void launch_zbatch(int32_t n, const uint64_t* zj, int k, const Batch& b, uint64_t* zb,
                   cudaStream_t st) {
  if (n == 0) return;
  prof_begin("zbatch", st);
  k_zbatch<<<static_cast<unsigned>((static_cast<int64_t>(n) * 32 + 255) / 256), 256, 0, st>>>(
      n, zj, k, b, zb);
  prof_end(st);
}

void launch_k1(int32_t n, const uint64_t* zj, Batch b, int32_t anchor_source,
               uint64_t* acc, cudaStream_t st, const int32_t* colors, int32_t color,
               int32_t wild) {
  if (n == 0) return;
  prof_begin("k1", st);
  k_k1<<<blocks_for(n, 256), 256, 0, st>>>(n, zj, b, anchor_source, acc, colors, color, wild);
  prof_end(st);
}

void launch_wtab(int k, uint64_t seed, uint64_t* wtab, cudaStream_t st) {
  k_wtab<<<blocks_for(static_cast<int64_t>(k) * k, 256), 256, 0, st>>>(k, seed, wtab);
}

void launch_zj(int32_t n, int k, uint64_t seed, const int32_t* vertex_off,
               const int32_t* vertex_shades, const uint64_t* wtab, uint64_t* zj,
               cudaStream_t st) {
  if (n == 0) return;
  prof_begin("zj", st);
  k_zj<<<blocks_for(n, 128), 128, 0, st>>>(n, k, seed, vertex_off, vertex_shades, wtab, zj);
  prof_end(st);
}

void launch_xor_combine(const uint64_t* parts, int nparts, int64_t n, uint64_t* out,
                        cudaStream_t st) {
  if (n == 0) return;
  prof_begin("xor_combine", st);
  const unsigned blocks = blocks_for(n, 256) < 148 * 8 ? blocks_for(n, 256) : 148 * 8;
  k_xor_combine<<<blocks, 256, 0, st>>>(parts, nparts, n, out);
  prof_end(st);
}

void launch_zj_ident(int32_t n, int k, uint64_t seed, const int32_t* vertex_off,
                     const int32_t* vertex_shades, uint64_t* zj, cudaStream_t st) {
  if (n == 0) return;
  prof_begin("zj", st);
  k_zj_ident<<<blocks_for(n, 256), 256, 0, st>>>(n, k, seed, vertex_off, vertex_shades, zj);
  prof_end(st);
}

void launch_zj_positional(int32_t n, int k, uint64_t seed, uint64_t* zj, cudaStream_t st) {
  if (n == 0) return;
  prof_begin("zj", st);
  k_zj_positional<<<blocks_for(n, 128), 128, 0, st>>>(n, k, seed, zj);
  prof_end(st);
}

void launch_ec_level(int64_t e0, int64_t e1, int directed, const int32_t* eu,
                     const int32_t* ev, const uint64_t* zb, int W, uint64_t seed, int ell,
                     const uint64_t* prev, uint64_t* cur, cudaStream_t st) {
  const int64_t arcs = (e1 - e0) * (directed ? 1 : 2);
  if (arcs <= 0) return;
  prof_begin("ec_level", st);
  k_ec_level<<<blocks_for(arcs * 32, 256), 256, 0, st>>>(e0, e1, directed, eu, ev, zb, W, seed,
                                                        ell, prev, cur);
  prof_end(st);
}

void launch_row_xor(int32_t n, int W, const uint64_t* rows, uint64_t* acc, cudaStream_t st) {
  if (n == 0) return;
  k_row_xor<<<blocks_for(n, 256), 256, 0, st>>>(n, W, rows, acc);
}

void launch_vc_dp_level(int64_t m, int directed, const int32_t* eu, const int32_t* ev,
                        const int32_t* ets, int32_t max_ts, const int32_t* colors,
                        int32_t tail_color, int32_t head_color, int32_t wild,
                        const int32_t* e_prev, int32_t* e_next, cudaStream_t st) {
  if (m == 0) return;
  k_vc_dp_level<<<blocks_for(m, 256), 256, 0, st>>>(m, directed, eu, ev, ets, max_ts, colors,
                                                   tail_color, head_color, wild, e_prev, e_next);
}

void launch_draw_y(uint64_t seed, int32_t level, int64_t n, const int32_t* edges,
                   uint64_t* out, cudaStream_t st) {
  if (n == 0) return;
  k_draw_y<<<blocks_for(n, 256), 256, 0, st>>>(seed, level, n, edges, out);
}

void launch_uniform_csr(int32_t n, int c, const int32_t* pattern, int32_t* off, int32_t* shades,
                        cudaStream_t st) {
  k_uniform_csr<<<blocks_for(static_cast<int64_t>(n) + 1, 256), 256, 0, st>>>(n, c, pattern, off,
                                                                               shades);
}

}  // namespace tsv

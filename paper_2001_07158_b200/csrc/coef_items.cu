// coef_items.cu -- the coefficient engine's arc pass as an item stream over
// compact shade frames (used whenever the shade table has vertices with a
// single shade).
//
// In the shade basis (coef_kernels.cu, top) the level-l state of a run is
// indexed by the l-subsets T of the k shades.  A vertex h with exactly one
// shade d has S_l[T] = v_{h,d} * U_l[T - {d}] for T containing d and 0
// otherwise, so its rows keep only U_l over the (l-1)-subsets WITHOUT d
// (its "frame", C(k-1, l-1) entries; v_{h,d} rides on the y of the arcs
// leaving h).  A vertex with several shades keeps full rows (C(k, l-1) U
// entries, mapped in place to S by k_coef_ztrans_tab).  For an arc t -> h
// of level l the entries that can be nonzero AND are ever read are the
// (l-1)-subsets T with d_t in T (single-shade tail) and d_h not in T
// (single-shade head): C(k-2, l-2) of them, against the C(k, l-1) lanes the
// point-to-entry mapping of k_coef_arcs spends.  Each (tail class, head
// class) pair has a host-built list of (input index, output index) items.
//
// A warp owns a chunk of the vertex-major arc stream.  Per 32 arcs it stages
// y' (= y * v_tail for single-shade tails), the pair's item list and the
// events (vertex start, referenced run end) in shared memory, flattens the
// items of the live arcs into one stream and walks it 32 items at a time:
// every lane forms one product -- with the arc's y' table when all 32 items
// belong to one arc (conflict-free GfTable lookups), else the general
// product with y' split once per arc -- and the products are XORed into the
// head's U prefix in shared memory arc by arc (in stream order, so a run end
// snapshots exactly the prefix up to its arc).  A snapshot writes the frame
// (<= C(k, l-1) words) to the run's state slot; at level k the prefix of
// each vertex piece is XORed into ulast (k_coef_readout finishes).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <utility>
#include <vector>

#include "coef.hpp"
#include "gf_device.cuh"
#include "layout.hpp"

namespace tsv {
namespace {

// rounds per super-round of the deep levels (source loads in flight per lane)
#ifndef TSV_ITEMS_SUB
#define TSV_ITEMS_SUB 2
#endif
#ifndef TSV_ITEMS_WARPS
#define TSV_ITEMS_WARPS 4
#endif
constexpr int kIW = TSV_ITEMS_WARPS;  // warps per block
constexpr unsigned kFull = 0xffffffffu;
constexpr uint32_t kEvStart = 1u, kEvPush = 2u;
#ifndef TSV_ITEMS_BIG
#define TSV_ITEMS_BIG 24
#endif
constexpr int kBig = TSV_ITEMS_BIG;
constexpr int kSub = 4;   // rounds per super-round (loads in flight per lane)  // items from which an arc gets whole rounds (table products)

// the prefix a vertex starts from: its carried U entry o (time windows), else 0
__device__ __forceinline__ uint64_t carry_entry(const CoefParams& P, int32_t h, int o) {
  if (!P.carry_in || h < 0 || !__ldg(P.carry_nz + h)) return 0ull;
  return __ldg(P.carry_in + static_cast<int64_t>(h) * P.carry_cs + o);
}

__device__ __forceinline__ bool color_ok(const int32_t* __restrict__ colors, int32_t x,
                                         int32_t c, int32_t wild) {
  return c == wild || __ldg(colors + x) == c;
}

// kSub: rounds per super-round (source loads in flight per lane; 4 for
// levels whose arcs carry many items, 1 otherwise)
template <bool FIRST, bool LAST, int kSub>
__global__ void __launch_bounds__(kIW * 32) k_coef_items(const CoefParams P) {
  extern __shared__ uint64_t dsm[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  // per-warp shared layout: GfTable (256-byte aligned) | acc[frame_multi]
  const uint32_t raw = static_cast<uint32_t>(__cvta_generic_to_shared(dsm));
  uint64_t* const tab = dsm + ((256u - (raw & 255u)) & 255u) / 8 +
                        static_cast<size_t>(wib) * P.warp_words;
  uint64_t* const acc = tab + GfTable::kWords;
  __shared__ uint32_t s_ys[kIW][12][32];
  __shared__ uint64_t s_y[kIW][32];
  __shared__ int64_t s_row[kIW][32];   // source row offset (-1: the value 1)
  __shared__ int32_t s_start[kIW][32]; // item stream offsets of the active arcs
  __shared__ int32_t s_cnt[kIW][32];   // item counts
  __shared__ int32_t s_poff[kIW][32];  // item list offset
  __shared__ int32_t s_dst[kIW][32];   // slot (levels < k) or head (level k)
  __shared__ int32_t s_hd[kIW][32];    // head
  __shared__ int16_t s_fr[kIW][32];    // head frame size
  __shared__ uint8_t s_ev[kIW][32];

  const int64_t c = static_cast<int64_t>(blockIdx.x) * kIW + wib;
  if (c >= P.g.C) return;  // warp-uniform
  const int k = P.k;
  const uint64_t pre = draw_prefix(P.seed, kRoleEdgeY);
  const uint64_t yb = static_cast<uint64_t>(P.ell - 1) + 0x165667b19e3779f9ull;
  const int64_t a0 = P.g.chunk_arc[c], a1 = P.g.chunk_arc[c + 1];
  int32_t run_ctr = P.g.chunk_run[c];
  int frame = P.frame_max;  // frame of the current head
  for (int o = lane; o < P.frame_max; o += 32) acc[o] = 0;

  for (int64_t base = a0; base < a1; base += 32) {
    const int nb = static_cast<int>(a1 - base < 32 ? a1 - base : 32);
    uint32_t meta = 0;
    int32_t sidx = -1, head = -1, tail = -1;
    uint64_t y = 0;
    if (lane < nb) {
      meta = __ldg(P.g.arc_meta + base + lane);
      sidx = FIRST ? __ldg(P.g.arc_tail + base + lane) : __ldg(P.g.arc_src + base + lane);
      tail = FIRST ? sidx : __ldg(P.g.arc_tail + base + lane);
    }
    const unsigned ends = __ballot_sync(kFull, lane < nb && (meta & kRunEnd));
    const int32_t myrun = run_ctr + __popc(ends & ((1u << lane) - 1u));
    run_ctr += __popc(ends);
    if (lane < nb) head = __ldg(P.g.run_head + myrun);
    const int hs = lane < nb ? __ldg(P.vsh + head) : -1;  // head shade class
    bool live = lane < nb && sidx >= 0 && hs != -1;
    if (FIRST) live = live && (P.anchor_source < 0 || sidx == P.anchor_source);
    if (LAST) live = live && __ldg(P.g.run_ts + myrun) <= P.max_ts;
    if (P.vc_color && live)
      live = tail >= 0 && color_ok(P.vc_color, tail, P.vc_tail, P.vc_wild) &&
             color_ok(P.vc_color, head, P.vc_head, P.vc_wild);
    int ts = -1;
    if (live) {
      ts = __ldg(P.vsh + tail);
      live = ts != -1 && (FIRST || __ldg(P.sflag + sidx) != 0);
    }
    int nitem = 0, poff = 0;
    if (live) {
      const int pt = (ts >= 0 ? ts : k) * (k + 1) + (hs >= 0 ? hs : k);
      nitem = __ldg(P.item_cnt + pt);
      poff = __ldg(P.item_off + pt);
      live = nitem > 0;
      if (!live) nitem = 0;
    }
    if (live) y = draw_edge_y(pre, yb, meta & kEdgeMask);
    if (live && ts >= 0) y = gf_mul(y, __ldg(P.vsv + tail));  // v_tail rides on y
    bool push;
    int32_t dst = -1;
    if (LAST) {  // last arc of its vertex within this chunk: flush the piece
      const bool chunk_end = base + lane + 1 >= a1;
      uint32_t nmeta = __shfl_down_sync(kFull, meta, 1);
      if (lane == 31 && !chunk_end) nmeta = __ldg(P.g.arc_meta + base + 32);
      push = lane < nb && hs != -1 && (chunk_end || (nmeta & kVStart));
      dst = head;
    } else {
      dst = (lane < nb && hs != -1 && (meta & kRunEnd)) ? __ldg(P.g.run_slot + myrun) : -1;
      push = dst >= 0;
    }
    const bool vst = lane < nb && (meta & kVStart);
    const bool act = live || push || vst;
    const unsigned actm = __ballot_sync(kFull, act);
    const int nact = __popc(actm);
    // stream positions: arcs with >= kBig items start on a 32-item round
    // boundary (all their full rounds use the arc's y' table), smaller ones
    // are packed (general products)
    const bool big = nitem >= kBig;
    int my_s, total;
    if (__any_sync(kFull, big)) {
      // aligned exclusive scan, sequential over the arcs (at most 32)
      int pos = 0;
      my_s = 0;
      for (int j = 0; j < 32; ++j) {
        const int nj = __shfl_sync(kFull, nitem, j);
        if (nj >= kBig) pos = (pos + 31) & ~31;
        if (lane == j) my_s = pos;
        pos += nj;
      }
      total = pos;
    } else {
      int incl = nitem;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int o = __shfl_up_sync(kFull, incl, d);
        if (lane >= d) incl += o;
      }
      my_s = incl - nitem;
      total = __shfl_sync(kFull, incl, 31);
    }
    if (act) {
      const int ai = __popc(actm & ((1u << lane) - 1u));
      s_start[wib][ai] = my_s;
      s_cnt[wib][ai] = nitem;
      s_poff[wib][ai] = poff;
      s_dst[wib][ai] = dst;
      s_hd[wib][ai] = head;
      s_fr[wib][ai] = static_cast<int16_t>(hs >= 0 ? P.frame_single : P.frame_multi);
      s_ev[wib][ai] = (vst ? kEvStart : 0u) | (push ? kEvPush : 0u);
      s_y[wib][ai] = y;
      s_row[wib][ai] = !live ? 0
                       : FIRST ? (ts >= 0 ? -1 : static_cast<int64_t>(sidx) * k)
                               : static_cast<int64_t>(sidx) * P.rs_in;
      const KSplit ks = ksplit(y);  // a big arc's last round may be shared
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        s_ys[wib][j][ai] = ks.l.c[j];
        s_ys[wib][4 + j][ai] = ks.h.c[j];
        s_ys[wib][8 + j][ai] = ks.m.c[j];
      }
    }
    __syncwarp();
    // lane j keeps active arc j's item range [as, ae)
    const int as = lane < nact ? s_start[wib][lane] : INT32_MAX;
    const int ae = lane < nact ? as + s_cnt[wib][lane] : INT32_MAX;

    int ea = 0;      // next active arc with pending events
    int tab_arc = -1;
    // item q0 + lane -> (arc, output entry, source value); the arcs whose
    // ranges meet the round are found with one ballot
    auto locate = [&](int q0, int& ia, int& out, uint64_t& u, bool& uni) {
      ia = -1;
      out = 0;
      u = 0;
      const int q = q0 + lane;
      unsigned m = __ballot_sync(kFull, lane < nact && as < q0 + 32 && ae > q0 && ae > as);
      uni = __popc(m) == 1;
      if (uni) {
        const int j = __ffs(m) - 1;
        if (q < __shfl_sync(kFull, ae, j)) ia = j;
      } else {
        while (m) {
          const int j = __ffs(m) - 1;
          m &= m - 1;
          const int sj = __shfl_sync(kFull, as, j), ej = __shfl_sync(kFull, ae, j);
          if (q >= sj && q < ej) ia = j;
        }
      }
      if (ia >= 0) {
        const int2 it = __ldg(P.items + s_poff[wib][ia] + (q - s_start[wib][ia]));
        out = it.y;
        const int64_t row = s_row[wib][ia];
        u = row < 0 ? 1ull : FIRST ? __ldg(P.zj + row + it.x) : __ldg(P.s_prev + row + it.x);
      }
    };
    // super-rounds of kSub rounds: every lane's kSub source loads are in
    // flight before the first product
    for (int Q0 = 0; ea < nact; Q0 += 32 * kSub) {
      int ia_s[kSub], out_s[kSub];
      uint64_t u_s[kSub];
      bool uni_s[kSub];
#pragma unroll
      for (int r = 0; r < kSub; ++r) locate(Q0 + 32 * r, ia_s[r], out_s[r], u_s[r], uni_s[r]);
#pragma unroll
      for (int r = 0; r < kSub; ++r) {
      const int q0 = Q0 + 32 * r;
      const int ia = ia_s[r], out = out_s[r];
      const uint64_t u = u_s[r];
      const bool uni = uni_s[r];
      uint64_t prod = 0;
      // one arc's items only (the table's arc is the one with a range here)
      const int ia0 = __reduce_max_sync(kFull, ia);
      const bool uniform = uni && ia0 >= 0 && s_cnt[wib][ia0] >= kBig;
      if (uniform) {  // all 32 items of one arc: its y' table
        if (tab_arc != ia0) {
          __syncwarp();
          GfTable{tab}.build(s_y[wib][ia0], lane);
          __syncwarp();
          tab_arc = ia0;
        }
        prod = u ? GfTable{tab}.mul(u) : 0ull;
      } else if (ia >= 0 && u) {
        KSplit ys;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          ys.l.c[j] = s_ys[wib][j][ia];
          ys.h.c[j] = s_ys[wib][4 + j][ia];
          ys.m.c[j] = s_ys[wib][8 + j][ia];
        }
        prod = gf_mul_presplit(ys, u);
      }
      // events in stream order, arc by arc
      while (ea < nact) {
        const int sa = s_start[wib][ea], se = sa + s_cnt[wib][ea];
        if (sa >= q0 + 32) break;  // its items start in a later round
        const uint32_t ev = s_ev[wib][ea];
        if ((ev & kEvStart) && sa >= q0) {  // first part of a new vertex: reset
          __syncwarp();
          frame = s_fr[wib][ea];
          const int32_t hd = s_hd[wib][ea];
          for (int o = lane; o < frame; o += 32) acc[o] = carry_entry(P, hd, o);
          __syncwarp();
        }
        if (ia == ea) acc[out] ^= prod;
        __syncwarp();
        if (se > q0 + 32) break;  // continues in the next round
        if (ev & kEvPush) {
          const int32_t d = s_dst[wib][ea];
          const int fr = s_fr[wib][ea];
          if (LAST) {
            for (int o = lane; o < fr; o += 32) {
              const uint64_t x = acc[o];
              if (x)
                atomicXor(reinterpret_cast<unsigned long long*>(P.ulast +
                                                                static_cast<int64_t>(d) * k + o),
                          static_cast<unsigned long long>(x));
            }
          } else {
            bool nz = false;
            uint64_t* rowp = P.ubuf + static_cast<int64_t>(d) * P.rs_out;
            for (int o = lane; o < fr; o += 32) {
              const uint64_t x = acc[o];
              rowp[o] = x;
              nz = nz || x != 0;
            }
            if (__any_sync(kFull, nz) && lane == 0) P.sflag_out[d] = 1;
          }
        }
        ++ea;
      }
      }  // sub-rounds
    }
    __syncwarp();
  }
  if (!LAST) {  // chunk tail prefix for k_coef_fixup (frame of the last vertex)
    for (int o = lane; o < frame; o += 32) P.agg[c * P.E + o] = acc[o];
  }
}


// Small frames (frame_max <= 32 * NO, i.e. k <= 7): the same item stream,
// but a batch's products are first stored to per-arc rows in shared memory
// (prow[arc][entry]; items of one arc have distinct outputs, so a plain
// store) and the head prefixes are then walked arc by arc with lane o
// holding entry o (and o + 32) of the prefix in registers.  The walk visits
// only the arcs with an event (vertex start, live products, referenced run
// end), taken from warp ballots, and needs no shared accumulator or
// per-arc warp barrier: the serial part of k_coef_items costs ~10
// instructions per event instead of ~40.
#ifndef TSV_REG_MINB
#define TSV_REG_MINB 7  // <= 72 registers: 7 blocks of 4 warps per SM
#endif
template <bool FIRST, bool LAST, int NO>
__global__ void __launch_bounds__(kIW * 32, TSV_REG_MINB)
    k_coef_items_reg(const CoefParams P, int fmp) {
  extern __shared__ uint64_t dsm[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  uint64_t* const prow = dsm + static_cast<size_t>(wib) * 32 * fmp;
  __shared__ uint32_t s_ys[kIW][12][32];
  __shared__ int64_t s_row[kIW][32];   // source row offset (-1: the value 1)
  __shared__ int32_t s_start[kIW][33]; // item stream offsets of the live arcs
  __shared__ int32_t s_poff[kIW][32];  // item list offset
  __shared__ int8_t s_lane[kIW][32];   // the live arc's lane (its prow row)
  __shared__ uint64_t s_om[kIW][32];   // by lane: outputs the arc's items reach

  const int k = P.k;
  const int fm = P.frame_max;
  const uint64_t pre = draw_prefix(P.seed, kRoleEdgeY);
  const uint64_t yb = static_cast<uint64_t>(P.ell - 1) + 0x165667b19e3779f9ull;
  // persistent warps: the first chunk by warp id, then from the counter
  // (chunks hold ~A / 9500 arcs, so one chunk per warp left a 30% tail wave)
  const int64_t nwarps = static_cast<int64_t>(gridDim.x) * kIW;
  for (int64_t c = static_cast<int64_t>(blockIdx.x) * kIW + wib; c < P.g.C;) {
  const int64_t a0 = P.g.chunk_arc[c], a1 = P.g.chunk_arc[c + 1];
  int32_t run_ctr = P.g.chunk_run[c];
  int frame = fm;  // frame of the current head
  uint64_t acc0 = 0, acc1 = 0;  // prefix entries lane, lane + 32

  for (int64_t base = a0; base < a1; base += 32) {
    const int nb = static_cast<int>(a1 - base < 32 ? a1 - base : 32);
    uint32_t meta = 0;
    int32_t sidx = -1, head = -1, tail = -1;
    uint64_t y = 0;
    if (lane < nb) {
      meta = __ldg(P.g.arc_meta + base + lane);
      sidx = FIRST ? __ldg(P.g.arc_tail + base + lane) : __ldg(P.g.arc_src + base + lane);
      tail = FIRST ? sidx : __ldg(P.g.arc_tail + base + lane);
    }
    const unsigned ends = __ballot_sync(kFull, lane < nb && (meta & kRunEnd));
    const int32_t myrun = run_ctr + __popc(ends & ((1u << lane) - 1u));
    run_ctr += __popc(ends);
    if (lane < nb) head = __ldg(P.g.run_head + myrun);
    const int hs = lane < nb ? __ldg(P.vsh + head) : -1;  // head shade class
    bool live = lane < nb && sidx >= 0 && hs != -1;
    if (FIRST) live = live && (P.anchor_source < 0 || sidx == P.anchor_source);
    if (LAST) live = live && __ldg(P.g.run_ts + myrun) <= P.max_ts;
    int ts = -1;
    if (live) {
      ts = __ldg(P.vsh + tail);
      live = ts != -1 && (FIRST || __ldg(P.sflag + sidx) != 0);
    }
    int nitem = 0, poff = 0;
    uint64_t omask = 0;  // outputs the arc's items reach (its prow entries)
    if (live) {
      const int pt = (ts >= 0 ? ts : k) * (k + 1) + (hs >= 0 ? hs : k);
      nitem = __ldg(P.item_cnt + pt);
      poff = __ldg(P.item_off + pt);
      omask = __ldg(P.item_omask + pt);
      live = nitem > 0;
      if (!live) nitem = 0;
    }
    if (live) y = draw_edge_y(pre, yb, meta & kEdgeMask);
    if (live && ts >= 0) y = gf_mul(y, __ldg(P.vsv + tail));  // v_tail rides on y
    bool push;
    int32_t dst = -1;
    if (LAST) {  // last arc of its vertex within this chunk: flush the piece
      const bool chunk_end = base + lane + 1 >= a1;
      uint32_t nmeta = __shfl_down_sync(kFull, meta, 1);
      if (lane == 31 && !chunk_end) nmeta = __ldg(P.g.arc_meta + base + 32);
      push = lane < nb && hs != -1 && (chunk_end || (nmeta & kVStart));
      dst = head;
    } else {
      dst = (lane < nb && hs != -1 && (meta & kRunEnd)) ? __ldg(P.g.run_slot + myrun) : -1;
      push = dst >= 0;
    }
    const int myfr = hs >= 0 ? P.frame_single : P.frame_multi;
    const unsigned vstm = __ballot_sync(kFull, lane < nb && (meta & kVStart));
    const unsigned livem = __ballot_sync(kFull, live);
    const unsigned pushm = __ballot_sync(kFull, push);

    // compact the live arcs; exclusive scan of their item counts
    int incl = nitem;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int o = __shfl_up_sync(kFull, incl, d);
      if (lane >= d) incl += o;
    }
    const int total = __shfl_sync(kFull, incl, 31);
    const int nlive = __popc(livem);
    __syncwarp();  // the previous batch's readers of the staging arrays are done
    s_om[wib][lane] = omask;
    if (live) {
      const int ai = __popc(livem & ((1u << lane) - 1u));
      s_start[wib][ai] = incl - nitem;
      s_poff[wib][ai] = poff;
      s_lane[wib][ai] = static_cast<int8_t>(lane);
      s_row[wib][ai] = FIRST ? (ts >= 0 ? -1 : static_cast<int64_t>(sidx) * k)
                             : static_cast<int64_t>(sidx) * P.rs_in;
      const KSplit ks = ksplit(y);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        s_ys[wib][j][ai] = ks.l.c[j];
        s_ys[wib][4 + j][ai] = ks.h.c[j];
        s_ys[wib][8 + j][ai] = ks.m.c[j];
      }
    }
    // a live arc's row holds exactly the outputs its items reach (omask);
    // the walk reads no other entry, so the rows need no clearing
    if (lane == 0) s_start[wib][nlive] = total;
    __syncwarp();

    // item q -> live arc j with s_start[j] <= q < s_start[j + 1]
    for (int q0 = 0; q0 < total; q0 += 64) {
      int jj[2], out[2];
      uint64_t u[2];
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int q = q0 + 32 * r + lane;
        jj[r] = -1;
        out[r] = 0;
        u[r] = 0;
        if (q < total) {
          int j = 0;
#pragma unroll
          for (int st = 16; st >= 1; st >>= 1)
            if (j + st < nlive && s_start[wib][j + st] <= q) j += st;
          jj[r] = j;
          const int2 it = __ldg(P.items + s_poff[wib][j] + (q - s_start[wib][j]));
          out[r] = it.y;
          const int64_t row = s_row[wib][j];
          u[r] = row < 0 ? 1ull : FIRST ? __ldg(P.zj + row + it.x) : __ldg(P.s_prev + row + it.x);
        }
      }
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        if (jj[r] >= 0 && !u[r]) prow[s_lane[wib][jj[r]] * fmp + out[r]] = 0ull;
        if (jj[r] >= 0 && u[r]) {
          const int j = jj[r];
          KSplit ys;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            ys.l.c[i] = s_ys[wib][i][j];
            ys.h.c[i] = s_ys[wib][4 + i][j];
            ys.m.c[i] = s_ys[wib][8 + i][j];
          }
          prow[s_lane[wib][j] * fmp + out[r]] = gf_mul_presplit(ys, u[r]);
        }
      }
    }
    __syncwarp();

    // walk the arcs with events in stream order
    unsigned ev = vstm | livem | pushm;
    if constexpr (NO == 0) {
      // frames <= 16 words: the two half-warps walk two parts of the batch at
      // once, split at a vertex start near the middle (half 1 begins with a
      // fresh prefix; half 0 continues the carried one); lane o & 15 holds
      // entry o & 15 of its half's prefix.  (Two entries per lane for frames
      // <= 32 measured slower than the one-half walk: C2 +2%, C3 +5%.)
      const int h = lane >> 4, o = lane & 15;
      const unsigned mid = static_cast<unsigned>(nb >> 1);
      const unsigned hi = vstm & ~((1u << mid) - 1u) & ~1u;
      const unsigned lo = vstm & ((1u << mid) - 1u) & ~1u;
      const int sp = hi ? __ffs(hi) - 1 : lo ? 31 - __clz(lo) : 32;
      const unsigned below = sp >= 32 ? kFull : ((1u << sp) - 1u);
      unsigned evh = h == 0 ? (ev & below) : (ev & ~below);
      if (sp < 32 && h == 1) acc0 = 0;
      while (__any_sync(kFull, evh != 0)) {
        const int a = evh ? __ffs(evh) - 1 : 0;
        const bool on = evh != 0;
        if (on) evh &= evh - 1;
        const unsigned bit = on ? 1u << a : 0u;
        const int fra = __shfl_sync(kFull, myfr, a);
        const int32_t d = __shfl_sync(kFull, dst, a);
        const int32_t hd = __shfl_sync(kFull, head, a);
        if (vstm & bit) {
          acc0 = o < fra ? carry_entry(P, hd, o) : 0ull;
          frame = fra;
        }
        if (livem & bit) {
          const uint64_t om = s_om[wib][a];
          if ((om >> o) & 1u) acc0 ^= prow[a * fmp + o];
        }
        const bool ps = (pushm & bit) != 0;
        if (LAST) {
          if (ps && o < fra && acc0)
            atomicXor(reinterpret_cast<unsigned long long*>(P.ulast +
                                                            static_cast<int64_t>(d) * k + o),
                      static_cast<unsigned long long>(acc0));
        } else {
          if (ps && o < fra) P.ubuf[static_cast<int64_t>(d) * P.rs_out + o] = acc0;
          const unsigned nzb = __ballot_sync(kFull, ps && o < fra && acc0 != 0);
          if (ps && o == 0 && ((nzb >> (16 * h)) & 0xffffu)) P.sflag_out[d] = 1;
        }
      }
      if (sp < 32) {  // the batch's last vertex ran in half 1: carry its prefix
        acc0 = __shfl_sync(kFull, acc0, o + 16);
        frame = __shfl_sync(kFull, frame, 16);
      }
      continue;
    }
    while (ev) {
      const int a = __ffs(ev) - 1;
      ev &= ev - 1;
      const unsigned bit = 1u << a;
      if (vstm & bit) {
        frame = __shfl_sync(kFull, myfr, a);
        const int32_t hd = __shfl_sync(kFull, head, a);
        acc0 = lane < frame ? carry_entry(P, hd, lane) : 0ull;
        if (NO > 1) acc1 = lane + 32 < frame ? carry_entry(P, hd, lane + 32) : 0ull;
      }
      if (livem & bit) {
        const uint64_t om = s_om[wib][a];
        if ((om >> lane) & 1u) acc0 ^= prow[a * fmp + lane];
        if (NO > 1 && ((om >> (32 + lane)) & 1u)) acc1 ^= prow[a * fmp + 32 + lane];
      }
      if (pushm & bit) {
        const int32_t d = __shfl_sync(kFull, dst, a);
        const int fr = __shfl_sync(kFull, myfr, a);
        if (LAST) {
          uint64_t* up = P.ulast + static_cast<int64_t>(d) * k;
          if (lane < fr && acc0)
            atomicXor(reinterpret_cast<unsigned long long*>(up + lane),
                      static_cast<unsigned long long>(acc0));
          if (NO > 1 && lane + 32 < fr && acc1)
            atomicXor(reinterpret_cast<unsigned long long*>(up + 32 + lane),
                      static_cast<unsigned long long>(acc1));
        } else {
          uint64_t* rowp = P.ubuf + static_cast<int64_t>(d) * P.rs_out;
          bool nz = false;
          if (lane < fr) {
            rowp[lane] = acc0;
            nz = acc0 != 0;
          }
          if (NO > 1 && lane + 32 < fr) {
            rowp[32 + lane] = acc1;
            nz = nz || acc1 != 0;
          }
          if (__any_sync(kFull, nz) && lane == 0) P.sflag_out[d] = 1;
        }
      }
    }
  }
  if (!LAST) {  // chunk tail prefix for k_coef_fixup (frame of the last vertex)
    if (lane < frame && (NO != 0 || lane < 16)) P.agg[c * P.E + lane] = acc0;
    if (NO > 1 && lane + 32 < frame) P.agg[c * P.E + 32 + lane] = acc1;
  }
  if (!P.chunk_ctr) break;
  int64_t nx = 0;
  if (lane == 0) nx = atomicAdd(P.chunk_ctr, 1) + nwarps;
  c = __shfl_sync(kFull, nx, 0);
  }
}

// Resident blocks per SM of a kernel at (threads, dynamic shared bytes),
// cached: the occupancy query is not free and runs once per launch otherwise.
int resident_blocks(const void* f, int threads, size_t smem) {
  static std::mutex mu;
  static std::vector<std::pair<std::pair<const void*, size_t>, int>> done;
  std::lock_guard<std::mutex> lk(mu);
  const auto key = std::make_pair(f, smem);
  for (auto& d : done)
    if (d.first == key) return d.second;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, f, threads, smem) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  done.emplace_back(key, per_sm);
  return per_sm;
}

// Opt a kernel into `bytes` of dynamic shared memory (raised only, per
// kernel and device).
void allow_smem(const void* f, size_t bytes) {
  static std::mutex mu;
  static std::vector<std::pair<std::pair<const void*, int>, size_t>> done;
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_pair(f, dev);
  std::lock_guard<std::mutex> lk(mu);
  for (auto& d : done)
    if (d.first == key) {
      if (bytes > d.second) {
        cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(bytes));
        d.second = bytes;
      }
      return;
    }
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
  done.emplace_back(key, bytes);
}

}  // namespace

void launch_coef_items(const CoefParams& p, cudaStream_t st) {
  if (p.g.C == 0) return;
  prof_begin(p.last ? "coef_arcs_last" : p.ell == 2 ? "coef_arcs_first" : "coef_arcs", st);
  const size_t smem = static_cast<size_t>(kIW) * p.warp_words * 8 + 256;
  const unsigned blocks = static_cast<unsigned>((p.g.C + kIW - 1) / kIW);
  // (every instantiation has the same signature, so a static inside the
  // generic lambda would be shared by all of them: keep the size per kernel)
  auto go = [&](auto kern) {
    allow_smem(reinterpret_cast<const void*>(kern), smem);
    kern<<<blocks, kIW * 32, smem, st>>>(p);
  };
  const bool first = p.ell == 2, last = p.last;
  const char* reg_env = std::getenv("TSV_ITEMS_REG");
  if (p.frame_max <= 64 && !(reg_env && std::strcmp(reg_env, "0") == 0)) {
    const int fmp = p.frame_max | 1;  // odd row stride: conflict-free 8-byte column reads
    const size_t rsm = static_cast<size_t>(kIW) * 32 * fmp * 8;
    auto go2 = [&](auto kern) {
      allow_smem(reinterpret_cast<const void*>(kern), rsm);
      unsigned nb = blocks;
      if (p.chunk_ctr) {  // persistent grid: every resident block slot once
        const int per_sm = resident_blocks(reinterpret_cast<const void*>(kern), kIW * 32, rsm);
        const unsigned cap = static_cast<unsigned>(p.sms * per_sm);
        if (cap < nb) nb = cap;
      }
      kern<<<nb, kIW * 32, rsm, st>>>(p, fmp);
    };
    const char* sp_env = std::getenv("TSV_WALK_SPLIT");
    const int no = p.frame_max > 32 ? 2
                   : (p.frame_max <= 16 && !(sp_env && sp_env[0] == '0')) ? 0 : 1;
    if (first && last)
      no == 2 ? go2(k_coef_items_reg<true, true, 2>)
              : no == 1 ? go2(k_coef_items_reg<true, true, 1>) : go2(k_coef_items_reg<true, true, 0>);
    else if (first)
      no == 2 ? go2(k_coef_items_reg<true, false, 2>)
              : no == 1 ? go2(k_coef_items_reg<true, false, 1>) : go2(k_coef_items_reg<true, false, 0>);
    else if (last)
      no == 2 ? go2(k_coef_items_reg<false, true, 2>)
              : no == 1 ? go2(k_coef_items_reg<false, true, 1>) : go2(k_coef_items_reg<false, true, 0>);
    else
      no == 2 ? go2(k_coef_items_reg<false, false, 2>)
              : no == 1 ? go2(k_coef_items_reg<false, false, 1>) : go2(k_coef_items_reg<false, false, 0>);
    prof_end(st);
    return;
  }
  // items of a single -> single arc: C(k-2, ell-2)
  const int64_t ss = static_cast<int64_t>(p.frame_single) * (p.ell - 1) / (p.k - 1);
  const bool deep = ss >= 32 || (p.frame_max == p.frame_multi && p.frame_multi >= 64);
  if (first && last)
    go(k_coef_items<true, true, 1>);
  else if (first)
    go(k_coef_items<true, false, 1>);
  else if (last)
    go(k_coef_items<false, true, 1>);
  else if (deep)
    go(k_coef_items<false, false, TSV_ITEMS_SUB>);
  else
    go(k_coef_items<false, false, 1>);
  prof_end(st);
}

}  // namespace tsv

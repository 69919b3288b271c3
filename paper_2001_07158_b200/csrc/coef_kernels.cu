// coef_kernels.cu -- the temporal sieve in coefficient (top-degree) form.
//
// For a fixed graph and seed, S_l(A) of every run is a polynomial in the
// bits a_1..a_k of the sieve point A: z_u(A) = XOR_j a_j z_{u,j} is linear,
// y and XOR are constants and sums.  At 0/1 points it equals its multilinear
// reduction, and over GF(2) the sum over all 2^k points of a multilinear
// monomial a_T is 2^(k-|T|) copies of it: nonzero only for T = [k].  So the
// reference's accumulator acc[u] = XOR_A P[u][k][max_ts](A)
// (/root/reference/proj/core/src/sieve.cpp:294-306) is the coefficient of
// a_1..a_k in the level-k polynomial, and only the degree-l part of level l
// can reach it (S_l has degree <= l; each level raises the degree by at most
// one).  The degree-l part of S_l[run] is indexed by the l-subsets T of [k]:
//
//   U_l[run][T'] = XOR_{arcs a of head up to run} y(e_a, l-1) * S_{l-1}[src_a][T']
//   S_l[run][T]  = XOR_{j in T} z_{head,j} * U_l[run][T \ {j}]     (|T| = l)
//
// with S_1[v][{j}] = z_{v,j}.  Bit-identical accumulators for C(k, l-1)
// products per arc at level l instead of 2^k (C2: 62 vs 320 per arc over
// all levels).  The engine runs two kernels per level:
//
//   k_coef_arcs   one pass over the vertex-major arc stream (layout.hpp):
//                 products y * S_{l-1}[src] for the C(k,l-1) entries of
//                 each arc (a lane group per arc, entries across its lanes),
//                 segmented prefix XOR per head, U stored at the ends of runs
//                 some arc of the next level reads (state slots); level k
//                 XORs each vertex piece's U into ulast[head].
//   k_coef_ztrans S_l[slot][T] from U[slot] (l products per entry, one
//                 thread per (slot, T)); k_coef_readout applies the same map
//                 to ulast for level k and XORs into acc.
//
// Subsets of a level are numbered in colex order (= increasing bit mask):
// entry e of level 1 is {e}, so S_1 rows are the z_{u,.} rows as stored.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "coef.hpp"
#include "gf_device.cuh"
#include "layout.hpp"

namespace tsv {
namespace {

constexpr int kCoefWarps = 4;
constexpr unsigned kFull = 0xffffffffu;
constexpr uint32_t kLive = 2u;  // staged: the arc's products can be nonzero
constexpr uint32_t kPush = 4u;  // staged: store / flush this arc's prefix

__device__ __forceinline__ bool has_color_c(const int32_t* __restrict__ colors, int32_t x,
                                            int32_t c, int32_t wild) {
  return c == wild || __ldg(colors + x) == c;
}

// One half-warp's GfTable window (16 lanes build a whole table).
__device__ __forceinline__ void build_window16_c(uint64_t* tab, uint64_t y, int w) {
  const uint32_t s = 4u * static_cast<uint32_t>(w);
  uint64_t h, lo;
  asm("shr.b64 %0, %1, %2;" : "=l"(h) : "l"(y), "r"(64u - s));
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

// One level's arc pass over the entry slice [e0, e0 + ne) of the C(k, l-1)
// input entries.  A warp owns a chunk; G = 32/LG arcs are in flight per step,
// one per group of LG lanes, and lane li of a group holds entries
// e0 + li + LG*p (p < PPT).  The y product: LG = 32 -> a warp table
// (GfTable), LG = 16 -> a half-warp table per arc, LG <= 8 -> general
// product with y split once per arc in shared memory.
template <int LG, int PPT, bool FIRST, bool LAST>
__global__ void __launch_bounds__(kCoefWarps * 32)
    k_coef_arcs(const CoefParams P) {
  constexpr int G = 32 / LG;
  constexpr bool kWarpTab = LG == 32;
  constexpr bool kHalfTab = LG == 16;
  constexpr bool kGeneral = LG <= 8;
  __shared__ uint32_t s_ys[kGeneral ? kCoefWarps : 1][12][32];
  __shared__ uint64_t s_yraw[kCoefWarps][32];
  __shared__ int32_t s_src[kCoefWarps][32];
  __shared__ uint32_t s_meta[kCoefWarps][32];
  __shared__ int32_t s_slot[kCoefWarps][32];
  __shared__ int32_t s_head[kCoefWarps][32];
  __shared__ int8_t s_idx[kCoefWarps][32];
  __shared__ int8_t s_hd[kCoefWarps][32];
  __shared__ __align__(256) uint64_t s_tab[kGeneral ? 1 : kCoefWarps][kHalfTab ? 2 : 1]
                                          [GfTable::kWords];

  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t c = static_cast<int64_t>(blockIdx.x) * kCoefWarps + wib;
  if (c >= P.g.C) return;  // warp-uniform
  const int g = lane / LG, li = lane % LG;
  bool ev[PPT];  // entry li + LG*p of the slice exists
#pragma unroll
  for (int p = 0; p < PPT; ++p) ev[p] = li + LG * p < P.ne;
  const int64_t E = P.E;

  const uint64_t pre = draw_prefix(P.seed, kRoleEdgeY);
  const uint64_t yb = static_cast<uint64_t>(P.ell - 1) + 0x165667b19e3779f9ull;
  const int64_t a0 = P.g.chunk_arc[c], a1 = P.g.chunk_arc[c + 1];
  int32_t run_ctr = P.g.chunk_run[c];
  const int last_lane = (G - 1) * LG + li;
  uint64_t carry[PPT];
#pragma unroll
  for (int p = 0; p < PPT; ++p) carry[p] = 0;

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
    bool live = lane < nb && sidx >= 0;
    if (FIRST) live = live && (P.anchor_source < 0 || sidx == P.anchor_source);
    if (LAST) live = live && __ldg(P.g.run_ts + myrun) <= P.max_ts;
    if (P.vc_color && live) {
      const int32_t tl = FIRST ? sidx : __ldg(P.g.arc_tail + base + lane);
      live = tl >= 0 && has_color_c(P.vc_color, tl, P.vc_tail, P.vc_wild) &&
             has_color_c(P.vc_color, head, P.vc_head, P.vc_wild);
    }
    // zero states: a head without shades has S = 0 (its products and stores
    // are never read), and a source whose state row is all zero adds nothing
    const bool hz = lane < nb && P.vsh && __ldg(P.vsh + head) == -1;
    if (live && P.vsh)
      live = !hz && (FIRST ? __ldg(P.vsh + sidx) != -1 : __ldg(P.sflag + sidx) != 0);
    // a single-shade tail's state is stored without its v (k_coef_zshift):
    // the arc multiplies by y * v_tail instead
    int8_t td = -2;  // the source's shade when it keeps its U row
    if (!FIRST && live && P.vsv) {
      const int32_t tl = __ldg(P.g.arc_tail + base + lane);
      td = __ldg(P.vsh + tl);
      if (td >= 0) y = gf_mul(y, __ldg(P.vsv + tl));
    }
    s_yraw[wib][lane] = y;
    if (kGeneral) {
      const KSplit ks = ksplit(y);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        s_ys[kGeneral ? wib : 0][j][lane] = ks.l.c[j];
        s_ys[kGeneral ? wib : 0][4 + j][lane] = ks.h.c[j];
        s_ys[kGeneral ? wib : 0][8 + j][lane] = ks.m.c[j];
      }
    }
    bool push;
    int32_t slot = -1;
    if (LAST) {  // last arc of its vertex within this chunk: flush the piece
      const bool chunk_end = base + lane + 1 >= a1;
      uint32_t nmeta = __shfl_down_sync(kFull, meta, 1);
      if (lane == 31 && !chunk_end) nmeta = __ldg(P.g.arc_meta + base + 32);
      push = lane < nb && !hz && (chunk_end || (nmeta & kVStart));
    } else {
      slot = (lane < nb && !hz && (meta & kRunEnd)) ? __ldg(P.g.run_slot + myrun) : -1;
      push = slot >= 0;
    }
    s_hd[wib][lane] = td;
    s_src[wib][lane] = sidx;
    s_meta[wib][lane] = (meta & (kVStart | kRunEnd)) | (live ? kLive : 0u) | (push ? kPush : 0u);
    s_slot[wib][lane] = slot;
    s_head[wib][lane] = head;
    run_ctr += __popc(ends);
    // only arcs with a product, a store or a prefix reset are stepped through
    const unsigned actm = __ballot_sync(kFull, lane < nb && (live || push || (meta & kVStart)));
    const int nact = __popc(actm);
    if ((actm >> lane) & 1u) s_idx[wib][__popc(actm & ((1u << lane) - 1u))] = lane;
    __syncwarp();

    auto fetch = [&](int q, uint64_t (&out)[PPT]) {
#pragma unroll
      for (int p = 0; p < PPT; ++p) out[p] = 0;
      const int i = q < nact ? s_idx[wib][q] : 0;
      if (q < nact && (s_meta[wib][i] & kLive)) {
        const int64_t src = s_src[wib][i];
        if (FIRST) {
          const uint64_t* row = P.zj + src * P.k + P.e0;
#pragma unroll
          for (int p = 0; p < PPT; ++p)
            if (ev[p]) out[p] = __ldg(row + li + LG * p);
        } else {
          const uint64_t* row = P.s_prev + src * P.rs_in;
          const int td = s_hd[wib][i];
          if (td >= 0) {  // U row of a single-shade source
            const int32_t* sm = P.smap + td * E + P.e0;
#pragma unroll
            for (int p = 0; p < PPT; ++p)
              if (ev[p]) {
                const int in = __ldg(sm + li + LG * p);
                if (in >= 0) out[p] = __ldg(row + in);
              }
          } else {
#pragma unroll
            for (int p = 0; p < PPT; ++p)
              if (ev[p]) out[p] = __ldg(row + P.e0 + li + LG * p);
          }
        }
      }
    };
    uint64_t nxt[PPT];
    fetch(g, nxt);
    const int steps = (nact + G - 1) / G;
#pragma unroll 1
    for (int s = 0; s < steps; ++s) {
      uint64_t v[PPT];
#pragma unroll
      for (int p = 0; p < PPT; ++p) v[p] = nxt[p];
      if (s + 1 < steps) fetch((s + 1) * G + g, nxt);
      const bool act = s * G + g < nact;
      const int i = act ? s_idx[wib][s * G + g] : 0;
      const uint32_t mt = act ? s_meta[wib][i] : 0u;
      const bool lv = (mt & kLive) != 0;
      if (__any_sync(kFull, lv)) {
        const int ia = act ? i : 0;
        if (kWarpTab) {
          GfTable T{s_tab[kGeneral ? 0 : wib][0]};
          __syncwarp();
          T.build(s_yraw[wib][ia], lane);
          __syncwarp();
#pragma unroll
          for (int p = 0; p < PPT; ++p) v[p] = lv ? T.mul(v[p]) : 0ull;
        } else if (kHalfTab) {
          uint64_t* tab = s_tab[kGeneral ? 0 : wib][kHalfTab ? g : 0];
          __syncwarp();
          build_window16_c(tab, s_yraw[wib][ia], li);
          __syncwarp();
#pragma unroll
          for (int p = 0; p < PPT; ++p) v[p] = lv ? GfTable{tab}.mul(v[p]) : 0ull;
        } else {
          KSplit ys;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            ys.l.c[j] = s_ys[kGeneral ? wib : 0][j][ia];
            ys.h.c[j] = s_ys[kGeneral ? wib : 0][4 + j][ia];
            ys.m.c[j] = s_ys[kGeneral ? wib : 0][8 + j][ia];
          }
#pragma unroll
          for (int p = 0; p < PPT; ++p) v[p] = lv ? gf_mul_presplit(ys, v[p]) : 0ull;
        }
      } else {
#pragma unroll
        for (int p = 0; p < PPT; ++p) v[p] = 0;
      }
      // segmented inclusive XOR-scan over the G groups (vertex starts cut it)
      bool f = (mt & kVStart) != 0;
      if (G > 1) {
#pragma unroll
        for (int d = 1; d < G; d <<= 1) {
          const bool fo = __shfl_up_sync(kFull, f, d * LG);
#pragma unroll
          for (int p = 0; p < PPT; ++p) {
            const uint64_t vo = __shfl_up_sync(kFull, v[p], d * LG);
            if (g >= d && !f) v[p] ^= vo;
          }
          if (g >= d) f = f || fo;
        }
      }
#pragma unroll
      for (int p = 0; p < PPT; ++p) {
        if (!f) v[p] ^= carry[p];
        carry[p] = (G > 1) ? __shfl_sync(kFull, v[p], last_lane) : v[p];
      }
      if (LAST) {
        if (mt & kPush) {
          const int64_t row = static_cast<int64_t>(s_head[wib][i]) * E + P.e0;
#pragma unroll
          for (int p = 0; p < PPT; ++p)
            if (ev[p] && v[p])
              atomicXor(reinterpret_cast<unsigned long long*>(P.ulast + row + li + LG * p),
                        static_cast<unsigned long long>(v[p]));
        }
      } else {
        bool nzr = false;
        if (mt & kPush) {
          const int64_t row = static_cast<int64_t>(s_slot[wib][i]) * P.rs_out + P.e0;
#pragma unroll
          for (int p = 0; p < PPT; ++p)
            if (ev[p]) {
              P.ubuf[row + li + LG * p] = v[p];
              nzr = nzr || v[p] != 0;
            }
        }
        const unsigned bm = __ballot_sync(kFull, nzr);
        const unsigned gm = LG == 32 ? kFull : ((1u << LG) - 1u) << (g * LG);
        if ((mt & kPush) && li == 0 && (bm & gm)) P.sflag_out[s_slot[wib][i]] = 1;
      }
    }
    __syncwarp();
  }
  if (!LAST && g == 0) {
#pragma unroll
    for (int p = 0; p < PPT; ++p)
      if (ev[p]) P.agg[c * E + P.e0 + li + LG * p] = carry[p];
  }
}

// A chunk whose first arc continues vertex h (split across chunks) started
// h's prefix from zero: its runs of h receive the XOR of the tail aggregates
// of the preceding chunks back to the one where h starts (U space, before
// the z map, so no product is needed).
__global__ void k_coef_fixup(const CoefParams P) {
  __shared__ uint64_t carry_s[kZAcc];  // E = C(k, l-1) <= kZAcc (k <= 12)
  __shared__ int any;
  const int32_t c = P.g.carry_list[blockIdx.x];
  const int32_t r0 = P.g.chunk_run[c];
  if (r0 >= P.g.R) return;
  const int32_t head = P.g.run_head[r0];
  const int32_t r1 = min(P.g.chunk_run[c + 1], P.g.vtx_run_off[head + 1]);
  if (r0 >= r1) return;
  const int dh = P.vsh ? P.vsh[head] : -2;
  if (dh == -1) return;  // shadeless: rows never read
  // entries of the head's rows: its compact frame in the item-stream layout
  const int E = (P.frame_single && dh >= 0) ? P.frame_single : P.E;
  if (threadIdx.x == 0) any = 0;
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    uint64_t carry = 0;
    for (int64_t cc = c - 1;; --cc) {
      carry ^= P.agg[cc * P.E + e];
      if (!P.g.chunk_carry[cc] || P.g.run_head[P.g.chunk_run[cc]] != head) break;
    }
    carry_s[e] = carry;
    if (carry) any = 1;
  }
  __syncthreads();
  if (!any) return;
  // every (run, entry) of the piece in parallel (hub pieces hold ~1e3 runs)
  const int n = (r1 - r0) * E;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int q = i / E, e = i - q * E;
    const uint64_t carry = carry_s[e];
    if (!carry) continue;
    const int32_t slot = P.g.run_slot[r0 + q];
    if (slot >= 0) {
      P.ubuf[static_cast<int64_t>(slot) * P.rs_out + e] ^= carry;
      P.sflag_out[slot] = 1;
    }
  }
}

// S_l[slot][T] = XOR_{j in T} z_{h,j} * U[slot][T - {j}] for the slots of
// heads with several shades (the others are stored mapped by k_coef_arcs),
// in place: the U row (C(k, l-1) entries) is replaced by the S row
// (C(k, l) entries) at the same row (stride rs).  Each z_{h,j} multiplies
// C(k-1, l-1) entries of every slot of head h, so a warp takes a window of
// 32 consecutive slots (slot_head is nondecreasing: slots are ranks in
// vertex-major run order) and, per head segment of the window and per j
// with z_{h,j} != 0, builds the table of z_{h,j} (GfTable, all 32 lanes)
// and spreads the (slot, T' without j) items of the segment over its lanes,
// XORing z_{h,j} * U[T'] into output T' + {j} of a shared-memory
// accumulator.  The multiplier is warp-uniform, so every lookup of a warp
// hits one 128-byte table window (conflict-free); within one j the outputs
// are distinct, so the accumulator needs no atomics.  A sub-batch's U rows
// are all read before its S rows are written.
constexpr int kZWarps = 4;
constexpr int kZWarpWords = GfTable::kWords + kZAcc;
__global__ void __launch_bounds__(kZWarps * 32)
    k_coef_ztrans_tab(int64_t S, int F, int K1, const int32_t* __restrict__ slot_head,
                      const uint64_t* __restrict__ zj, int k, uint64_t* rows, int rs,
                      const int2* __restrict__ jpairs, const int8_t* __restrict__ vsh,
                      uint8_t* __restrict__ sflag) {
  __shared__ __align__(256) uint64_t sm[kZWarps][kZWarpWords];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  uint64_t* const tab = sm[wib];
  uint64_t* const acc = sm[wib] + GfTable::kWords;
  GfTable T{tab};
  const int qmax = kZAcc / F < 32 ? kZAcc / F : 32;  // slots per sub-batch (F <= kZAcc)
  const float invK1 = 1.0f / static_cast<float>(K1);
  const float invF = 1.0f / static_cast<float>(F);
  const int64_t nwin = (S + 31) / 32;
  for (int64_t w = static_cast<int64_t>(blockIdx.x) * kZWarps + wib; w < nwin;
       w += static_cast<int64_t>(gridDim.x) * kZWarps) {
    const int64_t w0 = w * 32;
    const int nsl = static_cast<int>(S - w0 < 32 ? S - w0 : 32);
    const int32_t myh = lane < nsl ? __ldg(slot_head + w0 + lane) : -1;
    const int32_t prevh = __shfl_up_sync(kFull, myh, 1);
    unsigned starts = __ballot_sync(kFull, lane < nsl && (lane == 0 || myh != prevh));
    while (starts) {
      const int a = __ffs(starts) - 1;
      starts &= starts - 1;
      const int b = starts ? __ffs(starts) - 1 : nsl;
      const int32_t h = __shfl_sync(kFull, myh, a);
      if (vsh && __ldg(vsh + h) != -2) continue;  // stored mapped by k_coef_arcs
      const uint64_t zl = lane < k ? __ldg(zj + static_cast<int64_t>(h) * k + lane) : 0ull;
      for (int q0 = a; q0 < b; q0 += qmax) {
        const int qb = b - q0 < qmax ? b - q0 : qmax;
        const int64_t s0 = w0 + q0;
        const uint64_t* U0 = rows + s0 * rs;
        __syncwarp();
        for (int i = lane; i < qb * F; i += 32) acc[i] = 0;
        const int items = qb * K1;
        for (int j = 0; j < k; ++j) {
          const uint64_t zv = __shfl_sync(kFull, zl, j);
          if (zv == 0) continue;  // warp-uniform: shade j not in S(h)
          __syncwarp();
          T.build(zv, lane);
          __syncwarp();
          const int2* jp = jpairs + j * K1;
          for (int it = lane; it < items; it += 32) {
            int qq = __float2int_rz(static_cast<float>(it) * invK1);
            if ((qq + 1) * K1 <= it) ++qq;
            if (qq * K1 > it) --qq;
            const int2 p = __ldg(jp + (it - qq * K1));
            const uint64_t u = U0[static_cast<int64_t>(qq) * rs + p.x];
            if (u) acc[qq * F + p.y] ^= T.mul(u);
          }
        }
        __syncwarp();
        for (int i = lane; i < qb * F; i += 32) {
          int qq = __float2int_rz(static_cast<float>(i) * invF);
          if ((qq + 1) * F <= i) ++qq;
          if (qq * F > i) --qq;
          const uint64_t r = acc[i];
          rows[(s0 + qq) * rs + (i - qq * F)] = r;
          if (r) sflag[s0 + qq] = 1;
        }
      }
    }
  }
}

// Level k: acc[h] ^= scale * XOR_{c < k} z_{h, j_c} * ulast[h][in_c]
// (scale = det(W) in the shade basis, 1 for positional z).
__global__ void k_coef_readout(int32_t n, const uint64_t* __restrict__ zj, int k,
                               const uint64_t* __restrict__ ulast,
                               const int2* __restrict__ pairs, uint64_t scale,
                               const int8_t* __restrict__ vsh,
                               const uint64_t* __restrict__ vsv, uint64_t* __restrict__ acc) {
  const int64_t h = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (h >= n) return;
  const uint64_t* U = ulast + h * k;
  const uint64_t* z = zj + h * k;
  uint64_t r = 0;
  const int d = vsh ? __ldg(vsh + h) : -2;
  if (d == -1) return;
  if (d >= 0) {  // compact frame: the one entry [k] - {d}
    const uint64_t u = __ldg(U);
    if (u) r = gf_mul(__ldg(vsv + h), u);
  } else
  for (int cc = 0; cc < k; ++cc) {
    const int2 pr = __ldg(pairs + cc);
    const uint64_t u = __ldg(U + pr.x);
    if (u) r ^= gf_mul(__ldg(z + pr.y), u);
  }
  if (r && scale != 1) r = gf_mul(scale, r);
  if (r) acc[h] ^= r;
}

__global__ void k_vshade(int32_t n, int k, const uint64_t* __restrict__ rows,
                         int8_t* __restrict__ vsh, uint64_t* __restrict__ vsv) {
  const int64_t u = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (u >= n) return;
  int cnt = 0, d = -1;
  uint64_t v = 1;
  for (int j = 0; j < k; ++j) {
    const uint64_t x = __ldg(rows + u * k + j);
    if (x) ++cnt, d = j, v = x;
  }
  vsh[u] = static_cast<int8_t>(cnt == 0 ? -1 : cnt == 1 ? d : -2);
  vsv[u] = cnt == 1 ? v : 1ull;
}

__global__ void k_slot_head(int64_t R, const int32_t* __restrict__ run_slot,
                            const int32_t* __restrict__ run_head, int32_t* __restrict__ slot_head) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= R) return;
  const int32_t s = run_slot[r];
  if (s >= 0) slot_head[s] = run_head[r];
}


// Multi-shade rows (or every row with positional z) in a compact list of
// (slot, head), built once per evaluation: the direct z map below then runs
// over exactly the rows it transforms (C2: 1/8 of the state slots).
__global__ void k_multi_slots(int64_t R, const int32_t* __restrict__ run_slot,
                              const int32_t* __restrict__ run_head,
                              const int8_t* __restrict__ vsh, int2* __restrict__ list,
                              int32_t* __restrict__ count) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  int32_t s = -1, h = -1;
  if (r < R) {
    s = run_slot[r];
    if (s >= 0) {
      h = run_head[r];
      if (vsh && __ldg(vsh + h) != -2) s = -1;
    }
  }
  const unsigned m = __ballot_sync(kFull, s >= 0);
  if (!m) return;
  int base = 0;
  if (lane == __ffs(m) - 1) base = atomicAdd(count, __popc(m));
  base = __shfl_sync(kFull, base, __ffs(m) - 1);
  if (s >= 0) list[base + __popc(m & ((1u << lane) - 1u))] = make_int2(s, h);
}

// Direct z map of the listed rows, in place: S_l[slot][T] =
// XOR_{j in T} z_{head,j} * U_l[slot][T - {j}] (pairs of level l: for each
// l-subset T its l pairs (rank of T - {j}, j)).  A block takes a tile of
// rows, forms every entry of the tile in shared memory (one thread per
// (row, T), general products), then -- after all of the tile's U entries
// are read -- writes the tile back.  Rows whose U is zero (sflag clear) are
// skipped: their S is zero and no arc reads them (the arc kernels test the
// flag whenever zero skipping is on; sflag = nullptr transforms every row,
// as the vertex-ordered sieve's arcs read rows without the test).
constexpr int kZdThreads = 256;
constexpr int kZdWords = 2048;  // shared output words per tile
__global__ void __launch_bounds__(kZdThreads)
    k_coef_ztrans_direct(const int2* __restrict__ list, const int32_t* __restrict__ count,
                         int F, int l, int spt, const uint64_t* __restrict__ zj, int k,
                         uint64_t* rows, int rs, const int2* __restrict__ pairs,
                         const uint8_t* __restrict__ sflag) {
  __shared__ uint64_t out[kZdWords];
  __shared__ int2 tile[kZdWords / 2];  // F >= 2 below level k
  const int64_t nrows = *count;
  const int64_t ntiles = (nrows + spt - 1) / spt;
  const float invF = 1.0f / static_cast<float>(F);
  for (int64_t tl = blockIdx.x; tl < ntiles; tl += gridDim.x) {
    const int64_t r0 = tl * spt;
    const int nr = static_cast<int>(nrows - r0 < spt ? nrows - r0 : spt);
    for (int i = threadIdx.x; i < nr; i += kZdThreads) {
      int2 e = list[r0 + i];
      if (sflag && !sflag[e.x]) e.x = -1;
      tile[i] = e;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nr * F; i += kZdThreads) {
      int q = __float2int_rz(static_cast<float>(i) * invF);
      if ((q + 1) * F <= i) ++q;
      if (q * F > i) --q;
      const int2 e = tile[q];
      if (e.x < 0) continue;
      const int t = i - q * F;
      const uint64_t* U = rows + static_cast<int64_t>(e.x) * rs;
      const uint64_t* z = zj + static_cast<int64_t>(e.y) * k;
      uint64_t r = 0;
      for (int c = 0; c < l; ++c) {
        const int2 pr = __ldg(pairs + t * l + c);
        const uint64_t u = U[pr.x];
        const uint64_t zv = __ldg(z + pr.y);
        if (u && zv) r ^= gf_mul(zv, u);
      }
      out[i] = r;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nr * F; i += kZdThreads) {
      int q = __float2int_rz(static_cast<float>(i) * invF);
      if ((q + 1) * F <= i) ++q;
      if (q * F > i) --q;
      const int2 e = tile[q];
      if (e.x >= 0) rows[static_cast<int64_t>(e.x) * rs + (i - q * F)] = out[i];
    }
    __syncthreads();
  }
}

template <int LG, int PPT>
void arcs_dispatch(const CoefParams& p, cudaStream_t st) {
  const unsigned blocks = static_cast<unsigned>((p.g.C + kCoefWarps - 1) / kCoefWarps);
  const bool first = p.ell == 2, last = p.last;
  if (first && last)
    k_coef_arcs<LG, PPT, true, true><<<blocks, kCoefWarps * 32, 0, st>>>(p);
  else if (first)
    k_coef_arcs<LG, PPT, true, false><<<blocks, kCoefWarps * 32, 0, st>>>(p);
  else if (last)
    k_coef_arcs<LG, PPT, false, true><<<blocks, kCoefWarps * 32, 0, st>>>(p);
  else
    k_coef_arcs<LG, PPT, false, false><<<blocks, kCoefWarps * 32, 0, st>>>(p);
}

}  // namespace

CoefTables coef_tables(int k) {
  CoefTables t;
  t.k = k;
  std::vector<std::vector<int64_t>> C(static_cast<size_t>(k) + 1,
                                      std::vector<int64_t>(static_cast<size_t>(k) + 2, 0));
  for (int a = 0; a <= k; ++a) {
    C[a][0] = 1;
    for (int b = 1; b <= a; ++b) C[a][b] = C[a - 1][b - 1] + (b <= a - 1 ? C[a - 1][b] : 0);
  }
  t.count.resize(static_cast<size_t>(k) + 1);
  for (int l = 0; l <= k; ++l) t.count[l] = C[k][l];
  // colex rank of a subset: sum over its i-th smallest element x of C(x, i+1)
  auto rank = [&](uint64_t mask) {
    int64_t r = 0;
    int i = 0;
    for (int x = 0; x < k; ++x)
      if ((mask >> x) & 1ull) r += (x >= i + 1 ? C[x][i + 1] : 0), ++i;
    return r;
  };
  t.pairs.resize(static_cast<size_t>(k) + 1);
  for (int l = 2; l <= k; ++l) {
    std::vector<int2>& v = t.pairs[l];
    v.reserve(static_cast<size_t>(t.count[l] * l));
    uint64_t T = (1ull << l) - 1;  // l-subsets in increasing mask order (Gosper)
    const uint64_t end = 1ull << k;
    while (T < end) {
      for (int j = 0; j < k; ++j)
        if ((T >> j) & 1ull)
          v.push_back(make_int2(static_cast<int>(rank(T & ~(1ull << j))), j));
      const uint64_t cbit = T & (~T + 1), rr = T + cbit;
      T = (((rr ^ T) >> 2) / cbit) | rr;
    }
  }
  t.jpairs.resize(static_cast<size_t>(k) + 1);
  for (int l = 2; l <= k; ++l) {
    std::vector<std::vector<int2>> per(static_cast<size_t>(k));
    const std::vector<int2>& v = t.pairs[l];
    for (size_t i = 0; i < v.size(); ++i)  // output o = i / l, pair (in, j)
      per[v[i].y].push_back(make_int2(v[i].x, static_cast<int>(i / l)));
    for (int j = 0; j < k; ++j) {
      std::sort(per[j].begin(), per[j].end(),
                [](const int2& x, const int2& y) { return x.x < y.x; });
      t.jpairs[l].insert(t.jpairs[l].end(), per[j].begin(), per[j].end());
    }
  }
  t.smap.resize(static_cast<size_t>(k) + 1);
  for (int l = 2; l <= k; ++l) {
    const int64_t F = t.count[l];
    std::vector<int32_t>& m = t.smap[l];
    m.assign(static_cast<size_t>(k * F), -1);
    const std::vector<int2>& v = t.pairs[l];
    for (size_t i = 0; i < v.size(); ++i)  // output o = i / l, pair (in, j)
      m[static_cast<size_t>(v[i].y * F) + i / l] = v[i].x;
  }
  return t;
}

CoefItems coef_items(int k, int l) {
  // binomials and colex ranks (compact frame d: the bit d removed)
  int64_t C[33][33] = {};
  for (int a = 0; a <= 32; ++a) {
    C[a][0] = 1;
    for (int b = 1; b <= a; ++b) C[a][b] = C[a - 1][b - 1] + C[a - 1][b];
  }
  auto rank = [&](uint64_t mask) {
    int64_t r = 0;
    int i = 0;
    for (int x = 0; mask; ++x, mask >>= 1)
      if (mask & 1ull) r += C[x][i + 1], ++i;
    return static_cast<int32_t>(r);
  };
  auto squeeze = [](uint64_t mask, int d) {  // drop bit d
    const uint64_t lo = mask & ((1ull << d) - 1ull);
    return lo | ((mask >> (d + 1)) << d);
  };
  CoefItems t;
  const int K1 = k + 1;
  t.off.assign(static_cast<size_t>(K1 * K1), 0);
  t.cnt.assign(static_cast<size_t>(K1 * K1), 0);
  for (int tc = 0; tc <= k; ++tc)
    for (int hc = 0; hc <= k; ++hc) {
      t.off[tc * K1 + hc] = static_cast<int32_t>(t.items.size());
      if (tc < k && tc == hc) continue;  // same single shade twice: zero
      // U entries T of the head: (l-1)-subsets, in increasing mask order
      for (uint64_t T = (1ull << (l - 1)) - 1; T < (1ull << k);) {
        const bool ok = (tc == k || ((T >> tc) & 1ull)) && (hc == k || !((T >> hc) & 1ull));
        if (ok) {
          const int32_t in = tc == k ? rank(T) : rank(squeeze(T & ~(1ull << tc), tc));
          const int32_t out = hc == k ? rank(T) : rank(squeeze(T, hc));
          t.items.push_back(make_int2(in, out));
        }
        if (T == 0) break;
        const uint64_t cbit = T & (~T + 1), rr = T + cbit;
        T = (((rr ^ T) >> 2) / cbit) | rr;
      }
      t.cnt[tc * K1 + hc] = static_cast<int32_t>(t.items.size()) - t.off[tc * K1 + hc];
    }
  return t;
}

int coef_group_lanes(int ne) { return ne <= 4 ? 4 : ne <= 8 ? 8 : ne <= 16 ? 16 : 32; }

void launch_coef_arcs(const CoefParams& p, cudaStream_t st) {
  if (p.g.C == 0 || p.ne <= 0) return;
  prof_begin(p.last ? "coef_arcs_last" : p.ell == 2 ? "coef_arcs_first" : "coef_arcs", st);
  const int lg = coef_group_lanes(p.ne);
  if (lg == 4) {
    arcs_dispatch<4, 1>(p, st);
  } else if (lg == 8) {
    arcs_dispatch<8, 1>(p, st);
  } else if (lg == 16) {
    arcs_dispatch<16, 1>(p, st);
  } else if (p.ne <= 32) {
    arcs_dispatch<32, 1>(p, st);
  } else if (p.ne <= 64) {
    arcs_dispatch<32, 2>(p, st);
  } else {
    arcs_dispatch<32, 4>(p, st);
  }
  prof_end(st);
}

void launch_coef_fixup(const CoefParams& p, cudaStream_t st) {
  if (p.g.ncarry == 0) return;
  prof_begin("coef_fixup", st);
  k_coef_fixup<<<p.g.ncarry, 256, 0, st>>>(p);
  prof_end(st);
}

void launch_coef_ztrans(int64_t S, int F, int l, const int32_t* slot_head, const uint64_t* zj,
                        int k, int E, uint64_t* rows, int rs, const int2* jpairs,
                        const int8_t* vsh, uint8_t* sflag, int sm_count, cudaStream_t st) {
  (void)E;
  if (S == 0) return;
  prof_begin("coef_ztrans", st);
  static int per_sm = 0;
  if (!per_sm &&
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_coef_ztrans_tab, kZWarps * 32,
                                                    0) != cudaSuccess)
    per_sm = 1;
  const int K1 = static_cast<int>(static_cast<int64_t>(F) * l / k);  // C(k-1, l-1)
  const int64_t nwin = (S + 31) / 32;
  const int64_t want = (nwin + kZWarps - 1) / kZWarps;
  const int64_t cap = static_cast<int64_t>(sm_count) * (per_sm > 0 ? per_sm : 1);
  k_coef_ztrans_tab<<<static_cast<unsigned>(want < cap ? want : cap), kZWarps * 32, 0, st>>>(
      S, F, K1, slot_head, zj, k, rows, rs, jpairs, vsh, sflag);
  prof_end(st);
}

void launch_coef_readout(int32_t n, const uint64_t* zj, int k, const uint64_t* ulast,
                         const int2* pairs, uint64_t scale, const int8_t* vsh,
                         const uint64_t* vsv, uint64_t* acc, cudaStream_t st) {
  if (n == 0) return;
  prof_begin("coef_readout", st);
  k_coef_readout<<<(n + 255) / 256, 256, 0, st>>>(n, zj, k, ulast, pairs, scale, vsh, vsv, acc);
  prof_end(st);
}

void launch_vshade(int32_t n, int k, const uint64_t* rows, int8_t* vsh, uint64_t* vsv,
                   cudaStream_t st) {
  if (n == 0) return;
  k_vshade<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(n, k, rows, vsh, vsv);
}

void launch_slot_head(int64_t R, const int32_t* run_slot, const int32_t* run_head,
                      int32_t* slot_head, cudaStream_t st) {
  if (R == 0) return;
  k_slot_head<<<static_cast<unsigned>((R + 255) / 256), 256, 0, st>>>(R, run_slot, run_head,
                                                                       slot_head);
}

void launch_multi_slots(int64_t R, const int32_t* run_slot, const int32_t* run_head,
                        const int8_t* vsh, int2* list, int32_t* count, cudaStream_t st) {
  cudaMemsetAsync(count, 0, 4, st);
  if (R == 0) return;
  k_multi_slots<<<static_cast<unsigned>((R + 255) / 256), 256, 0, st>>>(R, run_slot, run_head,
                                                                         vsh, list, count);
}

void launch_coef_ztrans_direct(int64_t S, int F, int l, const int2* list, const int32_t* count,
                               const uint64_t* zj, int k, uint64_t* rows, int rs,
                               const int2* pairs, const uint8_t* sflag, int sm_count,
                               int64_t rows_hint, cudaStream_t st) {
  if (S == 0) return;
  prof_begin("coef_ztrans", st);
  // rows per tile: as many as the shared tile holds, but few enough that the
  // expected rows (rows_hint) still give every SM ~8 blocks -- C2 lists a
  // few 10^4 rows (latency-bound, dependent gathers), C5 every slot
  const int64_t want = std::max<int64_t>(1, rows_hint / (static_cast<int64_t>(sm_count) * 8));
  const int spt = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(kZdWords / F, want)));
  static int per_sm = 0;
  if (!per_sm && cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_coef_ztrans_direct,
                                                               kZdThreads, 0) != cudaSuccess)
    per_sm = 1;
  const int64_t tiles = (S + spt - 1) / spt;  // upper bound (the list is <= S)
  const int64_t cap = static_cast<int64_t>(sm_count) * (per_sm > 0 ? per_sm : 1);
  k_coef_ztrans_direct<<<static_cast<unsigned>(tiles < cap ? tiles : cap), kZdThreads, 0, st>>>(
      list, count, F, l, spt, zj, k, rows, rs, pairs, sflag);
  prof_end(st);
}

}  // namespace tsv

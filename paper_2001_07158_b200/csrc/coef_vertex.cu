// coef_vertex.cu -- the coefficient engine (coef_kernels.cu) in VERTEX-LANE
// form, for the case the BASELINE headline runs: every vertex carries several
// shades (k-TempPath: all k of them), small k, bounded in-degree (C5: n=1e8,
// m=1e9, k=5).
//
// Same algebra as coef_kernels.cu (derivation at its top):
//
//   U_l[run][T'] = XOR_{arcs a of head up to run} y(e_a, l-1) * S_{l-1}[src_a][T']
//   S_l[run][T]  = XOR_{j in T} z_{head,j} * U_l[run][T \ {j}]
//
// but organised for instruction count, not for arc parallelism:
//
//  * one LANE owns one head vertex and walks its arcs in time order, so the
//    per-vertex prefix XOR is a register accumulation -- no segmented scan,
//    no shuffles, no chunk carry fix-up, no per-arc staging;
//  * lanes of a warp take vertices of equal in-degree (a work list sorted by
//    arc count, built once per graph), so they step together;
//  * the arc product y * x multiplies by the arc's y split once (Karatsuba
//    holes, gf_device.cuh) and the products of a run accumulate UNREDUCED
//    (128-bit, class-masked): one reduction per referenced run end instead of
//    one per product;
//  * the z map S = z_h ^ U is fused: a referenced run end pushes its U row to
//    a per-warp shared-memory queue; whenever 32 rows are queued, every lane
//    maps one row (z_{h,j} split once per j, L products per output summed
//    unreduced, one reduction per output) and stores the S row -- the rows
//    never make a round trip through HBM as U, and no lane idles while
//    others map;
//  * level k is fused with the readout: acc[h] ^= det(W) * XOR_j z_{h,j} *
//    U_k[h][[k] - {j}] from the lane's own accumulator (no ulast buffer).
//
// Reads per live arc: its metadata and one row of C(k, l-1) words.  Writes:
// one row of C(k, l) words per referenced run.  Bit-identical to the other
// engines (tests/test_gpu_parity.py, tests/test_gpu_full.py).
#include <cuda_runtime.h>

#include <cub/cub.cuh>

#include <climits>
#include <cstdint>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

#include "coef.hpp"
#include "gf_device.cuh"
#include "layout.hpp"

// z map form: 2 = paired (E + F products per row instead of L * F, below),
// 0 = direct sums (measured at C5 x0.1: 70.2 ms -> 68.1 ms per evaluation;
// fully unrolled pairing was slower, 87 ms: register spills)
#ifndef TSV_ZPAIR
#define TSV_ZPAIR 2
#endif
// resident blocks per SM the register budget is sized for (1: unbounded;
// capping at 8 two-warp blocks spilled and ran slower)
// products interleaved per loop trip (arc products / z map); 1 = rolled
#ifndef TSV_VUNROLL
#define TSV_VUNROLL 1
#endif
#ifndef TSV_ZUNROLL
#define TSV_ZUNROLL 1
#endif
#ifndef TSV_VMINB
#define TSV_VMINB 7
#endif
// arc products y * row through the lane table (gf_device.cuh LaneTable: the
// arc's y multiplies C(k, l-1) entries, the table build is paid once per
// arc; measured 1.96e11 products/s against 1.18e11 for the holes product);
// 0 = holes + Karatsuba as in the z map
#ifndef TSV_VTABLE
#define TSV_VTABLE 1
#endif
// the lane table serves levels with at least this many input entries
#ifndef TSV_VTABLE_MINE
#define TSV_VTABLE_MINE 1
#endif

namespace tsv {
namespace {

constexpr unsigned kFullV = 0xffffffffu;
#ifndef TSV_VWARPS
#define TSV_VWARPS 2
#endif
constexpr int kVWarps = TSV_VWARPS;   // warps per block
constexpr int kQCap = 64;    // queued rows per warp (ring)

// Row stride of level l's state rows: C(k, l) words padded to a multiple of
// four (32 bytes, one DRAM sector) when TSV_VPAD, so that every row starts
// on a sector and a row write never shares a sector with a neighbor row.
#ifndef TSV_VPAD
#define TSV_VPAD 0
#endif
__host__ __device__ constexpr int vpad(int w) { return TSV_VPAD ? (w + 3) & ~3 : w; }
constexpr int kVUnroll = TSV_VUNROLL, kZUnroll = TSV_ZUNROLL;

__host__ __device__ constexpr int binom_c(int n, int r) {
  if (r < 0 || r > n) return 0;
  int v = 1;
  for (int i = 0; i < r; ++i) v = v * (n - i) / (i + 1);
  return v;
}

// Colex rank of a subset mask (the order of CoefTables: increasing mask
// within a level): sum over its i-th smallest element x of C(x, i+1).
__host__ __device__ constexpr int colex_rank(unsigned mask) {
  int r = 0, i = 0;
  for (int x = 0; x < 32; ++x)
    if ((mask >> x) & 1u) {
      r += binom_c(x, i + 1);
      ++i;
    }
  return r;
}

// For the l-subsets T of [k] in colex order: T's mask, and for each j in T
// the rank of T - {j} among the (l-1)-subsets.
template <int K, int L>
struct SubsetTab {
  static constexpr int F = binom_c(K, L);
  unsigned mask[F > 0 ? F : 1] = {};
  int less[F > 0 ? F : 1][K] = {};  // less[o][j] = rank(T_o - {j}) if j in T_o, else -1
  constexpr SubsetTab() {
    int o = 0;
    for (unsigned T = 0; T < (1u << K); ++T) {
      int pc = 0;
      for (int x = 0; x < K; ++x) pc += (T >> x) & 1u;
      if (pc != L) continue;
      mask[o] = T;
      for (int j = 0; j < K; ++j) less[o][j] = ((T >> j) & 1u) ? colex_rank(T & ~(1u << j)) : -1;
      ++o;
    }
  }
};

// 128-bit unreduced carry-less product accumulation (class-masked).
__device__ __forceinline__ void clmul_acc(const KSplit& a, uint64_t b, u128& acc) {
  const u128 p = clmul64_kara_s(a, ksplit(b));
  acc.lo ^= p.lo;
  acc.hi ^= p.hi;
}

// Reduction with ALU shifts (the FMA pipe carries the wide multiplies).
__device__ __forceinline__ uint64_t gf_reduce_alu(u128 p) {
  const uint64_t h = p.hi;
  const uint64_t over = (h >> 60) ^ (h >> 61) ^ (h >> 63);  // x^64.. terms of the first fold
  const uint64_t f1 = h ^ (h << 1) ^ (h << 3) ^ (h << 4);
  return p.lo ^ f1 ^ over ^ (over << 1) ^ (over << 3) ^ (over << 4);
}

struct VertArgs {
  CoefParams P;              // graph, seed, levels, rows (s_prev, ubuf), max_ts, anchor
  const int32_t* wl_head;    // work list sorted by arc count (descending)
  const int64_t* wl_start;   // first arc of the vertex
  const int32_t* wl_count;   // arcs of the vertex
  int64_t nv;                // vertices in the list
  uint64_t det;              // det(W) of the shade basis (readout)
  uint64_t* acc;             // level k: per-vertex accumulators (XORed into)
  // peer stores (multi-GPU): the readers of every state slot
  // (one byte per slot, own bit cleared by self_clear) and the ranks' level
  // buffers as mapped on this device; rmask == nullptr: local rows only
  const unsigned int* rmask;
  uint64_t* peer[8];
  unsigned self_clear;
};

// Row loads allocate in L1 (TSV_VROW_L1, default): a row spans two to four
// 32-byte sectors and its entry loads merge there; without allocation every
// entry load is its own L2 request (measured: level k 5.7 -> 9.2 ms at C5
// x0.1).
#ifndef TSV_VROW_L1
#define TSV_VROW_L1 1
#endif
__device__ __forceinline__ uint64_t ld_row64(const uint64_t* p) {
  uint64_t v;
#if TSV_VROW_L1
  asm volatile("ld.global.nc.u64 %0, [%1];" : "=l"(v) : "l"(p));
#else
  asm volatile("ld.global.nc.L1::no_allocate.u64 %0, [%1];" : "=l"(v) : "l"(p));
#endif
  return v;
}
__device__ __forceinline__ void ld_row128(const uint64_t* p, uint64_t& a, uint64_t& b) {
#if TSV_VROW_L1
  asm volatile("ld.global.nc.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p));
#else
  asm volatile("ld.global.nc.L1::no_allocate.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p));
#endif
}

// Per-warp shared state.  Lane-minor layouts ([entry][slot]) keep every
// access conflict-free.  The lane's running prefix U and the current / next
// source rows live in registers; the paired z map's W row and the lane
// table share the warp's scratch block (the table is dead during a flush).
template <int E, int F, int L, bool LAST>
struct VertSmem {
  uint64_t q[LAST ? 1 : E][kQCap];      // queued U rows (ring)
  int32_t q_slot[kQCap], q_head[kQCap];
  uint8_t pin[F > 0 ? F : 1][L], pj[F > 0 ? F : 1][L];  // output o: (rank of T_o - {j}, j) pairs
  uint8_t pmask[E];                     // input entry P's subset mask (paired z map)
  uint8_t pmem[E][L > 1 ? L - 1 : 1];   // the members j of P, ascending
};

// scratch bytes per warp: the lane table (4 KB, 4 KB aligned) or, without
// it, the W rows of the paired z map
template <int E, bool TAB>
__host__ __device__ constexpr unsigned vert_scratch() {
  return TAB ? 4096u : static_cast<unsigned>(E + 8) * 256u;  // W rows + the row's z_j
}

template <int K, int L>
__host__ __device__ constexpr bool vert_uses_table() {
  return TSV_VTABLE && binom_c(K, L - 1) >= TSV_VTABLE_MINE;
}

template <int K, int L, bool FIRST, bool LAST>
__global__ void __launch_bounds__(kVWarps * 32, TSV_VMINB) k_coef_vertex(const VertArgs A) {
  constexpr int E = binom_c(K, L - 1);  // input entries (row of level L-1)
  constexpr int F = binom_c(K, L);      // output entries
  constexpr bool kTab = vert_uses_table<K, L>();
  // the paired z map pays E + F products against L * F
  constexpr bool kZPairOk = !LAST && E + F < L * F;
  using Sm = VertSmem<E, F, L, LAST>;
  const CoefParams& P = A.P;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  // dynamic shared memory: the warps' scratch blocks (4 KB aligned in the
  // shared window when they hold lane tables), then their VertSmem blocks
  extern __shared__ __align__(16) uint8_t vsm_raw[];
  const uint32_t raw_s = static_cast<uint32_t>(__cvta_generic_to_shared(vsm_raw));
  const uint32_t scr_s = kTab ? (raw_s + 4095u) & ~4095u : raw_s;
  constexpr unsigned kScr = vert_scratch<E, kTab>();
  uint8_t* const scr_g = vsm_raw + (scr_s - raw_s);
  Sm& S = reinterpret_cast<Sm*>(scr_g + kScr * kVWarps)[wib];
  // W[p][lane] of the paired z map: entries c = p + 1 of the lane's table
  // column (entry 0 stays the table's zero)
  uint64_t* const wrow = reinterpret_cast<uint64_t*>(scr_g + kScr * wib) + (kTab ? 32 : 0) + lane;
  LaneTable LT;
  if (kTab) LT.init(scr_s + kScr * wib, lane);
  if (!LAST && lane == 0) {  // output pairs of the z map (colex order, coef_tables)
    constexpr SubsetTab<K, L> TL{};
    constexpr SubsetTab<K, L - 1> TP{};
    for (int p = 0; p < E; ++p) {
      S.pmask[p] = static_cast<uint8_t>(TP.mask[p]);
      int c = 0;
      for (int j = 0; j < K; ++j)
        if ((TP.mask[p] >> j) & 1u) S.pmem[p][c++] = static_cast<uint8_t>(j);
    }
    for (int o = 0; o < F; ++o) {
      int c = 0;
      for (int j = 0; j < K; ++j)
        if (TL.less[o][j] >= 0) {
          S.pin[o][c] = static_cast<uint8_t>(TL.less[o][j]);
          S.pj[o][c] = static_cast<uint8_t>(j);
          ++c;
        }
    }
  }
  const int64_t task = static_cast<int64_t>(blockIdx.x) * kVWarps + wib;
  const int64_t idx = task * 32 + lane;
  if (task * 32 >= A.nv) return;  // warp-uniform
  const bool act = idx < A.nv;
  const int32_t h = act ? __ldg(A.wl_head + idx) : 0;
  const int64_t a0 = act ? __ldg(A.wl_start + idx) : 0;
  const int cnt = act ? __ldg(A.wl_count + idx) : 0;
  int32_t run = act ? __ldg(P.g.vtx_run_off + h) : 0;
  const int steps = __reduce_max_sync(kFullV, cnt);
  const uint64_t pre = draw_prefix(P.seed, kRoleEdgeY);
  const uint64_t yb = static_cast<uint64_t>(L - 1) + 0x165667b19e3779f9ull;
  const uint64_t* __restrict__ rows = FIRST ? P.zj : P.s_prev;
  uint64_t u[E];  // the lane's running prefix U_L
#pragma unroll
  for (int e = 0; e < E; ++e) u[e] = 0;
  int qh = 0, qn = 0;  // ring head, queued count (warp-uniform)

  // z map of `take` queued rows (one per lane), stored as S rows of F words:
  // S[T] = XOR_{j in T} z_j * U[T - {j}], the L products of an output summed
  // in raw class form (gf_device.cuh ClassAcc): one Karatsuba combine, one
  // class mask and one reduction per output
  auto flush = [&](int take) {
    __syncwarp();
    if (lane < take) {
      const int qi = (qh + lane) & (kQCap - 1);
      const int32_t hd = S.q_head[qi];
      uint64_t z[K];
#pragma unroll
      for (int j = 0; j < K; ++j) z[j] = __ldg(P.zj + static_cast<int64_t>(hd) * K + j);
      const int64_t out_off = static_cast<int64_t>(S.q_slot[qi]) * vpad(F);
      uint64_t* out = P.ubuf + out_off;
      // the other ranks that read this row get it now (NVLink peer stores)
      unsigned pm = 0;
      if (A.rmask)
        pm = (__ldg(A.rmask + (S.q_slot[qi] >> 2)) >> (8 * (S.q_slot[qi] & 3))) & A.self_clear;
      auto put = [&](int o, uint64_t v) {
        out[o] = v;
        for (unsigned m = pm; m; m &= m - 1) A.peer[__ffs(m) - 1][out_off + o] = v;
      };
#if TSV_ZPAIR == 2
      // paired z map: with z_X = XOR_{j in X} z_j,
      //   z_T * (XOR_{P in T, |P| = L-1} U[P])
      //     = XOR_P XOR_{j in T} z_j U[P] = S[T] ^ XOR_{P in T} z_P U[P]
      // (j = T - P gives S[T]'s terms, j in P the rest), so
      //   S[T] = z_T * XOR_P U[P]  ^  XOR_P W[P],   W[P] = z_P * U[P]:
      // one product per input entry and one per output (C5, L = 3: 20
      // instead of 30).  W rides in shared memory, the loops stay rolled.
      if constexpr (kZPairOk) {
        // the row's z_j next to its W entries (table entries E+1 .. E+K of
        // the lane's column): the output loop picks them by a dynamic index
        static_assert(E + K <= 15, "lane-table column holds W and z");
#pragma unroll
        for (int j = 0; j < K; ++j) wrow[(E + j) * 32] = z[j];
#pragma unroll kZUnroll
        for (int p = 0; p < E; ++p) {
          uint64_t zp = 0;
#pragma unroll
          for (int c = 0; c < L - 1; ++c) zp ^= wrow[(E + S.pmem[p][c]) * 32];
          wrow[p * 32] = gf_reduce_alu(clmul64_kara_s(ksplit(zp), ksplit(S.q[p][qi])));
        }
#pragma unroll kZUnroll
        for (int o = 0; o < F; ++o) {
          uint64_t zt = 0, su = 0, sw = 0;
#pragma unroll
          for (int c = 0; c < L; ++c) {
            const int j = S.pj[o][c], pi = S.pin[o][c];
            zt ^= wrow[(E + j) * 32];  // z_j of this row (stored below)
            su ^= S.q[pi][qi];
            sw ^= wrow[pi * 32];
          }
          put(o, gf_reduce_alu(clmul64_kara_s(ksplit(zt), ksplit(su))) ^ sw);
        }
      } else
#endif
      {
#pragma unroll 1
        for (int o = 0; o < F; ++o) {
          ClassAcc ca;
          class_zero(ca);
#pragma unroll
          for (int c = 0; c < L; ++c) {
            const int j = S.pj[o][c];
            uint64_t zj = z[0];
#pragma unroll
            for (int jj = 1; jj < K; ++jj) zj = j == jj ? z[jj] : zj;
            class_acc(ksplit(zj), ksplit(S.q[S.pin[o][c]][qi]), ca);
          }
          put(o, gf_reduce_alu(class_finish(ca)));
        }
      }
    }
    qh = (qh + take) & (kQCap - 1);
    qn -= take;
    __syncwarp();
  };

  // Software pipeline over the lane's arcs, so that no global load is
  // waited for where it is issued: step i's metadata is loaded two steps
  // ahead, its source row (registers) and its run's slot one step ahead.
  auto ld_meta = [&](int i, uint32_t& meta, int32_t& src) {
    meta = 0;
    src = -1;
    if (i < cnt) {
      const int64_t a = a0 + i;
      meta = __ldg(P.g.arc_meta + a);
      src = FIRST ? __ldg(P.g.arc_tail + a) : __ldg(P.g.arc_src + a);
      if (FIRST && P.anchor_source >= 0 && src != P.anchor_source) src = -1;
    }
  };
  auto ld_row = [&](int32_t src, uint64_t (&x)[E]) {
    if (src >= 0) {
      constexpr int kStride = FIRST ? E : vpad(E);
      const uint64_t* row = rows + static_cast<int64_t>(src) * kStride;
      if constexpr (kStride % 2 == 0) {  // 16-byte aligned rows
#pragma unroll
        for (int e = 0; e + 1 < E; e += 2) ld_row128(row + e, x[e], x[e + 1]);
        if constexpr (E % 2) x[E - 1] = ld_row64(row + E - 1);
      } else {
#pragma unroll
        for (int e = 0; e < E; ++e) x[e] = ld_row64(row + e);
      }
    }
  };
  // what a step needs of its run: the state slot at a run end (levels < k)
  auto ld_run = [&](uint32_t meta, int32_t src, int32_t r) -> int32_t {
    (void)src;
    if (LAST) return -1;
    return (meta & kRunEnd) ? __ldg(P.g.run_slot + r) : -1;
  };
  uint32_t m0, m1;
  int32_t s0, s1;
  ld_meta(0, m0, s0);
  ld_meta(1, m1, s1);
  uint64_t xc[E], xn[E];
  ld_row(s0, xc);
  int32_t r0 = ld_run(m0, s0, run);
  // horizon below t: a vertex's arcs are in time order, so it is done at
  // its first arc past max_ts -- an arc past the horizon only feeds rows
  // that arcs past the horizon read, and no accumulator -- and the warp
  // stops when all its lanes are.  At max_ts = t no timestamp is read.
  const bool hz = P.below_t;
  int32_t t0 = INT32_MAX, t1 = INT32_MAX;
  if (hz && cnt > 0) t0 = __ldg(P.g.run_ts + run);
  for (int i = 0; i < steps; ++i) {
    uint32_t m2;
    int32_t s2;
    ld_meta(i + 2, m2, s2);
    ld_row(s1, xn);
    const bool runend = (m0 & kRunEnd) != 0;
    const int32_t run1 = run + (runend ? 1 : 0);
    const int32_t r1 = ld_run(m1, s1, run1);
    if (hz) t1 = i + 1 < cnt ? __ldg(P.g.run_ts + run1) : INT32_MAX;
    const bool past = hz && t0 > P.max_ts;
    if (hz && !__any_sync(kFullV, !past)) break;
    const bool live = s0 >= 0 && !past;
    if (live) {
      const uint64_t y = draw_edge_y(pre, yb, m0 & kEdgeMask);
      if constexpr (kTab) {
        LT.build(y);
#pragma unroll
        for (int e = 0; e < E; ++e) u[e] ^= gf_reduce124(LT.clmul(xc[e], 0u));
      } else {
        const KSplit ys = ksplit(y);
#pragma unroll kVUnroll
        for (int e = 0; e < E; ++e) u[e] ^= gf_reduce_alu(clmul64_kara_s(ys, ksplit(xc[e])));
      }
    }
    if (!LAST) {
      const int32_t slot = past ? -1 : r0;  // -1 unless a referenced run ends here
      const unsigned push = __ballot_sync(kFullV, slot >= 0);
      if (push) {
        if (slot >= 0) {
          const int qi = (qh + qn + __popc(push & ((1u << lane) - 1u))) & (kQCap - 1);
          S.q_slot[qi] = slot;
          S.q_head[qi] = h;
#pragma unroll
          for (int e = 0; e < E; ++e) S.q[e][qi] = u[e];
        }
        qn += __popc(push);
        if (qn >= 32) flush(32);
      }
    }
    run = run1;
    m0 = m1;
    s0 = s1;
    m1 = m2;
    s1 = s2;
    r0 = r1;
    t0 = t1;
#pragma unroll
    for (int e = 0; e < E; ++e) xc[e] = xn[e];
  }
  if (!LAST) {
    while (qn > 0) flush(qn < 32 ? qn : 32);
  } else if (act && cnt > 0) {
    // readout: acc[h] ^= det * XOR_j z_{h,j} * U_k[[k] - {j}]; U_k entries are
    // the (k-1)-subsets, [k] - {j} has colex rank k-1-j
    ClassAcc ca;
    class_zero(ca);
#pragma unroll
    for (int j = 0; j < K; ++j)
      class_acc(ksplit(__ldg(P.zj + static_cast<int64_t>(h) * K + j)), ksplit(u[K - 1 - j]), ca);
    uint64_t v = gf_reduce_alu(class_finish(ca));
    if (A.det != 1) v = gf_mul(A.det, v);
    if (v) A.acc[h] ^= v;
  }
}

template <int K, int L, bool FIRST, bool LAST>
void vertex_launch(const VertArgs& a, unsigned blocks, cudaStream_t st) {
  constexpr int E = binom_c(K, L - 1);
  constexpr bool kTab = vert_uses_table<K, L>();
  using Sm = VertSmem<E, binom_c(K, L), L, LAST>;
  const size_t dyn =
      vert_scratch<E, kTab>() * kVWarps + (kTab ? 4096u : 0u) + sizeof(Sm) * kVWarps + 16;
  if (dyn > 48u * 1024u)  // per device: set whenever the opt-in size is needed
    cudaFuncSetAttribute(k_coef_vertex<K, L, FIRST, LAST>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(dyn));
  k_coef_vertex<K, L, FIRST, LAST><<<blocks, dim3(kVWarps * 32), dyn, st>>>(a);
}

template <int K>
void vertex_dispatch(const VertArgs& a, int l, cudaStream_t st) {
  const unsigned blocks =
      static_cast<unsigned>((a.nv + 32 * kVWarps - 1) / (32 * kVWarps));
  if (!blocks) return;
  if (l == 2 && l == K) vertex_launch<K, 2, true, true>(a, blocks, st);
  else if (l == 2) vertex_launch<K, 2, true, false>(a, blocks, st);
  else if (l == K) {
    if constexpr (K >= 3) vertex_launch<K, K, false, true>(a, blocks, st);
  } else {
    if constexpr (K >= 4) {
      if (l == 3) vertex_launch<K, 3, false, false>(a, blocks, st);
      if constexpr (K >= 5)
        if (l == 4) vertex_launch<K, 4, false, false>(a, blocks, st);
    }
  }
}

// ---- work list: vertices with arcs, sorted by arc count (descending) -------

__global__ void k_vstart_pos(int64_t A, const uint32_t* __restrict__ meta,
                             uint8_t* __restrict__ f) {
  const int64_t a = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (a < A) f[a] = (meta[a] & kVStart) ? 1 : 0;
}

__global__ void k_has_runs(int32_t n, const int32_t* __restrict__ vro, uint8_t* __restrict__ f) {
  const int64_t x = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (x < n) f[x] = vro[x + 1] > vro[x] ? 1 : 0;
}

// list entries i0 .. i0+nv of the nvall vertex starts
__global__ void k_counts(int64_t nv, int64_t i0, int64_t nvall, int64_t A,
                         const int64_t* __restrict__ start, int32_t* __restrict__ cnt,
                         int32_t* __restrict__ pos) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= nv) return;
  const int64_t g = i0 + i;
  cnt[i] = static_cast<int32_t>((g + 1 < nvall ? start[g + 1] : A) - start[g]);
  pos[i] = static_cast<int32_t>(i);
}

__global__ void k_gather_start(int64_t nv, int64_t i0, const int32_t* __restrict__ perm,
                               const int64_t* __restrict__ start,
                               const int32_t* __restrict__ head_in, int64_t* __restrict__ s_out,
                               int32_t* __restrict__ h_out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= nv) return;
  const int64_t p = i0 + perm[i];
  s_out[i] = start[p];
  h_out[i] = head_in[p];
}

// [lower_bound(heads, lo), lower_bound(heads, hi)) of the increasing list
__global__ void k_list_range(const int32_t* __restrict__ heads, int64_t nv, int32_t lo,
                             int32_t hi, int64_t* __restrict__ out) {
  for (int w = 0; w < 2; ++w) {
    const int32_t key = w ? hi : lo;
    int64_t a = 0, b = nv;
    while (a < b) {
      const int64_t mid = (a + b) >> 1;
      if (heads[mid] < key) a = mid + 1;
      else b = mid;
    }
    out[w] = a;
  }
}

// referenced runs (state slots) among runs [0, r): slots are assigned in
// run order, so this is the first slot of the runs from r on
__global__ void k_count_slots(const int32_t* __restrict__ run_slot, int64_t r,
                              unsigned long long* __restrict__ out) {
  __shared__ unsigned long long part[8];
  unsigned long long c = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < r;
       i += (int64_t)gridDim.x * blockDim.x)
    c += run_slot[i] >= 0;
  for (int d = 16; d; d >>= 1) c += __shfl_down_sync(0xffffffffu, c, d);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long s = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += part[w];
    atomicAdd(out, s);
  }
}

inline unsigned nblk_v(int64_t n) { return static_cast<unsigned>((n + 255) / 256); }

}  // namespace

bool vertex_engine_supports(int k) { return k >= 2 && k <= kVertexMaxK; }

int vertex_row_words(int k, int l) { return vpad(binom_c(k, l)); }

void build_vertex_list(const DevGraph& g, VertList& out, cudaStream_t st,
                       const std::function<void*(size_t)>& alloc,
                       const std::function<void(void*)>& release, int32_t v_lo, int32_t v_hi) {
  const int64_t A = g.A;
  const int32_t n = g.n;
  out = VertList{};
  if (v_hi < 0) v_hi = n;
  if (A == 0 || n == 0 || v_lo >= v_hi) return;
  auto ck = [](cudaError_t e) {
    if (e != cudaSuccess)
      throw std::runtime_error(std::string("vertex list: ") + cudaGetErrorString(e));
  };
  // vertex starts in arc order (= increasing vertex id; at most n of them) ...
  uint8_t* vf = static_cast<uint8_t*>(alloc(static_cast<size_t>(A)));
  int64_t* vs = static_cast<int64_t*>(alloc((static_cast<size_t>(n) + 1) * 8));
  int64_t* cnt64 = static_cast<int64_t*>(alloc(8));
  k_vstart_pos<<<nblk_v(A), 256, 0, st>>>(A, g.arc_meta, vf);
  cub::CountingInputIterator<int64_t> it(0);
  size_t tmp = 0;
  ck(cub::DeviceSelect::Flagged(nullptr, tmp, it, vf, vs, cnt64, A, st));
  void* t = alloc(tmp ? tmp : 8);
  ck(cub::DeviceSelect::Flagged(t, tmp, it, vf, vs, cnt64, A, st));
  release(t);
  int64_t nv = 0;
  ck(cudaMemcpyAsync(&nv, cnt64, 8, cudaMemcpyDeviceToHost, st));
  ck(cudaStreamSynchronize(st));
  release(vf);
  release(cnt64);
  // ... which are the vertices with runs, in increasing id
  uint8_t* hf = static_cast<uint8_t*>(alloc(static_cast<size_t>(n)));
  int32_t* heads = static_cast<int32_t*>(alloc(static_cast<size_t>(nv) * 4 + 4));
  int32_t* cnt32 = static_cast<int32_t*>(alloc(8));
  k_has_runs<<<nblk_v(n), 256, 0, st>>>(n, g.vtx_run_off, hf);
  cub::CountingInputIterator<int32_t> it32(0);
  tmp = 0;
  ck(cub::DeviceSelect::Flagged(nullptr, tmp, it32, hf, heads, cnt32, n, st));
  t = alloc(tmp ? tmp : 8);
  ck(cub::DeviceSelect::Flagged(t, tmp, it32, hf, heads, cnt32, n, st));
  release(t);
  release(hf);
  release(cnt32);
  // the vertices of [v_lo, v_hi): a contiguous range [i0, i1) of the list
  int64_t* rng = static_cast<int64_t*>(alloc(16));
  k_list_range<<<1, 1, 0, st>>>(heads, nv, v_lo, v_hi, rng);
  int64_t hr[2] = {0, 0};
  ck(cudaMemcpyAsync(hr, rng, 16, cudaMemcpyDeviceToHost, st));
  ck(cudaStreamSynchronize(st));
  release(rng);
  const int64_t i0 = hr[0];
  const int64_t nvall = nv;
  nv = hr[1] - hr[0];
  if (nv <= 0) {
    release(vs);
    release(heads);
    return;
  }
  // arc counts; sort by count (descending), carrying the list position
  int32_t* counts = static_cast<int32_t*>(alloc(static_cast<size_t>(nv) * 4 + 4));
  int32_t* pos = static_cast<int32_t*>(alloc(static_cast<size_t>(nv) * 4 + 4));
  int32_t* counts_s = static_cast<int32_t*>(alloc(static_cast<size_t>(nv) * 4 + 4));
  int32_t* pos_s = static_cast<int32_t*>(alloc(static_cast<size_t>(nv) * 4 + 4));
  k_counts<<<nblk_v(nv), 256, 0, st>>>(nv, i0, nvall, A, vs, counts, pos);
  tmp = 0;
  ck(cub::DeviceRadixSort::SortPairsDescending(nullptr, tmp, counts, counts_s, pos, pos_s,
                                               static_cast<int>(nv), 0, 32, st));
  t = alloc(tmp ? tmp : 8);
  ck(cub::DeviceRadixSort::SortPairsDescending(t, tmp, counts, counts_s, pos, pos_s,
                                               static_cast<int>(nv), 0, 32, st));
  release(t);
  release(counts);
  release(pos);
  int64_t* start_s = static_cast<int64_t*>(alloc(static_cast<size_t>(nv) * 8 + 8));
  int32_t* head_s = static_cast<int32_t*>(alloc(static_cast<size_t>(nv) * 4 + 4));
  k_gather_start<<<nblk_v(nv), 256, 0, st>>>(nv, i0, pos_s, vs, heads, start_s, head_s);
  ck(cudaGetLastError());
  ck(cudaStreamSynchronize(st));
  release(pos_s);
  release(vs);
  release(heads);
  out.nv = nv;
  out.head = head_s;
  out.start = start_s;
  out.count = counts_s;
}

namespace {

// reader mask of every state slot: bit q set when an arc whose head rank q
// owns reads the slot (one byte per slot, packed four to a word)
__global__ void k_reader_mask(const int64_t* __restrict__ wl_start,
                              const int32_t* __restrict__ wl_count, int64_t nv,
                              const int32_t* __restrict__ arc_src, int q,
                              unsigned int* __restrict__ mask) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= nv) return;
  const int64_t a0 = wl_start[i];
  const int c = wl_count[i];
  const unsigned bit = 1u << q;
  for (int j = 0; j < c; ++j) {
    const int32_t s = arc_src[a0 + j];
    if (s >= 0) atomicOr(mask + (s >> 2), bit << (8 * (s & 3)));
  }
}

__global__ void k_mask_flags(const unsigned int* __restrict__ mask, int64_t lo, int64_t hi, int q,
                             uint8_t* __restrict__ f) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= hi - lo) return;
  const int64_t s = lo + i;
  f[i] = ((mask[s >> 2] >> (8 * (s & 3))) >> q) & 1u;
}

template <bool PACK>
__global__ void k_rows_move(const int32_t* __restrict__ slots, int64_t count, int F,
                            const uint64_t* __restrict__ src, uint64_t* __restrict__ dst) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= count * F) return;
  const int64_t r = i / F;
  const int e = static_cast<int>(i - r * F);
  const int64_t s = slots[r];
  if (PACK) dst[i] = src[s * F + e];
  else dst[s * F + e] = src[i];
}

}  // namespace

void build_exchange_lists(const DevGraph& g, const std::vector<const VertList*>& lists,
                          const std::vector<int64_t>& slot_lo, const std::vector<int64_t>& slot_hi,
                          int rank, ExchangeLists& out, cudaStream_t st,
                          const std::function<void*(size_t)>& alloc,
                          const std::function<void(void*)>& release) {
  auto ck = [](cudaError_t e) {
    if (e != cudaSuccess)
      throw std::runtime_error(std::string("exchange lists: ") + cudaGetErrorString(e));
  };
  const int world = static_cast<int>(lists.size());
  const int64_t S = std::max<int64_t>(g.S, 1);
  auto* mask = static_cast<unsigned int*>(alloc(static_cast<size_t>((S + 3) / 4) * 4));
  ck(cudaMemsetAsync(mask, 0, static_cast<size_t>((S + 3) / 4) * 4, st));
  for (int q = 0; q < world; ++q) {
    const VertList* vl = lists[q];
    if (vl->nv)
      k_reader_mask<<<nblk_v(vl->nv), 256, 0, st>>>(vl->start, vl->count, vl->nv,
                                                     g.arc_src, q, mask);
  }
  out = ExchangeLists{};
  out.reader_mask = mask;
  out.send_count.assign(world, 0);
  out.recv_count.assign(world, 0);
  // send to q: my slots with bit q; receive from q: q's slots with my bit
  std::vector<int32_t*> parts_s(world, nullptr), parts_r(world, nullptr);
  int64_t* cnt = static_cast<int64_t*>(alloc(8));
  auto select = [&](int64_t lo, int64_t hi, int bitq, int32_t** outp, int64_t* n) {
    *outp = nullptr;
    *n = 0;
    if (hi <= lo) return;
    uint8_t* f = static_cast<uint8_t*>(alloc(static_cast<size_t>(hi - lo)));
    int32_t* o = static_cast<int32_t*>(alloc(static_cast<size_t>(hi - lo) * 4));
    k_mask_flags<<<nblk_v(hi - lo), 256, 0, st>>>(mask, lo, hi, bitq, f);
    cub::CountingInputIterator<int32_t> it(static_cast<int32_t>(lo));
    size_t tmp = 0;
    ck(cub::DeviceSelect::Flagged(nullptr, tmp, it, f, o, cnt, hi - lo, st));
    void* t = alloc(tmp ? tmp : 8);
    ck(cub::DeviceSelect::Flagged(t, tmp, it, f, o, cnt, hi - lo, st));
    ck(cudaMemcpyAsync(n, cnt, 8, cudaMemcpyDeviceToHost, st));
    ck(cudaStreamSynchronize(st));
    release(t);
    release(f);
    *outp = o;
  };
  for (int q = 0; q < world; ++q) {
    if (q == rank) continue;
    select(slot_lo[rank], slot_hi[rank], q, &parts_s[q], &out.send_count[q]);
    select(slot_lo[q], slot_hi[q], rank, &parts_r[q], &out.recv_count[q]);
  }
  release(cnt);
  // one array per direction, peers in rank order
  int64_t ts = 0, tr = 0;
  for (int q = 0; q < world; ++q) ts += out.send_count[q], tr += out.recv_count[q];
  out.send_slots = static_cast<int32_t*>(alloc(static_cast<size_t>(ts) * 4 + 4));
  out.recv_slots = static_cast<int32_t*>(alloc(static_cast<size_t>(tr) * 4 + 4));
  int64_t os = 0, orr = 0;
  for (int q = 0; q < world; ++q) {
    if (out.send_count[q])
      ck(cudaMemcpyAsync(out.send_slots + os, parts_s[q], out.send_count[q] * 4,
                         cudaMemcpyDeviceToDevice, st));
    if (out.recv_count[q])
      ck(cudaMemcpyAsync(out.recv_slots + orr, parts_r[q], out.recv_count[q] * 4,
                         cudaMemcpyDeviceToDevice, st));
    os += out.send_count[q];
    orr += out.recv_count[q];
  }
  ck(cudaStreamSynchronize(st));
  for (int q = 0; q < world; ++q) {
    if (parts_s[q]) release(parts_s[q]);
    if (parts_r[q]) release(parts_r[q]);
  }
  out.send_total = ts;
  out.recv_total = tr;
}

void launch_rows_pack(const int32_t* slots, int64_t count, int F, const uint64_t* rows,
                      uint64_t* buf, cudaStream_t st) {
  if (count <= 0) return;
  prof_begin("vertex_exchange", st);
  k_rows_move<true><<<nblk_v(count * F), 256, 0, st>>>(slots, count, F, rows, buf);
  prof_end(st);
}

void launch_rows_unpack(const int32_t* slots, int64_t count, int F, const uint64_t* buf,
                        uint64_t* rows, cudaStream_t st) {
  if (count <= 0) return;
  prof_begin("vertex_exchange", st);
  k_rows_move<false><<<nblk_v(count * F), 256, 0, st>>>(slots, count, F, buf, rows);
  prof_end(st);
}

int64_t count_slots_before(const DevGraph& g, int64_t r, cudaStream_t st,
                           const std::function<void*(size_t)>& alloc,
                           const std::function<void(void*)>& release) {
  if (r <= 0) return 0;
  auto* d = static_cast<unsigned long long*>(alloc(8));
  cudaMemsetAsync(d, 0, 8, st);
  k_count_slots<<<148 * 4, 256, 0, st>>>(g.run_slot, r, d);
  unsigned long long h = 0;
  cudaMemcpyAsync(&h, d, 8, cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  release(d);
  return static_cast<int64_t>(h);
}

void launch_coef_vertex(const CoefParams& p, const VertList& vl, uint64_t det, uint64_t* acc,
                        cudaStream_t st, const VertPeers* peers) {
  if (vl.nv == 0) return;
  VertArgs a;
  a.rmask = nullptr;
  a.self_clear = 0xffu;
  for (int q = 0; q < 8; ++q) a.peer[q] = nullptr;
  if (peers && peers->reader_mask && !p.last) {
    a.rmask = peers->reader_mask;
    a.self_clear = 0xffu & ~(1u << peers->rank);
    for (int q = 0; q < 8; ++q) {
      a.peer[q] = peers->peer[q];
      if (!a.peer[q]) a.self_clear &= ~(1u << q);  // no buffer given: not stored
    }
  }
  a.P = p;
  a.wl_head = vl.head;
  a.wl_start = vl.start;
  a.wl_count = vl.count;
  a.nv = vl.nv;
  a.det = det;
  a.acc = acc;
  prof_begin(p.last ? "coef_vertex_last" : p.ell == 2 ? "coef_vertex_first" : "coef_vertex", st);
  switch (p.k) {
    case 2: vertex_dispatch<2>(a, p.ell, st); break;
    case 3: vertex_dispatch<3>(a, p.ell, st); break;
    case 4: vertex_dispatch<4>(a, p.ell, st); break;
    case 5: vertex_dispatch<5>(a, p.ell, st); break;
    default: break;
  }
  prof_end(st);
}

}  // namespace tsv

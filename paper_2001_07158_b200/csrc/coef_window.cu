// coef_window.cu -- time windows for the coefficient engine (coef_kernels.cu,
// coef_items.cu), for evaluations whose state rows do not fit in HBM at once
// (C4: k_eff = 12, ~1e8 referenced runs x up to 462 words per level).
//
// The DP P[l][v][t] (sieve.cpp:199-256) runs forward in time, and a state
// row is read only by arcs whose time lies after it, so the arcs can be
// processed in windows of consecutive timestamps [t_a, t_b) -- every level
// of one window before the next window -- keeping per vertex and level only
// the state as of the window start (the CARRY: the prefix U_l of the
// vertex's runs so far, in the row form of the engine):
//
//  * an arc of the window whose tail has no run in the window before it
//    reads the tail's carried state: its source is the CARRY SLOT S_w + tail
//    (k_win_src), a row filled from the carry before the level's z map
//    (k_win_carry_slots);
//  * a head's prefix within the window starts from its carry instead of
//    zero (CoefParams::carry_in, read at the vertex start by the item-stream
//    kernels), so every window row already holds it (U space: the z map of
//    multi-shade rows follows);
//  * every vertex's LAST run of the window gets a state slot
//    (build_run_slots with vtx_run_off), whose row is the vertex's carry for
//    the next window (k_win_carry_out);
//  * level k XORs each vertex piece into ulast as before: it accumulates over
//    the windows, and the readout runs once at the end.
//
// Window boundaries fall between distinct timestamps (a run is one (head,
// ts) pair), edge ids are the original graph's (y draws unchanged), so the
// accumulators are bit-identical to the one-pass engine.
#include <cuda_runtime.h>

#include <cstdint>

#include "coef.hpp"
#include "layout.hpp"

namespace tsv {
namespace {

constexpr int kWT = 256;
inline unsigned nblk_w(int64_t n) { return static_cast<unsigned>((n + kWT - 1) / kWT); }

__device__ __forceinline__ int frame_of(const int8_t* __restrict__ vsh, int32_t v, int frs,
                                        int frm) {
  const int c = __ldg(vsh + v);
  return c == -1 ? 0 : (c >= 0 && frs > 0 ? frs : frm);
}

__global__ void k_win_src(int64_t A, int32_t* __restrict__ arc_src,
                          const int32_t* __restrict__ arc_tail, int64_t base) {
  const int64_t a = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (a >= A) return;
  const int32_t t = arc_tail[a];
  if (arc_src[a] < 0 && t >= 0) arc_src[a] = static_cast<int32_t>(base + t);
}

__global__ void k_win_edge_ids(int64_t A, uint32_t* __restrict__ meta,
                               const int32_t* __restrict__ oid, int64_t base) {
  const int64_t a = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (a >= A) return;
  const uint32_t mt = meta[a];
  const int64_t e = base + (mt & kEdgeMask);
  meta[a] = (mt & ~kEdgeMask) | static_cast<uint32_t>(oid ? oid[e] : e);
}

// carry slots S_w + v <- carry[v] (the state as of the window start)
__global__ void k_win_carry_slots(int32_t n, int64_t Sw, const int8_t* __restrict__ vsh, int frs,
                                  int frm, uint64_t* __restrict__ rows, int rs,
                                  uint8_t* __restrict__ sflag, const uint64_t* __restrict__ carry,
                                  int cs, const uint8_t* __restrict__ cnz) {
  const int64_t v = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (v >= n) return;
  const bool nz = cnz[v] != 0;
  if (lane == 0) sflag[Sw + v] = nz ? 1 : 0;
  if (!nz) return;
  const int fr = frame_of(vsh, static_cast<int32_t>(v), frs, frm);
  uint64_t* row = rows + (Sw + v) * rs;
  const uint64_t* c = carry + v * cs;
  for (int e = lane; e < fr; e += 32) row[e] = c[e];
}

// carry[v] <- the row of v's last run in the window (its prefix started
// from the carry, CoefParams::carry_in)
__global__ void k_win_carry_out(int32_t n, const int32_t* __restrict__ vro,
                                const int32_t* __restrict__ run_slot,
                                const int8_t* __restrict__ vsh, int frs, int frm,
                                const uint64_t* __restrict__ rows, int rs,
                                const uint8_t* __restrict__ sflag, uint64_t* __restrict__ carry,
                                int cs, uint8_t* __restrict__ cnz) {
  const int64_t v = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (v >= n) return;
  const int32_t r0 = vro[v], r1 = vro[v + 1];
  if (r1 <= r0) return;  // no run in the window: the carry stands
  const int32_t s = run_slot[r1 - 1];
  const bool nz = s >= 0 && sflag[s] != 0;
  if (lane == 0) cnz[v] = nz ? 1 : 0;
  if (!nz) return;
  const int fr = frame_of(vsh, static_cast<int32_t>(v), frs, frm);
  const uint64_t* row = rows + static_cast<int64_t>(s) * rs;
  uint64_t* c = carry + v * cs;
  for (int e = lane; e < fr; e += 32) c[e] = row[e];
}

// (slot, head) list of the carry slots of multi-shade vertices (z map)
__global__ void k_win_multi_list(int32_t n, int64_t Sw, const int8_t* __restrict__ vsh,
                                 int2* __restrict__ list, int32_t* __restrict__ count) {
  const int64_t v = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const bool mine = v < n && __ldg(vsh + v) == -2;
  const unsigned m = __ballot_sync(0xffffffffu, mine);
  if (!m) return;
  int base = 0;
  if (lane == __ffs(m) - 1) base = atomicAdd(count, __popc(m));
  base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
  if (mine)
    list[base + __popc(m & ((1u << lane) - 1u))] =
        make_int2(static_cast<int>(Sw + v), static_cast<int>(v));
}

// out[i] = first index j with ts[j] == ts[pos[i]] (ts nondecreasing)
__global__ void k_ts_group_start(const int32_t* __restrict__ ts, const int64_t* __restrict__ pos,
                                 int nb, int64_t* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nb) return;
  const int64_t p = pos[i];
  const int32_t key = ts[p];
  int64_t a = 0, b = p;
  while (a < b) {
    const int64_t mid = (a + b) >> 1;
    if (ts[mid] < key) a = mid + 1;
    else b = mid;
  }
  out[i] = a;
}

}  // namespace

void launch_win_src(int64_t A, int32_t* arc_src, const int32_t* arc_tail, int64_t base,
                    cudaStream_t st) {
  if (A > 0) k_win_src<<<nblk_w(A), kWT, 0, st>>>(A, arc_src, arc_tail, base);
}

void launch_win_edge_ids(int64_t A, uint32_t* meta, const int32_t* oid, int64_t base,
                         cudaStream_t st) {
  if (A > 0) k_win_edge_ids<<<nblk_w(A), kWT, 0, st>>>(A, meta, oid, base);
}

void launch_win_carry(const WinCarryArgs& a, cudaStream_t st) {
  if (a.n <= 0) return;
  prof_begin("coef_win_carry", st);
  const int64_t thr = static_cast<int64_t>(a.n) * 32;
  k_win_carry_slots<<<nblk_w(thr), kWT, 0, st>>>(a.n, a.Sw, a.vsh, a.frs, a.frm, a.rows, a.rs,
                                                 a.sflag, a.carry, a.cs, a.cnz);
  k_win_carry_out<<<nblk_w(thr), kWT, 0, st>>>(a.n, a.vro, a.run_slot, a.vsh, a.frs, a.frm, a.rows,
                                               a.rs, a.sflag, a.carry, a.cs, a.cnz);
  prof_end(st);
}

void launch_win_multi_list(int32_t n, int64_t Sw, const int8_t* vsh, int2* list, int32_t* count,
                           cudaStream_t st) {
  cudaMemsetAsync(count, 0, 4, st);
  if (n > 0) k_win_multi_list<<<nblk_w(n), kWT, 0, st>>>(n, Sw, vsh, list, count);
}

void launch_ts_group_start(const int32_t* ts, const int64_t* pos, int nb, int64_t* out,
                           cudaStream_t st) {
  if (nb > 0) k_ts_group_start<<<(nb + 127) / 128, 128, 0, st>>>(ts, pos, nb, out);
}

}  // namespace tsv

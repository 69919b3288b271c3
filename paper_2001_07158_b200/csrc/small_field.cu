// small_field.cu -- the temporal sieve over GF(2^b), b in {8, 16, 32}: the
// reference's `--field-bits 8|16|32` (tools/main.cpp:70), which measures the
// false-negative rate (2k-1)/2^b of small fields.  Bit-exact with
// temporal_impl<uint8_t|uint16_t|uint32_t> (sieve.cpp:170-307 through the
// dispatch at :637-649): same moduli (gf.hpp:36-42), same draws truncated to
// b bits with the same nonzero re-mix (gf.hpp:147-153).
//
// This is the point form in its plainest shape -- one
// thread per (head vertex, sieve point) walking the vertex's arcs in time
// order over the vertex-major layout, the tail states gathered by slot --
// not a tuned engine: GF(2^64) is the width every BASELINE config and the
// solver default use.
#include <cuda_runtime.h>

#include <cstdint>

#include "engine.hpp"
#include "gf_device.cuh"
#include "layout.hpp"
#include "small_field.cuh"

namespace tsv {
namespace {

// z_{u,j} = XOR_{d in S(u)} v_{u,d} * w_{d,j} (sieve.cpp:83-101); j, d 1-based
template <typename Word>
__global__ void k_small_zj(int32_t n, int k, uint64_t pre_v, uint64_t pre_w,
                           const int32_t* __restrict__ off, const int32_t* __restrict__ shades,
                           Word* __restrict__ zj) {
  const int64_t u = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (u >= n) return;
  for (int j = 0; j < k; ++j) {
    Word z = 0;
    for (int32_t i = off[u]; i < off[u + 1]; ++i) {
      const int d = shades[i];
      z ^= smul<Word>(sdraw<Word>(pre_v, static_cast<uint64_t>(u), d, 0),
                      sdraw<Word>(pre_w, static_cast<uint64_t>(d), j + 1, 0));
    }
    zj[u * k + j] = z;
  }
}

template <typename Word>
__device__ __forceinline__ Word z_of(const Word* __restrict__ zj, int k, int64_t u, uint64_t A) {
  Word z = 0;
  for (int j = 0; j < k; ++j)
    if ((A >> j) & 1ull) z ^= zj[u * k + j];
  return z;
}

// One level over a batch of W points [pb, pb + W): thread (vertex i, point w).
//   P[h][l][i] = P[h][l][i-1] ^ z_h^A * XOR_{arcs (t -> h, i)} y(e, l-1) * P[t][l-1][i-1]
// with the tail's state at its last run before the arc (arc_src, a slot),
// P[t][1] = z_t^A, anchor: level 2 only from the source; level k: the prefix
// at the last run <= max_ts XORed into acc[h] over the batch's points.
template <typename Word, bool FIRST, bool LAST>
__global__ void k_small_level(const DevGraph g, const int32_t* __restrict__ head,
                              const int64_t* __restrict__ start, const int32_t* __restrict__ count,
                              int64_t nv, const Word* __restrict__ zj, int k, int ell, uint64_t pre_y,
                              int32_t anchor, const Word* __restrict__ s_prev,
                              Word* __restrict__ s_cur, int W, uint64_t pb, uint64_t pe,
                              int32_t max_ts, uint64_t* __restrict__ acc) {
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t i = idx / W;
  const int w = static_cast<int>(idx - i * W);
  if (i >= nv) return;
  const uint64_t A = pb + static_cast<uint64_t>(w);
  const bool on = A < pe;
  const int32_t h = head[i];
  const int64_t a0 = start[i];
  const int cnt = count[i];
  int32_t run = g.vtx_run_off[h];
  const Word zh = on ? z_of(zj, k, h, A) : Word(0);
  Word prefix = 0, sum = 0;
  for (int j = 0; j < cnt; ++j) {
    const int64_t a = a0 + j;
    const uint32_t meta = g.arc_meta[a];
    if (on) {
      int32_t src = FIRST ? g.arc_tail[a] : g.arc_src[a];
      bool live = src >= 0;
      if (FIRST) live = live && (anchor < 0 || src == anchor);
      if (LAST) live = live && g.run_ts[run] <= max_ts;
      if (live) {
        const Word x = FIRST ? z_of(zj, k, src, A) : s_prev[static_cast<int64_t>(src) * W + w];
        if (x) sum ^= smul<Word>(sdraw<Word>(pre_y, meta & kEdgeMask, ell - 1, 0), x);
      }
    }
    if (meta & kRunEnd) {
      if (sum) prefix ^= smul<Word>(zh, sum);
      sum = 0;
      if (!LAST && on) {
        const int32_t s = g.run_slot[run];
        if (s >= 0) s_cur[static_cast<int64_t>(s) * W + w] = prefix;
      }
      ++run;
    }
  }
  if (LAST && on && prefix)
    atomicXor(reinterpret_cast<unsigned long long*>(acc + h),
              static_cast<unsigned long long>(prefix));
}

// k = 1: acc[u] ^= XOR over the batch's points of z_u^A (only the source when
// anchored; sieve.cpp:294-306)
template <typename Word>
__global__ void k_small_k1(int32_t n, const Word* __restrict__ zj, uint64_t pb, uint64_t pe,
                           int32_t anchor, uint64_t* __restrict__ acc) {
  const int64_t u = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (u >= n || (anchor >= 0 && u != anchor)) return;
  Word x = 0;
  for (uint64_t A = pb; A < pe; ++A) x ^= z_of(zj, 1, u, A);
  acc[u] ^= x;
}

template <typename Word>
void run_small(const SmallFieldArgs& a, cudaStream_t st) {
  const int32_t n = a.g.n;
  const uint64_t pre_v = draw_prefix(a.seed, kRoleShadeV), pre_w = draw_prefix(a.seed, kRoleShadeW);
  const uint64_t pre_y = draw_prefix(a.seed, kRoleEdgeY);
  Word* zj = static_cast<Word*>(a.alloc(static_cast<size_t>(n) * a.k * sizeof(Word) + 8));
  if (n) k_small_zj<Word><<<(n + 127) / 128, 128, 0, st>>>(n, a.k, pre_v, pre_w, a.off, a.shades, zj);
  if (a.k == 1) {
    if (n) k_small_k1<Word><<<(n + 127) / 128, 128, 0, st>>>(n, zj, a.pb, a.pe, a.anchor, a.acc);
    a.release(zj);
    return;
  }
  const int64_t S = a.g.S > 0 ? a.g.S : 1;
  const int W = a.W;
  Word* s0 = static_cast<Word*>(a.alloc(static_cast<size_t>(S) * W * sizeof(Word)));
  Word* s1 = static_cast<Word*>(a.alloc(static_cast<size_t>(S) * W * sizeof(Word)));
  const int64_t thr = a.nv * W;
  const unsigned blocks = static_cast<unsigned>((thr + 127) / 128);
  for (uint64_t pb = a.pb; pb < a.pe && a.nv; pb += W) {
    const uint64_t pe = pb + W < a.pe ? pb + W : a.pe;
    Word *prev = s1, *cur = s0;
    for (int ell = 2; ell <= a.k; ++ell) {
      const bool first = ell == 2, last = ell == a.k;
      if (first && last)
        k_small_level<Word, true, true><<<blocks, 128, 0, st>>>(
            a.g, a.head, a.start, a.count, a.nv, zj, a.k, ell, pre_y, a.anchor, prev, cur, W, pb,
            pe, a.max_ts, a.acc);
      else if (first)
        k_small_level<Word, true, false><<<blocks, 128, 0, st>>>(
            a.g, a.head, a.start, a.count, a.nv, zj, a.k, ell, pre_y, a.anchor, prev, cur, W, pb,
            pe, a.max_ts, a.acc);
      else if (last)
        k_small_level<Word, false, true><<<blocks, 128, 0, st>>>(
            a.g, a.head, a.start, a.count, a.nv, zj, a.k, ell, pre_y, a.anchor, prev, cur, W, pb,
            pe, a.max_ts, a.acc);
      else
        k_small_level<Word, false, false><<<blocks, 128, 0, st>>>(
            a.g, a.head, a.start, a.count, a.nv, zj, a.k, ell, pre_y, a.anchor, prev, cur, W, pb,
            pe, a.max_ts, a.acc);
      Word* t = prev;
      prev = cur;
      cur = t;
    }
  }
  a.release(s0);
  a.release(s1);
  a.release(zj);
}

template <typename Word>
__global__ void k_small_zj64(int32_t n, int k, uint64_t pre_v, uint64_t pre_w,
                             const int32_t* __restrict__ off, const int32_t* __restrict__ shades,
                             uint64_t* __restrict__ zj) {
  const int64_t u = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (u >= n) return;
  for (int j = 0; j < k; ++j) {
    Word z = 0;
    for (int32_t i = off[u]; i < off[u + 1]; ++i) {
      const int d = shades[i];
      z ^= smul<Word>(sdraw<Word>(pre_v, static_cast<uint64_t>(u), d, 0),
                      sdraw<Word>(pre_w, static_cast<uint64_t>(d), j + 1, 0));
    }
    zj[u * k + j] = z;
  }
}

}  // namespace

void launch_small_zj64(int bits, int32_t n, int k, uint64_t seed, const int32_t* off,
                       const int32_t* shades, uint64_t* zj, cudaStream_t st) {
  if (n <= 0) return;
  const uint64_t pv = draw_prefix(seed, kRoleShadeV), pw = draw_prefix(seed, kRoleShadeW);
  const unsigned b = static_cast<unsigned>((n + 127) / 128);
  if (bits == 8) k_small_zj64<uint8_t><<<b, 128, 0, st>>>(n, k, pv, pw, off, shades, zj);
  else if (bits == 16) k_small_zj64<uint16_t><<<b, 128, 0, st>>>(n, k, pv, pw, off, shades, zj);
  else k_small_zj64<uint32_t><<<b, 128, 0, st>>>(n, k, pv, pw, off, shades, zj);
}

void launch_small_field(const SmallFieldArgs& a, cudaStream_t st) {
  prof_begin("small_field", st);
  if (a.bits == 8) run_small<uint8_t>(a, st);
  else if (a.bits == 16) run_small<uint16_t>(a, st);
  else run_small<uint32_t>(a, st);
  prof_end(st);
}

}  // namespace tsv

// finalize.cu -- the reference's finalize (sieve.cpp:136-159, fold_checksum
// :35-49) on the device: sink restriction, flagged count and the FNV-1a-64
// checksum over (u, acc[u]) little-endian byte pairs of the nonzero
// accumulators in ascending u.
//
// FNV-1a is a sequential hash (h = (h ^ byte) * P mod 2^64), ~2 s on one host
// core at n = 1e8 nonzero accumulators -- longer than the C5 sieve itself.
// It parallelizes exactly because of two facts:
//
//  (1) the LOW BYTE of h evolves on its own: XOR with a byte only touches the
//      low 8 bits, and the low 8 bits of a product depend only on the low 8
//      bits of its factors.  So a range of entries maps the incoming low byte
//      L through a permutation of 256 states, which a block computes by
//      running all 256 start states at once (one per thread);
//  (2) given the true low byte L at a range's start, run the full 64-bit hash
//      from h = L.  If the true start is h = L + D (D = 0 mod 256), every
//      step keeps the same low byte and maps (x + D) -> ((x ^ b) + D) * P, so
//      the true end is h_end(L) + D * P^(16 c) for the range's c entries.
//
// Host side: compose the ranges' permutations in order (start bytes), run
// (2) per range on the device, then fold the corrections in order.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "engine.hpp"

namespace tsv {
namespace {

constexpr uint64_t kFnvBasis = 1469598103934665603ull;
constexpr uint64_t kFnvPrime = 1099511628211ull;
constexpr int kFinRange = 8192;   // entries (vertices) per range
constexpr int kFinTile = 1024;    // entries staged in shared memory at a time

__global__ void k_sink_only(uint64_t* acc, int64_t n, int64_t sink) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    if (i != sink) acc[i] = 0;
}

// Phase 1: per range, the permutation of the low byte (perm[r][s]) and the
// nonzero count.  256 threads = 256 start states; entries are staged in
// shared memory (compacted to the nonzero ones) and read as broadcasts.
__global__ void __launch_bounds__(256) k_fnv_perm(const uint64_t* __restrict__ acc, int64_t n,
                                                  uint8_t* __restrict__ perm,
                                                  int32_t* __restrict__ cnt) {
  __shared__ uint2 ent[kFinTile][2];  // (u lo, u hi), (acc lo, acc hi)
  __shared__ int s_n;
  __shared__ int s_warp[8];
  const int64_t r = blockIdx.x;
  const int64_t lo = r * kFinRange;
  const int64_t hi = min(n, lo + kFinRange);
  uint32_t L = threadIdx.x;  // only the low byte is meaningful
  int total = 0;
  for (int64_t t0 = lo; t0 < hi; t0 += kFinTile) {
    if (threadIdx.x == 0) s_n = 0;
    __syncthreads();
    // ordered compaction of the tile's nonzero entries: warp ballots + a
    // block scan over 8 warps (each thread owns 4 consecutive entries)
    const int base = threadIdx.x * 4;
    uint64_t a[4];
    int mine = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t i = t0 + base + j;
      a[j] = i < hi ? acc[i] : 0;
      mine += a[j] != 0;
    }
    int incl = mine;  // inclusive scan in the warp
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, d);
      if ((threadIdx.x & 31) >= d) incl += y;
    }
    if ((threadIdx.x & 31) == 31) s_warp[threadIdx.x >> 5] = incl;
    __syncthreads();
    int woff = 0;
    for (int w = 0; w < (threadIdx.x >> 5); ++w) woff += s_warp[w];
    int pos = woff + incl - mine;
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (a[j]) {
        const uint64_t u = static_cast<uint64_t>(t0 + base + j);
        ent[pos][0] = make_uint2(static_cast<uint32_t>(u), static_cast<uint32_t>(u >> 32));
        ent[pos][1] = make_uint2(static_cast<uint32_t>(a[j]), static_cast<uint32_t>(a[j] >> 32));
        ++pos;
      }
    if (threadIdx.x == 255) s_n = woff + incl;
    __syncthreads();
    const int m = s_n;
    for (int e = 0; e < m; ++e) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint2 x = ent[e][h];
        // only the low byte of L matters: XOR the whole shifted word, the
        // bits above 8 never reach the low byte
        L = (L ^ x.x) * 0xb3u;
        L = (L ^ (x.x >> 8)) * 0xb3u;
        L = (L ^ (x.x >> 16)) * 0xb3u;
        L = (L ^ (x.x >> 24)) * 0xb3u;
        L = (L ^ x.y) * 0xb3u;
        L = (L ^ (x.y >> 8)) * 0xb3u;
        L = (L ^ (x.y >> 16)) * 0xb3u;
        L = (L ^ (x.y >> 24)) * 0xb3u;
      }
    }
    total += m;
    __syncthreads();
  }
  perm[r * 256 + threadIdx.x] = static_cast<uint8_t>(L);
  if (threadIdx.x == 0) cnt[r] = total;
}

__device__ __forceinline__ uint64_t fnv_word(uint64_t h, uint64_t x) {
#pragma unroll
  for (int i = 0; i < 8; ++i) h = (h ^ ((x >> (8 * i)) & 0xff)) * kFnvPrime;
  return h;
}

// Phase 2: per range, the full hash from h = its true start byte, and
// P^(16 * count).  One warp per range: the lanes load 32 consecutive
// accumulators (coalesced, next batch prefetched) and every lane runs the
// same sequential hash over the warp's values (shuffle broadcast).
__global__ void __launch_bounds__(128) k_fnv_range(const uint64_t* __restrict__ acc, int64_t n,
                                                   int64_t nr, const uint8_t* __restrict__ lstart,
                                                   const int32_t* __restrict__ cnt,
                                                   uint64_t* __restrict__ hend,
                                                   uint64_t* __restrict__ pw) {
  const int64_t r = blockIdx.x * 4 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= nr) return;
  const int64_t lo = r * kFinRange;
  const int64_t hi = min(n, lo + kFinRange);
  uint64_t h = lstart[r];
  uint64_t nxt = lo + lane < hi ? acc[lo + lane] : 0;
  for (int64_t b = lo; b < hi; b += 32) {
    const uint64_t v = nxt;
    nxt = b + 32 + lane < hi ? acc[b + 32 + lane] : 0;
    unsigned nz = __ballot_sync(0xffffffffu, v != 0);
    while (nz) {
      const int j = __ffs(nz) - 1;
      nz &= nz - 1;
      const uint64_t a = __shfl_sync(0xffffffffu, v, j);
      h = fnv_word(h, static_cast<uint64_t>(b + j));
      h = fnv_word(h, a);
    }
  }
  if (lane == 0) {
    hend[r] = h;
    // P^(16 c) by squaring
    uint64_t e = 16ull * static_cast<uint64_t>(cnt[r]), bb = kFnvPrime, p = 1;
    while (e) {
      if (e & 1) p *= bb;
      bb *= bb;
      e >>= 1;
    }
    pw[r] = p;
  }
}

}  // namespace

void device_finalize(uint64_t* d_acc, int64_t n, int64_t sink, cudaStream_t st,
                     uint64_t* checksum, int64_t* flagged) {
  if (sink >= 0 && n > 0) {
    prof_begin("finalize", st);
    k_sink_only<<<static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 148 * 16)), 256, 0,
                  st>>>(d_acc, n, sink);
    prof_end(st);
    // one candidate left: hash it on the host
    uint64_t a = 0;
    if (sink < n && cudaMemcpyAsync(&a, d_acc + sink, 8, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
      throw std::runtime_error("device finalize: copy failed");
    uint64_t h = kFnvBasis;
    if (a) {
      for (int i = 0; i < 8; ++i) h = (h ^ ((static_cast<uint64_t>(sink) >> (8 * i)) & 0xff)) * kFnvPrime;
      for (int i = 0; i < 8; ++i) h = (h ^ ((a >> (8 * i)) & 0xff)) * kFnvPrime;
    }
    *checksum = h;
    *flagged = a ? 1 : 0;
    return;
  }
  const int64_t nr = (n + kFinRange - 1) / kFinRange;
  if (nr == 0) {
    *checksum = kFnvBasis;
    *flagged = 0;
    return;
  }
  uint8_t* d_perm = nullptr;
  int32_t* d_cnt = nullptr;
  uint64_t *d_h = nullptr, *d_pw = nullptr;
  uint8_t* d_ls = nullptr;
  auto ck = [](cudaError_t e) {
    if (e != cudaSuccess) throw std::runtime_error(std::string("device finalize: ") + cudaGetErrorString(e));
  };
  ck(cudaMallocAsync(reinterpret_cast<void**>(&d_perm), nr * 256, st));
  ck(cudaMallocAsync(reinterpret_cast<void**>(&d_cnt), nr * 4, st));
  ck(cudaMallocAsync(reinterpret_cast<void**>(&d_h), nr * 8, st));
  ck(cudaMallocAsync(reinterpret_cast<void**>(&d_pw), nr * 8, st));
  ck(cudaMallocAsync(reinterpret_cast<void**>(&d_ls), nr, st));
  std::vector<uint8_t> perm(static_cast<size_t>(nr) * 256), ls(static_cast<size_t>(nr));
  std::vector<uint64_t> hend(static_cast<size_t>(nr)), pw(static_cast<size_t>(nr));
  std::vector<int32_t> cnt(static_cast<size_t>(nr));
  prof_begin("finalize", st);
  k_fnv_perm<<<static_cast<unsigned>(nr), 256, 0, st>>>(d_acc, n, d_perm, d_cnt);
  prof_end(st);
  ck(cudaGetLastError());
  ck(cudaMemcpyAsync(perm.data(), d_perm, perm.size(), cudaMemcpyDeviceToHost, st));
  ck(cudaMemcpyAsync(cnt.data(), d_cnt, cnt.size() * 4, cudaMemcpyDeviceToHost, st));
  ck(cudaStreamSynchronize(st));
  uint32_t L = kFnvBasis & 0xff;
  for (int64_t r = 0; r < nr; ++r) {
    ls[r] = static_cast<uint8_t>(L);
    L = perm[static_cast<size_t>(r) * 256 + L];
  }
  ck(cudaMemcpyAsync(d_ls, ls.data(), ls.size(), cudaMemcpyHostToDevice, st));
  prof_begin("finalize", st);
  k_fnv_range<<<static_cast<unsigned>((nr + 3) / 4), 128, 0, st>>>(d_acc, n, nr, d_ls, d_cnt,
                                                                         d_h, d_pw);
  prof_end(st);
  ck(cudaGetLastError());
  ck(cudaMemcpyAsync(hend.data(), d_h, hend.size() * 8, cudaMemcpyDeviceToHost, st));
  ck(cudaMemcpyAsync(pw.data(), d_pw, pw.size() * 8, cudaMemcpyDeviceToHost, st));
  cudaFreeAsync(d_perm, st);
  cudaFreeAsync(d_cnt, st);
  cudaFreeAsync(d_h, st);
  cudaFreeAsync(d_pw, st);
  cudaFreeAsync(d_ls, st);
  ck(cudaStreamSynchronize(st));
  uint64_t h = kFnvBasis;
  int64_t f = 0;
  for (int64_t r = 0; r < nr; ++r) {
    // true start h = ls[r] + D, D = h - ls[r] (a multiple of 256)
    h = hend[r] + (h - ls[r]) * pw[r];
    f += cnt[r];
  }
  *checksum = h;
  *flagged = f;
}

}  // namespace tsv

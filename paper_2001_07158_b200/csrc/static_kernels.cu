// static_kernels.cu -- the static-projection engines (junction sieve used by
// the default `--preprocess both`, and the plain static sieve).
//
// Reference: /root/reference/proj/core/src/sieve.cpp static_impl :311-369 and
// junction_impl :376-473 over StaticProjection (graph.cpp:148-199).  Both are
// timestamp-free: state is dense per vertex (n x W words per layer).  A level
// is one pass over the head-sorted arc list of the projection:
//
//   out[head] ^= f_head * XOR_{arcs (tail -> head)} y(e, lvl) * g_tail * src[tail]
//
// with f = z (walks-ending family) or 1, and g = z (walks-starting family) or
// 1.  A warp owns a chunk of arcs; a head split across chunks gets partial
// sums, combined with 64-bit atomic XOR (exact: the map is linear).
#include <cuda_runtime.h>

#include "engine.hpp"
#include "gf_device.cuh"
#include "small_field.cuh"

namespace tsv {
namespace {

constexpr int kWarps = 8;
constexpr unsigned kFull = 0xffffffffu;

template <int PPT>
__device__ __forceinline__ void zvals(const uint64_t* __restrict__ zj, int k, int32_t u,
                                      uint64_t pb, uint64_t pe, uint64_t (&z)[PPT]) {
  const int lane = threadIdx.x & 31;
  const uint64_t* row = zj + static_cast<int64_t>(u) * k;
#pragma unroll
  for (int p = 0; p < PPT; ++p) z[p] = 0;
  for (int j = 0; j < k; ++j) {
    const uint64_t r = __ldg(row + j);
#pragma unroll
    for (int p = 0; p < PPT; ++p)
      if (((pb + lane + 32 * p) >> j) & 1ull) z[p] ^= r;
  }
#pragma unroll
  for (int p = 0; p < PPT; ++p)
    if (pb + lane + 32 * p >= pe) z[p] = 0;
}

template <int PPT, int BITS>
__global__ void __launch_bounds__(kWarps * 32) k_static_level(const StaticLevel P) {
  constexpr int W = 32 * PPT;
  __shared__ uint64_t s_y[kWarps][32];
  __shared__ int32_t s_head[kWarps][32], s_tail[kWarps][32];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t c = static_cast<int64_t>(blockIdx.x) * kWarps + wib;
  if (c >= P.C) return;
  const int64_t a0 = P.chunk_arc[c], a1 = P.chunk_arc[c + 1];
  const uint64_t pre = draw_prefix(P.seed, P.role);
  const uint64_t yb = static_cast<uint64_t>(P.level) + 0x165667b19e3779f9ull;
  uint64_t acc[PPT];
#pragma unroll
  for (int p = 0; p < PPT; ++p) acc[p] = 0;
  for (int64_t base = a0; base < a1; base += 32) {
    const int nb = static_cast<int>(a1 - base < 32 ? a1 - base : 32);
    int32_t h = -1, t = 0;
    uint64_t y = 0;
    if (lane < nb) {
      h = __ldg(P.arc_head + base + lane);
      t = __ldg(P.arc_tail + base + lane);
      y = fdraw_y<BITS>(pre, yb, static_cast<uint64_t>(P.level),
                        static_cast<uint32_t>(__ldg(P.arc_edge + base + lane)));
    }
    s_y[wib][lane] = y;
    s_head[wib][lane] = h;
    s_tail[wib][lane] = t;
    __syncwarp();
    for (int i = 0; i < nb; ++i) {
      const int32_t head = s_head[wib][i], tail = s_tail[wib][i];
      uint64_t val[PPT];
      if (P.src) {
#pragma unroll
        for (int p = 0; p < PPT; ++p) val[p] = __ldg(P.src + static_cast<int64_t>(tail) * W + lane + 32 * p);
      } else {
#pragma unroll
        for (int p = 0; p < PPT; ++p) val[p] = 1;  // the all-ones base layer
      }
      if (P.tail_times_z) {
        uint64_t z[PPT];
        zvals<PPT>(P.zj, P.k, tail, P.pb, P.pe, z);
#pragma unroll
        for (int p = 0; p < PPT; ++p) val[p] = P.src ? fmul<BITS>(z[p], val[p]) : z[p];
      }
      const uint64_t yy = s_y[wib][i];
#pragma unroll
      for (int p = 0; p < PPT; ++p) acc[p] ^= fmul<BITS>(yy, val[p]);
      const bool last = i + 1 >= nb || s_head[wib][i + 1] != head;  // flush per batch
      if (last) {
        if (P.head_times_z) {
          uint64_t z[PPT];
          zvals<PPT>(P.zj, P.k, head, P.pb, P.pe, z);
#pragma unroll
          for (int p = 0; p < PPT; ++p) acc[p] = fmul<BITS>(z[p], acc[p]);
        }
#pragma unroll
        for (int p = 0; p < PPT; ++p) {
          unsigned long long* dst = reinterpret_cast<unsigned long long*>(
              P.out + static_cast<int64_t>(head) * W + lane + 32 * p);
          if (acc[p]) atomicXor(dst, static_cast<unsigned long long>(acc[p]));
          acc[p] = 0;
        }
      }
    }
    __syncwarp();
  }
}

// E_1[u][w] = z_u^{pb+w}
template <int PPT>
__global__ void k_static_base(int32_t n, const uint64_t* __restrict__ zj, int k, uint64_t pb,
                              uint64_t pe, uint64_t* __restrict__ out) {
  const int64_t u = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (u >= n) return;
  uint64_t z[PPT];
  zvals<PPT>(zj, k, static_cast<int32_t>(u), pb, pe, z);
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int p = 0; p < PPT; ++p) out[u * 32 * PPT + lane + 32 * p] = z[p];
}

// acc[u] ^= XOR_w a[u][w] * b[u][w]  (b == nullptr: the all-ones layer)
template <int PPT, int BITS>
__global__ void k_static_readout(int32_t n, const uint64_t* __restrict__ a,
                                 const uint64_t* __restrict__ b, uint64_t* __restrict__ acc) {
  const int64_t u = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  if (u >= n) return;
  const int lane = threadIdx.x & 31;
  uint64_t x = 0;
#pragma unroll
  for (int p = 0; p < PPT; ++p) {
    const int64_t i = u * 32 * PPT + lane + 32 * p;
    x ^= b ? fmul<BITS>(a[i], b[i]) : a[i];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x ^= __shfl_xor_sync(kFull, x, o);
  if (lane == 0) acc[u] ^= x;
}

unsigned warps_blocks(int64_t warps) {
  return static_cast<unsigned>((warps + kWarps - 1) / kWarps);
}

}  // namespace

template <int BITS>
void static_level_bits(const StaticLevel& p, cudaStream_t st) {
  if (p.ppt == 2)
    k_static_level<2, BITS><<<warps_blocks(p.C), kWarps * 32, 0, st>>>(p);
  else
    k_static_level<1, BITS><<<warps_blocks(p.C), kWarps * 32, 0, st>>>(p);
}

void launch_static_level(const StaticLevel& p, cudaStream_t st) {
  if (p.C == 0) return;
  prof_begin("static_level", st);
  switch (p.bits) {
    case 8: static_level_bits<8>(p, st); break;
    case 16: static_level_bits<16>(p, st); break;
    case 32: static_level_bits<32>(p, st); break;
    default: static_level_bits<64>(p, st); break;
  }
  prof_end(st);
}

void launch_static_base(int32_t n, const uint64_t* zj, int k, uint64_t pb, uint64_t pe, int ppt,
                        uint64_t* out, cudaStream_t st) {
  if (n == 0) return;
  prof_begin("static_base", st);
  if (ppt == 2)
    k_static_base<2><<<warps_blocks(n), kWarps * 32, 0, st>>>(n, zj, k, pb, pe, out);
  else
    k_static_base<1><<<warps_blocks(n), kWarps * 32, 0, st>>>(n, zj, k, pb, pe, out);
  prof_end(st);
}

template <int BITS>
void static_readout_bits(int32_t n, const uint64_t* a, const uint64_t* b, int ppt, uint64_t* acc,
                         cudaStream_t st) {
  if (ppt == 2)
    k_static_readout<2, BITS><<<warps_blocks(n), kWarps * 32, 0, st>>>(n, a, b, acc);
  else
    k_static_readout<1, BITS><<<warps_blocks(n), kWarps * 32, 0, st>>>(n, a, b, acc);
}

void launch_static_readout(int32_t n, const uint64_t* a, const uint64_t* b, int ppt,
                           uint64_t* acc, cudaStream_t st, int bits) {
  if (n == 0) return;
  prof_begin("static_readout", st);
  switch (bits) {
    case 8: static_readout_bits<8>(n, a, b, ppt, acc, st); break;
    case 16: static_readout_bits<16>(n, a, b, ppt, acc, st); break;
    case 32: static_readout_bits<32>(n, a, b, ppt, acc, st); break;
    default: static_readout_bits<64>(n, a, b, ppt, acc, st); break;
  }
  prof_end(st);
}

}  // namespace tsv

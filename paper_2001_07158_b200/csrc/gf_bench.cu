// gf_bench.cu -- GF(2^64) multiply variants: self-test and throughput
// microbenchmarks (tsv_gf_mul_device / tsv_gf_bench).  The level kernels use
// the variants these numbers select ("GF(2^64) multiply").
//
// variant 0  production general multiply (gf_mul)
//         1  bit-serial reference
//         2  holes + Karatsuba
//         3  holes + schoolbook
//         4  warp-uniform multiplier, smem tables, 1 product per lane per y
//         5  ... 2 products per lane per y
//         6  ... 4 products per lane per y
#include <cuda_runtime.h>

#include "engine.hpp"
#include "gf_device.cuh"

namespace tsv {
namespace {

template <int V>
__device__ __forceinline__ uint64_t mul_v(uint64_t a, uint64_t b) {
  if (V == 1) return gf_mul_serial(a, b);
  if (V == 2) return gf_mul_kara(a, b);
  if (V == 3) return gf_mul_school(a, b);
  if (V == 9) return gf_mul_p5(a, b);
  return gf_mul(a, b);
}

__global__ void k_gf_mul(int variant, int64_t n, const uint64_t* a, const uint64_t* b,
                         uint64_t* out) {
  __shared__ __align__(256) uint64_t tabs[8][GfTable::kWords];
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (variant >= 4 && variant <= 6) {
    // products by a warp-uniform multiplier: every lane multiplies a[i] by
    // each of the warp's 32 b values in turn and keeps the one of its own
    // index, so all 32 tables are exercised.
    const int64_t base = i - lane;
    GfTable T{tabs[w]};
    uint64_t mine = 0;
    for (int j = 0; j < 32; ++j) {
      const int64_t src = base + j < n ? base + j : n - 1;
      const uint64_t y = b[src];
      __syncwarp();
      T.build(y, lane);
      __syncwarp();
      const uint64_t r = T.mul(i < n ? a[i] : 0);
      if (j == lane) mine = r;
    }
    if (i < n) out[i] = mine;
    return;
  }
  if (i >= n) return;
  switch (variant) {
    case 1: out[i] = mul_v<1>(a[i], b[i]); break;
    case 2: out[i] = mul_v<2>(a[i], b[i]); break;
    case 3: out[i] = mul_v<3>(a[i], b[i]); break;
    case 9: out[i] = mul_v<9>(a[i], b[i]); break;
    default: out[i] = mul_v<0>(a[i], b[i]); break;
  }
}

template <int V>
__global__ void k_gf_bench(int64_t iters, uint64_t* sink) {
  const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  uint64_t a0 = mix64(tid + 1), a1 = mix64(tid + 2), a2 = mix64(tid + 3), a3 = mix64(tid + 4);
  const uint64_t b = mix64(tid ^ 0x5555);
  for (int64_t it = 0; it < iters; ++it) {
    a0 = mul_v<V>(a0, b) ^ static_cast<uint64_t>(it);
    a1 = mul_v<V>(a1, b) ^ static_cast<uint64_t>(it);
    a2 = mul_v<V>(a2, b) ^ static_cast<uint64_t>(it);
    a3 = mul_v<V>(a3, b) ^ static_cast<uint64_t>(it);
  }
  sink[tid] = a0 ^ a1 ^ a2 ^ a3;
}

// Table products: per iteration the warp builds the table of a fresh y and
// each lane multiplies PPT values by it.
template <int PPT>
__global__ void k_gf_bench_table(int64_t iters, uint64_t* sink) {
  __shared__ __align__(256) uint64_t tabs[8][GfTable::kWords];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  uint64_t a[PPT];
#pragma unroll
  for (int p = 0; p < PPT; ++p) a[p] = mix64(tid * 8 + p);
  uint64_t y = mix64(blockIdx.x * 64 + w);
  GfTable T{tabs[w]};
  for (int64_t it = 0; it < iters; ++it) {
    __syncwarp();
    T.build(y, lane);
    __syncwarp();
#pragma unroll
    for (int p = 0; p < PPT; ++p) a[p] = T.mul(a[p]) ^ static_cast<uint64_t>(it);
    y = y * 0x9e3779b97f4a7c15ull + 1;
  }
  uint64_t x = 0;
#pragma unroll
  for (int p = 0; p < PPT; ++p) x ^= a[p];
  sink[tid] = x;
}

// Lane-table products (LaneTable): per iteration every lane builds the table
// of its own fresh y and multiplies PPT values by it.
template <int PPT>
__global__ void k_gf_bench_lanetab(int64_t iters, uint64_t* sink) {
  extern __shared__ uint8_t dyn_smem[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint32_t s0 = (static_cast<uint32_t>(__cvta_generic_to_shared(dyn_smem)) + 4095u) & ~4095u;
  LaneTable T;
  T.init(s0 + 4096u * w, lane);
  uint64_t a[PPT];
#pragma unroll
  for (int p = 0; p < PPT; ++p) a[p] = mix64(tid * 16 + p);
  uint64_t y = mix64(tid ^ 0x5555);
  for (int64_t it = 0; it < iters; ++it) {
#pragma unroll
    for (int p = 0; p < PPT; ++p) asm volatile("" ::"r"(lo32(a[p])));  // products done before the rebuild
    T.build(y);
    uint32_t gen;
    asm volatile("mov.u32 %0, %1;" : "=r"(gen) : "r"(static_cast<uint32_t>(it)));
#pragma unroll
    for (int p = 0; p < PPT; ++p)
      a[p] = gf_reduce124(T.clmul(a[p], gen)) ^ static_cast<uint64_t>(it);
    y = y * 0x9e3779b97f4a7c15ull + 1;
  }
  uint64_t x = 0;
#pragma unroll
  for (int p = 0; p < PPT; ++p) x ^= a[p];
  sink[tid] = x;
}

// self-test form: out[i] = a[i] * b[i] through the lane table
__global__ void k_gf_mul_lanetab(int64_t n, const uint64_t* a, const uint64_t* b, uint64_t* out) {
  extern __shared__ uint8_t dyn_smem[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint32_t s0 = (static_cast<uint32_t>(__cvta_generic_to_shared(dyn_smem)) + 4095u) & ~4095u;
  LaneTable T;
  T.init(s0 + 4096u * w, lane);
  T.build(i < n ? b[i] : 1);
  uint32_t gen;
  asm volatile("mov.u32 %0, %1;" : "=r"(gen) : "r"(0u));
  const uint64_t r = gf_reduce124(T.clmul(i < n ? a[i] : 0, gen));
  if (i < n) out[i] = r;
}

// Pipe probes: 8 independent mul.wide.u32 (V=7) or 3-input XORs (V=8) per
// iteration and thread, to calibrate the instruction costs of the variants.
template <int V>
__global__ void k_pipe_probe(int64_t iters, uint64_t* sink) {
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t a[8], b = tid * 0x9e3779b9u + 1;
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = tid * (j + 3) + 7;
  uint64_t acc = 0;
  for (int64_t it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (V == 7) {
        const uint64_t p = wmul(a[j], b);
        a[j] = static_cast<uint32_t>(p >> 32) ^ static_cast<uint32_t>(p);
      } else {
        a[j] = a[j] ^ b ^ a[(j + 1) & 7];
      }
    }
    b += 0x7f4a7c15u;
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) acc ^= a[j];
  sink[tid] = acc;
}

}  // namespace

void launch_gf_mul(int variant, int64_t n, const uint64_t* a, const uint64_t* b,
                   uint64_t* out, cudaStream_t st) {
  if (n == 0) return;
  const int threads = 256;
  const int64_t blocks = (n + threads - 1) / threads;
  if (variant == 10) {
    k_gf_mul_lanetab<<<static_cast<unsigned>(blocks), threads, 4096 * (threads / 32 + 1), st>>>(
        n, a, b, out);
    return;
  }
  k_gf_mul<<<static_cast<unsigned>(blocks), threads, 0, st>>>(variant, n, a, b, out);
}

// Returns products per launch for the given shape.
double launch_gf_bench(int variant, int64_t iters, uint64_t* sink, int blocks, int threads,
                       cudaStream_t st) {
  const double lanes = static_cast<double>(blocks) * threads;
  switch (variant) {
    case 1: k_gf_bench<1><<<blocks, threads, 0, st>>>(iters, sink); return 4.0 * iters * lanes;
    case 2: k_gf_bench<2><<<blocks, threads, 0, st>>>(iters, sink); return 4.0 * iters * lanes;
    case 3: k_gf_bench<3><<<blocks, threads, 0, st>>>(iters, sink); return 4.0 * iters * lanes;
    case 4: k_gf_bench_table<1><<<blocks, threads, 0, st>>>(iters, sink); return 1.0 * iters * lanes;
    case 5: k_gf_bench_table<2><<<blocks, threads, 0, st>>>(iters, sink); return 2.0 * iters * lanes;
    case 6: k_gf_bench_table<4><<<blocks, threads, 0, st>>>(iters, sink); return 4.0 * iters * lanes;
    case 7: k_pipe_probe<7><<<blocks, threads, 0, st>>>(iters, sink); return 8.0 * iters * lanes;
    case 8: k_pipe_probe<8><<<blocks, threads, 0, st>>>(iters, sink); return 8.0 * iters * lanes;
    case 9: k_gf_bench<9><<<blocks, threads, 0, st>>>(iters, sink); return 4.0 * iters * lanes;
    case 10: case 11: case 12: {
      // lane tables: 1 / 5 / 10 products per table build
      const size_t sm = 4096 * (static_cast<size_t>(threads) / 32 + 1);
      if (variant == 10) {
        cudaFuncSetAttribute(k_gf_bench_lanetab<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        k_gf_bench_lanetab<1><<<blocks, threads, sm, st>>>(iters, sink);
        return 1.0 * iters * lanes;
      }
      if (variant == 11) {
        cudaFuncSetAttribute(k_gf_bench_lanetab<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        k_gf_bench_lanetab<5><<<blocks, threads, sm, st>>>(iters, sink);
        return 5.0 * iters * lanes;
      }
      cudaFuncSetAttribute(k_gf_bench_lanetab<10>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      k_gf_bench_lanetab<10><<<blocks, threads, sm, st>>>(iters, sink);
      return 10.0 * iters * lanes;
    }
    default: k_gf_bench<0><<<blocks, threads, 0, st>>>(iters, sink); return 4.0 * iters * lanes;
  }
}

}  // namespace tsv

// coef_static.cu -- the static-projection sieves (the junction sieve of the
// default `--preprocess both`, and the plain static sieve) in the
// coefficient form of the temporal engine (coef_kernels.cu, top).
//
// Reference: junction_impl / static_impl, /root/reference/proj/core/src/
// sieve.cpp:311-473.  Per point A the junction sieve forms the walks-ending
// family E_l[u] (walks of l vertices ending at u, z of every vertex) and
// the walks-starting family S_b[u] (walks of b vertices starting at u, z of
// all but u) over the projection's arcs, and reads out
//   acc[u] = XOR_A XOR_{b=1..k} E_{k+1-b}[u](A) * S_b[u](A).
// E_l is a homogeneous polynomial of degree l in the point bits (one z per
// vertex of the walk, z linear), S_b of degree b-1, so every product is
// homogeneous of degree k and the XOR over all 2^k points keeps exactly the
// coefficient of the square-free top monomial (characteristic 2):
//   acc[u] = det(W) * XOR_b XOR_{|T| = k+1-b} E_{k+1-b}[u][T] * S_b[u][[k] - T]
// in the shade basis (z rows of v_{u,d}, det(W) = per(W) at the readout, as
// for the temporal engine).  The families run on coefficient rows:
//   E_1 = z,            E_l[h] = zmap_h( XOR_{t -> h} y(e, l-1) * E_{l-1}[t] )
//   S_1 = 1,            S_b[h] = XOR_{h -> v} y2(e, b-1) * zmap_v(S_{b-1}[v])
// with zmap_h(U)[T] = XOR_{j in T} z_{h,j} U[T - {j}], a row of C(k, l)
// words per vertex and level.  The static sieve is acc[u] = det * E_k[u][[k]].
//
// Arc pass: a warp owns a task of <= 256 arcs of one head (hubs of the
// power-law configs span many tasks, combined with 64-bit atomic XOR): per
// arc it builds the warp-uniform y's GfTable (2 KB of shared memory,
// gf_device.cuh) and multiplies the tail's row by it lane-strided, eight
// row loads in flight per lane.  z map pass: a warp per vertex takes
// z_{h,j} one j at a time, again as a table, over the (T - {j} -> T) pairs
// of CoefTables::jpairs.  Work per arc and level: C(k, l-1) table products
// instead of 2^k point products.
#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "coef.hpp"
#include "engine.hpp"
#include "gf_device.cuh"

namespace tsv {
namespace {

constexpr int kSW = 2;          // warps per block (2 x 17 KB of static shared memory)
constexpr int kRowMax = 924;    // C(12, 6): the largest row (k <= 12)

constexpr int kChunk = 256;     // arcs per task: hub vertices are split over warps

// Arc pass: a warp per task (<= kChunk arcs of one head) XORs
// XOR_{arcs} y(e) * src[tail] into dst[head] (zeroed; 64-bit atomics, since
// a hub's tasks run on several warps).
struct SArcs {
  int64_t ntask = 0;
  const int32_t* task_head = nullptr;
  const int64_t* task_a0 = nullptr;
  const int32_t* task_len = nullptr;
  const int32_t* tail = nullptr;
  const int32_t* edge = nullptr;
  const uint64_t* src = nullptr;      // n x E
  uint64_t* dst = nullptr;            // n x E
  int E = 0;
  uint64_t pre = 0, yb = 0;           // draw prefix (seed, role), level + round constant
};

__global__ void __launch_bounds__(kSW * 32) k_static_arcs(const SArcs P) {
  __shared__ __align__(256) uint64_t tabs[kSW][GfTable::kWords];
  __shared__ uint64_t su[kSW][kRowMax];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  GfTable T{tabs[w]};
  uint64_t* U = su[w];
  const int64_t nw = static_cast<int64_t>(gridDim.x) * kSW;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * kSW + w; i < P.ntask; i += nw) {
    const int32_t h = __ldg(P.task_head + i);
    const int64_t a0 = __ldg(P.task_a0 + i), a1 = a0 + __ldg(P.task_len + i);
    for (int e = lane; e < P.E; e += 32) U[e] = 0;
    for (int64_t a = a0; a < a1; ++a) {
      const int32_t t = __ldg(P.tail + a);
      const uint64_t y = draw_edge_y(P.pre, P.yb, static_cast<uint32_t>(__ldg(P.edge + a)));
      const uint64_t* row = P.src + static_cast<int64_t>(t) * P.E;
      __syncwarp();
      T.build(y, lane);
      __syncwarp();
      // kLd independent row loads in flight per lane (a row is up to 924
      // words; one load at a time left the pass latency-bound)
      constexpr int kLd = 8;
      for (int e0 = lane; e0 < P.E; e0 += 32 * kLd) {
        uint64_t x[kLd];
#pragma unroll
        for (int r = 0; r < kLd; ++r) {
          const int e = e0 + 32 * r;
          x[r] = e < P.E ? __ldg(row + e) : 0ull;
        }
#pragma unroll
        for (int r = 0; r < kLd; ++r)
          if (x[r]) U[e0 + 32 * r] ^= T.mul(x[r]);
      }
    }
    __syncwarp();
    uint64_t* out = P.dst + static_cast<int64_t>(h) * P.E;
    for (int e = lane; e < P.E; e += 32)
      if (U[e])
        atomicXor(reinterpret_cast<unsigned long long*>(out + e),
                  static_cast<unsigned long long>(U[e]));
  }
}

// z map per vertex: dst[h] = zmap_h(src[h]) (Ein -> Eout words), z_{h,j}
// one j at a time as a warp-uniform table over the (T - {j} -> T) pairs.
struct SZmap {
  int32_t n = 0;
  const uint64_t* src = nullptr;
  int Ein = 0;
  uint64_t* dst = nullptr;
  int Eout = 0;
  const uint64_t* zj = nullptr;
  int k = 0;
  const int2* jp = nullptr;  // k blocks of jcnt (in rank, out rank)
  int jcnt = 0;
};

__global__ void __launch_bounds__(kSW * 32) k_static_zmap(const SZmap P) {
  __shared__ __align__(256) uint64_t tabs[kSW][GfTable::kWords];
  __shared__ uint64_t su[kSW][kRowMax], ss[kSW][kRowMax];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  GfTable T{tabs[w]};
  uint64_t* U = su[w];
  uint64_t* S = ss[w];
  const int64_t nw = static_cast<int64_t>(gridDim.x) * kSW;
  for (int64_t h = static_cast<int64_t>(blockIdx.x) * kSW + w; h < P.n; h += nw) {
    bool any = false;
    for (int e = lane; e < P.Ein; e += 32) {
      U[e] = __ldg(P.src + h * P.Ein + e);
      any = any || U[e] != 0;
    }
    for (int e = lane; e < P.Eout; e += 32) S[e] = 0;
    if (__any_sync(0xffffffffu, any)) {
      for (int j = 0; j < P.k; ++j) {
        const uint64_t z = __ldg(P.zj + h * P.k + j);
        if (!z) continue;  // warp-uniform
        __syncwarp();
        T.build(z, lane);
        __syncwarp();
        const int2* pj = P.jp + static_cast<int64_t>(j) * P.jcnt;
        for (int p = lane; p < P.jcnt; p += 32) {  // T' -> T' + {j}: distinct outputs
          const int2 q = __ldg(pj + p);
          const uint64_t x = U[q.x];
          if (x) S[q.y] ^= T.mul(x);
        }
      }
    }
    __syncwarp();
    uint64_t* out = P.dst + h * P.Eout;
    for (int e = lane; e < P.Eout; e += 32) out[e] = S[e];
  }
}

// acc[u] ^= det * XOR_b XOR_{|T| = k+1-b} E_{k+1-b}[u][T] * S_b[u][comp(T)]
// (junction), or det * E_k[u][0] (static); warp per vertex
struct SReadout {
  int32_t n = 0;
  int k = 0;
  bool junction = true;
  const uint64_t* const* E = nullptr;  // E[l], l = 1..k (device array of pointers)
  const uint64_t* const* Sb = nullptr; // S[b], b = 1..k (S[1] unused: the constant 1)
  const int32_t* comp = nullptr;       // per level l: comp rank of each l-subset
  const int64_t* comp_off = nullptr;   // k+1
  const int* cnt = nullptr;            // C(k, l), l = 0..k
  uint64_t det = 1;
  uint64_t* acc = nullptr;
};

__global__ void __launch_bounds__(256) k_static_coef_readout(const SReadout R) {
  const int64_t u = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (u >= R.n) return;
  const int k = R.k;
  uint64_t x = 0;
  if (lane == 0) x = R.E[k][u];  // b = 1: E_k[u][[k]] * 1
  if (R.junction) {
    for (int b = 2; b <= k; ++b) {
      const int l = k + 1 - b;  // E_l (l-subsets) against S_b (its (b-1)-subsets)
      const int F = R.cnt[l], G = R.cnt[b - 1];
      const uint64_t* e = R.E[l] + u * F;
      const uint64_t* s = R.Sb[b] + u * G;
      const int32_t* cp = R.comp + R.comp_off[l];
      for (int o = lane; o < F; o += 32) {
        const uint64_t a = e[o];
        if (!a) continue;
        const uint64_t c = s[cp[o]];
        if (c) x ^= gf_mul(a, c);
      }
    }
  }
#pragma unroll
  for (int d = 16; d; d >>= 1) x ^= __shfl_xor_sync(0xffffffffu, x, d);
  if (lane == 0 && x) R.acc[u] ^= R.det == 1 ? x : gf_mul(R.det, x);
}

unsigned grid_for(int64_t warps) {
  const int64_t b = (warps + kSW - 1) / kSW;
  return static_cast<unsigned>(b < 148 * 64 ? b : 148 * 64);
}

}  // namespace

bool static_coef_supported(int k) { return k >= 1 && k <= 12; }

uint64_t static_coef_words(int32_t n, int k, bool junction) {
  // E_2..E_k rows (E_1 = the z table, n x k)
  uint64_t rows = 0, mx = 1;
  uint64_t c = 1;
  for (int l = 1; l <= k; ++l) {
    c = c * static_cast<uint64_t>(k - l + 1) / static_cast<uint64_t>(l);
    if (l >= 2) rows += c;
    if (c > mx) mx = c;
  }
  // + all S_b of the junction sieve (sum_b C(k, b-1), b = 2..k, kept for the
  // readout) and the arc-pass / z-map buffer
  const uint64_t srows = (junction ? (uint64_t{1} << k) - 2 : 0) + mx;
  return static_cast<uint64_t>(n) * (rows + srows + k);
}

void eval_static_coef(const StaticCoefInputs& in, cudaStream_t st,
                      const std::function<void*(size_t)>& alloc,
                      const std::function<void(void*)>& release) {
  const int k = in.k;
  const int32_t n = in.n;
  if (n == 0) return;
  const CoefTables& T = *in.tables;
  std::vector<int> cnt(static_cast<size_t>(k) + 1);
  for (int l = 0; l <= k; ++l) cnt[l] = static_cast<int>(T.count[l]);
  auto up = [&](const void* h, size_t bytes) {
    void* d = alloc(bytes ? bytes : 8);
    if (bytes && cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, st) != cudaSuccess)
      throw std::runtime_error("static coefficient sieve: upload failed");
    return d;
  };
  // jpairs per level, and the complement ranks of every level's subsets
  std::vector<const int2*> jp(static_cast<size_t>(k) + 1, nullptr);
  for (int l = 2; l <= k; ++l)
    jp[l] = static_cast<const int2*>(up(T.jpairs[l].data(), T.jpairs[l].size() * sizeof(int2)));
  std::vector<int32_t> comp;
  std::vector<int64_t> comp_off(static_cast<size_t>(k) + 1, 0);
  {
    // colex rank via binomials; subsets of each size in increasing mask order
    std::vector<std::vector<int64_t>> C(33, std::vector<int64_t>(34, 0));
    for (int a = 0; a <= 32; ++a) {
      C[a][0] = 1;
      for (int b = 1; b <= a; ++b) C[a][b] = C[a - 1][b - 1] + (b <= a - 1 ? C[a - 1][b] : 0);
    }
    auto rank = [&](uint64_t mask) {
      int64_t r = 0;
      int i = 0;
      for (int x = 0; x < k; ++x)
        if ((mask >> x) & 1ull) r += (x >= i + 1 ? C[x][i + 1] : 0), ++i;
      return r;
    };
    const uint64_t full = (1ull << k) - 1;
    for (int l = 0; l <= k; ++l) {
      comp_off[l] = static_cast<int64_t>(comp.size());
      if (l == 0) {
        comp.push_back(0);
        continue;
      }
      uint64_t m = (1ull << l) - 1;
      while (m <= full) {
        comp.push_back(static_cast<int32_t>(rank(full ^ m)));
        const uint64_t cb = m & (~m + 1), rr = m + cb;
        m = (((rr ^ m) >> 2) / cb) | rr;
      }
    }
  }
  const int32_t* d_comp = static_cast<const int32_t*>(up(comp.data(), comp.size() * 4));
  const int64_t* d_coff = static_cast<const int64_t*>(up(comp_off.data(), comp_off.size() * 8));
  const int* d_cnt = static_cast<const int*>(up(cnt.data(), cnt.size() * sizeof(int)));

  // tasks: per head, chunks of <= kChunk of its arcs (offsets n + 1)
  auto tasks = [&](const std::vector<int64_t>& off, SArcs& A) {
    std::vector<int32_t> th, tl;
    std::vector<int64_t> ta;
    for (int32_t h = 0; h < n; ++h)
      for (int64_t a = off[h]; a < off[h + 1]; a += kChunk) {
        th.push_back(h);
        ta.push_back(a);
        tl.push_back(static_cast<int32_t>(std::min<int64_t>(kChunk, off[h + 1] - a)));
      }
    A.ntask = static_cast<int64_t>(th.size());
    A.task_head = static_cast<const int32_t*>(up(th.data(), th.size() * 4));
    A.task_a0 = static_cast<const int64_t*>(up(ta.data(), ta.size() * 8));
    A.task_len = static_cast<const int32_t*>(up(tl.data(), tl.size() * 4));
  };
  int mx = 1;
  for (int l = 1; l <= k; ++l) mx = std::max(mx, cnt[l]);
  auto* ug = static_cast<uint64_t*>(alloc(static_cast<size_t>(n) * mx * 8));
  auto zmap = [&](const uint64_t* src, int lin, uint64_t* dst) {  // lin = src's subset size
    SZmap Z;
    Z.n = n;
    Z.src = src;
    Z.Ein = cnt[lin];
    Z.dst = dst;
    Z.Eout = cnt[lin + 1];
    Z.zj = in.zj;
    Z.k = k;
    Z.jp = jp[lin + 1];
    Z.jcnt = cnt[lin] * (k - lin) / k;  // C(k-1, lin)
    prof_begin("static_coef_zmap", st);
    k_static_zmap<<<grid_for(n), kSW * 32, 0, st>>>(Z);
    prof_end(st);
  };
  auto arcs = [&](SArcs A, const uint64_t* src, uint64_t* dst, int E, uint64_t role, int lvl) {
    A.src = src;
    A.dst = dst;
    A.E = E;
    A.pre = draw_prefix(in.seed, role);
    A.yb = static_cast<uint64_t>(lvl) + 0x165667b19e3779f9ull;
    cudaMemsetAsync(dst, 0, static_cast<size_t>(n) * E * 8, st);
    if (!A.ntask) return;
    prof_begin("static_coef_arcs", st);
    k_static_arcs<<<grid_for(A.ntask), kSW * 32, 0, st>>>(A);
    prof_end(st);
  };

  // walks-ending family E_2..E_k (E_1 = z): E_l = zmap(XOR_{t -> h} y E_{l-1}[t])
  SArcs IN, OUT;
  IN.tail = in.in_tail;
  IN.edge = in.in_edge;
  OUT.tail = in.out_tail;
  OUT.edge = in.out_edge;
  tasks(*in.h_in_off, IN);
  std::vector<uint64_t*> E(static_cast<size_t>(k) + 1, nullptr);
  E[1] = const_cast<uint64_t*>(in.zj);
  for (int l = 2; l <= k; ++l) {
    E[l] = static_cast<uint64_t*>(alloc(static_cast<size_t>(n) * cnt[l] * 8));
    arcs(IN, E[l - 1], ug, cnt[l - 1], kRoleEdgeY, l - 1);
    zmap(ug, l - 1, E[l]);
  }
  // walks-starting family S_2..S_k (S_1 = 1): S_b[h] = XOR_{h -> v} y2 * zmap_v(S_{b-1}[v])
  // (zmap(S_1) = z); every S_b is kept for the readout
  std::vector<uint64_t*> Sb(static_cast<size_t>(k) + 1, nullptr);
  if (in.junction) {
    tasks(*in.h_out_off, OUT);
    for (int b = 2; b <= k; ++b) {
      const uint64_t* Z = in.zj;
      if (b > 2) {
        zmap(Sb[b - 1], b - 2, ug);
        Z = ug;
      }
      Sb[b] = static_cast<uint64_t*>(alloc(static_cast<size_t>(n) * cnt[b - 1] * 8));
      arcs(OUT, Z, Sb[b], cnt[b - 1], 4 /* Role::edge_y2 */, b - 1);
    }
  }
  SReadout R;
  R.n = n;
  R.k = k;
  R.junction = in.junction;
  std::vector<const uint64_t*> Eh(E.begin(), E.end()), Sh(Sb.begin(), Sb.end());
  R.E = static_cast<const uint64_t* const*>(up(Eh.data(), Eh.size() * 8));
  R.Sb = static_cast<const uint64_t* const*>(up(Sh.data(), Sh.size() * 8));
  R.comp = d_comp;
  R.comp_off = d_coff;
  R.cnt = d_cnt;
  R.det = in.det;
  R.acc = in.acc;
  prof_begin("static_coef_readout", st);
  k_static_coef_readout<<<static_cast<unsigned>((static_cast<int64_t>(n) * 32 + 255) / 256), 256,
                          0, st>>>(R);
  prof_end(st);
  if (cudaGetLastError() != cudaSuccess)
    throw std::runtime_error("static coefficient sieve: launch failed");
  // (device buffers go back through `release` with the caller's stream)
  for (int l = 2; l <= k; ++l) release(E[l]);
  for (int b = 2; b <= k; ++b)
    if (Sb[b]) release(Sb[b]);
  release(ug);
}

}  // namespace tsv

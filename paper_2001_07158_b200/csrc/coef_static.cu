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
// A warp owns a head vertex: per arc it builds the warp-uniform y's GfTable
// (2 KB of shared memory, gf_device.cuh) and multiplies the tail's row by it
// lane-strided; the z map takes z_{h,j} one j at a time, again as a table,
// over the (T - {j} -> T) pairs of CoefTables::jpairs.  Work per arc and
// level: C(k, l-1) table products instead of 2^k point products.
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

struct SLevel {
  int64_t nlist = 0;                  // heads to process
  const int32_t* list = nullptr;      // head ids (nullptr: 0 .. nlist-1)
  const int64_t* off = nullptr;       // n+1: arcs of head h at [off[h], off[h+1]); nullptr: no arcs
  const int32_t* tail = nullptr;
  const int32_t* edge = nullptr;
  const uint64_t* src = nullptr;      // n x Ein
  int Ein = 0;
  uint64_t* dst = nullptr;            // n x Eout
  int Eout = 0;
  uint64_t pre = 0, yb = 0;           // draw prefix (seed, role), level + round constant
  const uint64_t* zj = nullptr;       // n x k; nullptr: no z map (Eout == Ein)
  int k = 0;
  const int2* jp = nullptr;           // k blocks of C(k-1, Ein's size) (in rank, out rank)
  int jcnt = 0;
  bool self = false;                  // U = src[h] (vertex z map, no arcs)
};

__global__ void __launch_bounds__(kSW * 32) k_static_coef(const SLevel P) {
  __shared__ __align__(256) uint64_t tabs[kSW][GfTable::kWords];
  __shared__ uint64_t su[kSW][kRowMax], ss[kSW][kRowMax];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  GfTable T{tabs[w]};
  uint64_t* U = su[w];
  uint64_t* S = ss[w];
  const int64_t nw = static_cast<int64_t>(gridDim.x) * kSW;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * kSW + w; i < P.nlist; i += nw) {
    const int32_t h = P.list ? P.list[i] : static_cast<int32_t>(i);
    if (P.self) {
      for (int e = lane; e < P.Ein; e += 32) U[e] = P.src[static_cast<int64_t>(h) * P.Ein + e];
    } else {
      for (int e = lane; e < P.Ein; e += 32) U[e] = 0;
      const int64_t a0 = P.off[h], a1 = P.off[h + 1];
      for (int64_t a = a0; a < a1; ++a) {
        const int32_t t = __ldg(P.tail + a);
        const uint64_t y = draw_edge_y(P.pre, P.yb, static_cast<uint32_t>(__ldg(P.edge + a)));
        const uint64_t* row = P.src + static_cast<int64_t>(t) * P.Ein;
        __syncwarp();
        T.build(y, lane);
        __syncwarp();
        for (int e = lane; e < P.Ein; e += 32) {
          const uint64_t x = __ldg(row + e);
          if (x) U[e] ^= T.mul(x);
        }
      }
    }
    __syncwarp();
    uint64_t* out = P.dst + static_cast<int64_t>(h) * P.Eout;
    if (!P.zj) {
      for (int e = lane; e < P.Eout; e += 32) out[e] = U[e];
      continue;
    }
    for (int e = lane; e < P.Eout; e += 32) S[e] = 0;
    for (int j = 0; j < P.k; ++j) {
      const uint64_t z = __ldg(P.zj + static_cast<int64_t>(h) * P.k + j);
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
    __syncwarp();
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
  // readout) and one z-mapped buffer
  const uint64_t srows = junction ? (uint64_t{1} << k) - 2 + mx : 0;
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

  // walks-ending family E_2..E_k (E_1 = z)
  std::vector<uint64_t*> E(static_cast<size_t>(k) + 1, nullptr);
  E[1] = const_cast<uint64_t*>(in.zj);
  SLevel L;
  L.zj = in.zj;
  L.k = k;
  for (int l = 2; l <= k; ++l) {
    E[l] = static_cast<uint64_t*>(alloc(static_cast<size_t>(n) * cnt[l] * 8));
    cudaMemsetAsync(E[l], 0, static_cast<size_t>(n) * cnt[l] * 8, st);
    L.nlist = n;  // heads without arcs write zero rows
    L.list = nullptr;
    L.off = in.in_off;
    L.tail = in.in_tail;
    L.edge = in.in_edge;
    L.src = E[l - 1];
    L.Ein = cnt[l - 1];
    L.dst = E[l];
    L.Eout = cnt[l];
    L.pre = draw_prefix(in.seed, kRoleEdgeY);
    L.yb = static_cast<uint64_t>(l - 1) + 0x165667b19e3779f9ull;
    L.jp = jp[l];
    L.jcnt = cnt[l - 1] * (k - l + 1) / k;  // C(k-1, l-1)
    L.self = false;
    if (L.nlist) {
      prof_begin("static_coef", st);
      k_static_coef<<<grid_for(L.nlist), kSW * 32, 0, st>>>(L);
      prof_end(st);
    }
  }
  // walks-starting family S_2..S_k (S_1 = 1): Z_b = zmap_v(S_{b-1}) per
  // vertex (Z_2 = z), then S_b[h] = XOR_{h -> v} y2 * Z_b[v]
  std::vector<uint64_t*> Sb(static_cast<size_t>(k) + 1, nullptr);
  if (in.junction) {
    uint64_t* zbuf = nullptr;
    for (int b = 2; b <= k; ++b) {
      const uint64_t* Z = in.zj;  // b = 2: zmap(1) = z
      if (b > 2) {
        zbuf = static_cast<uint64_t*>(alloc(static_cast<size_t>(n) * cnt[b - 1] * 8));
        SLevel V;
        V.nlist = n;
        V.src = Sb[b - 1];
        V.Ein = cnt[b - 2];
        V.dst = zbuf;
        V.Eout = cnt[b - 1];
        V.zj = in.zj;
        V.k = k;
        V.jp = jp[b - 1];
        V.jcnt = cnt[b - 2] * (k - b + 2) / k;  // C(k-1, b-2)
        V.self = true;
        prof_begin("static_coef", st);
        k_static_coef<<<grid_for(n), kSW * 32, 0, st>>>(V);
        prof_end(st);
        Z = zbuf;
      }
      Sb[b] = static_cast<uint64_t*>(alloc(static_cast<size_t>(n) * cnt[b - 1] * 8));
      cudaMemsetAsync(Sb[b], 0, static_cast<size_t>(n) * cnt[b - 1] * 8, st);
      SLevel O;
      O.nlist = n;
      O.list = nullptr;
      O.off = in.out_off;
      O.tail = in.out_tail;
      O.edge = in.out_edge;
      O.src = Z;
      O.Ein = cnt[b - 1];
      O.dst = Sb[b];
      O.Eout = cnt[b - 1];
      O.pre = draw_prefix(in.seed, 4);  // Role::edge_y2 (gf.hpp:116)
      O.yb = static_cast<uint64_t>(b - 1) + 0x165667b19e3779f9ull;
      O.zj = nullptr;
      if (O.nlist) {
        prof_begin("static_coef", st);
        k_static_coef<<<grid_for(O.nlist), kSW * 32, 0, st>>>(O);
        prof_end(st);
      }
      if (zbuf) {
        release(zbuf);
        zbuf = nullptr;
      }
      // S_{b-1} is still needed by the readout: all S_b are kept (they are
      // the smaller half of the rows: sum_b C(k, b-1) = 2^k - C(k, k))
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
}

}  // namespace tsv

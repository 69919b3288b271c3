// build_kernels.cu -- on-device construction of the engine's graph layout
// (the host build of TemporalGraph does not scale to 1e9
// edges).  Produces exactly the arrays of layout.cpp:
//
//   canonical edges  drop self-loops, orient u<v (undirected), sort by
//                    (ts,u,v), drop duplicates: edge id = index
//                    (/root/reference/proj/core/src/graph.cpp:22-43)
//   arcs             (head, tail, edge) stably sorted by head over edge
//                    order = (head, ts) order; runs = (head, ts) groups
//   arc_src          tail's last run with ts' < ts (binary search)
//
// Non-instant edge models (sieve.cpp:257-291; canonical input only): an arc
// departing at ts lands in slot ts + eps - 1 of its head (runs are (head,
// slot) groups) and reads its tail's state at ts - delta(tail), delta = the
// vertex delay (delay models) or 1; at level 2 it needs ts - delta >= 0.
//   chunks           fixed arc ranges; a vertex split by a chunk boundary is
//                    repaired by k_fixup, exactly like a split hub
//
// Sorting uses CUB's radix sort (library primitive shipped with the CUDA
// toolkit); everything else is our own kernels.
#include <cuda_runtime.h>

#include <cub/cub.cuh>

#include <functional>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>

#include "engine.hpp"
#include "layout.hpp"

namespace tsv {
namespace {

constexpr int kT = 256;

// TSV_TRACE_BUILD=1: phase times of the device build on stderr
struct BuildTrace {
  bool on = false;
  cudaStream_t st;
  std::chrono::steady_clock::time_point t0;
  explicit BuildTrace(cudaStream_t s) : st(s), t0(std::chrono::steady_clock::now()) {
    const char* e = std::getenv("TSV_TRACE_BUILD");
    on = e && e[0] == '1';
  }
  void mark(const char* what) {
    if (!on) return;
    cudaStreamSynchronize(st);
    const double ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    std::fprintf(stderr, "[build] %-28s %9.1f ms\n", what, ms);
  }
};

unsigned nblk(int64_t n) { return static_cast<unsigned>((n + kT - 1) / kT); }

int bits_for(uint64_t x) {  // bits needed to represent values < x + 1
  int b = 1;
  while (b < 64 && (x >> b)) ++b;
  return b;
}

__global__ void k_validate_orient(int64_t m, int32_t n, const int32_t* __restrict__ u,
                                  const int32_t* __restrict__ v, const int32_t* __restrict__ ts,
                                  int directed, uint64_t* __restrict__ key_uv,
                                  uint32_t* __restrict__ key_ts, uint8_t* __restrict__ keep,
                                  BuildStatus* st) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= m) return;
  int32_t a = u[i], b = v[i];
  const int32_t t = ts[i];
  if (a < 0 || a >= n || b < 0 || b >= n) {
    atomicMin(reinterpret_cast<unsigned long long*>(&st->first_bad_endpoint),
              static_cast<unsigned long long>(i));
    keep[i] = 0;
    return;
  }
  if (t < 1) {
    atomicMin(reinterpret_cast<unsigned long long*>(&st->first_bad_ts),
              static_cast<unsigned long long>(i));
    keep[i] = 0;
    return;
  }
  if (a == b) {  // (t = 0 takes the largest timestamp of the edges kept)
    atomicAdd(reinterpret_cast<unsigned long long*>(&st->self_loops), 1ull);
    keep[i] = 0;
    return;
  }
  atomicMax(&st->max_ts, t);
  if (!directed && a > b) {
    const int32_t s = a;
    a = b;
    b = s;
  }
  key_uv[i] = static_cast<uint64_t>(a) * static_cast<uint64_t>(n) + static_cast<uint64_t>(b);
  key_ts[i] = static_cast<uint32_t>(t);
  keep[i] = 1;
}

// canonical-input variant: validate order instead of sorting
__global__ void k_check_canonical(int64_t m, int32_t n, const int32_t* __restrict__ u,
                                  const int32_t* __restrict__ v, const int32_t* __restrict__ ts,
                                  int directed, BuildStatus* st) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const int32_t a = u[i], b = v[i], t = ts[i];
  if (a < 0 || a >= n || b < 0 || b >= n) {
    atomicMin(reinterpret_cast<unsigned long long*>(&st->first_bad_endpoint),
              static_cast<unsigned long long>(i));
    return;
  }
  if (t < 1) {
    atomicMin(reinterpret_cast<unsigned long long*>(&st->first_bad_ts),
              static_cast<unsigned long long>(i));
    return;
  }
  atomicMax(&st->max_ts, t);
  bool ok = a != b && (directed || a < b);
  if (i > 0) {
    const int32_t pa = u[i - 1], pb = v[i - 1], pt = ts[i - 1];
    ok = ok && (pt != t ? pt < t : pa != a ? pa < a : pb < b);
  }
  if (!ok) atomicExch(&st->not_canonical, 1);
}

__global__ void k_unique_flags(int64_t m, const uint32_t* __restrict__ kts,
                               const uint64_t* __restrict__ kuv, uint8_t* __restrict__ flag) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= m) return;
  flag[i] = (i == 0 || kts[i] != kts[i - 1] || kuv[i] != kuv[i - 1]) ? 1 : 0;
}

__global__ void k_unpack_edges(int64_t m, int32_t n, const uint32_t* __restrict__ kts,
                               const uint64_t* __restrict__ kuv, int32_t* __restrict__ eu,
                               int32_t* __restrict__ ev, int32_t* __restrict__ ets) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const uint64_t k = kuv[i];
  eu[i] = static_cast<int32_t>(k / static_cast<uint64_t>(n));
  ev[i] = static_cast<int32_t>(k % static_cast<uint64_t>(n));
  ets[i] = static_cast<int32_t>(kts[i]);
}

// arcs in edge order: (head v, tail u) [+ (head u, tail v) when undirected]
__global__ void k_make_arcs(int64_t m, int directed, const int32_t* __restrict__ eu,
                            const int32_t* __restrict__ ev, uint32_t* __restrict__ head,
                            uint32_t* __restrict__ idx) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= m) return;
  if (directed) {
    head[i] = static_cast<uint32_t>(ev[i]);
    idx[i] = static_cast<uint32_t>(i);
  } else {
    head[2 * i] = static_cast<uint32_t>(ev[i]);
    idx[2 * i] = static_cast<uint32_t>(2 * i);
    head[2 * i + 1] = static_cast<uint32_t>(eu[i]);
    idx[2 * i + 1] = static_cast<uint32_t>(2 * i + 1);
  }
}

// Landing slot of edge e: ts + eps - 1 under transition-time models.
__device__ __forceinline__ int32_t slot_of(const int32_t* __restrict__ ets,
                                           const int32_t* __restrict__ eps, uint32_t e) {
  if (!eps) return ets[e];
  const int64_t s = static_cast<int64_t>(ets[e]) + eps[e] - 1;
  return s > INT32_MAX ? INT32_MAX : static_cast<int32_t>(s);
}

// (head << 32 | slot) keys of the arcs in edge order (transition models,
// where slots are not monotone in edge order)
__global__ void k_arc_keys(int64_t m, int directed, const int32_t* __restrict__ eu,
                           const int32_t* __restrict__ ev, const int32_t* __restrict__ ets,
                           const int32_t* __restrict__ eps, uint64_t* __restrict__ key,
                           uint32_t* __restrict__ idx) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const uint64_t s = static_cast<uint32_t>(slot_of(ets, eps, static_cast<uint32_t>(i)));
  if (directed) {
    key[i] = (static_cast<uint64_t>(ev[i]) << 32) | s;
    idx[i] = static_cast<uint32_t>(i);
  } else {
    key[2 * i] = (static_cast<uint64_t>(ev[i]) << 32) | s;
    idx[2 * i] = static_cast<uint32_t>(2 * i);
    key[2 * i + 1] = (static_cast<uint64_t>(eu[i]) << 32) | s;
    idx[2 * i + 1] = static_cast<uint32_t>(2 * i + 1);
  }
}

__global__ void k_key_heads(int64_t A, const uint64_t* __restrict__ key,
                            uint32_t* __restrict__ head) {
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j < A) head[j] = static_cast<uint32_t>(key[j] >> 32);
}

// After the sort by (head, slot): tail/edge/slot of every arc, run starts.
__global__ void k_arc_fields(int64_t A, int directed, const uint32_t* __restrict__ head,
                             const uint32_t* __restrict__ idx, const int32_t* __restrict__ eu,
                             const int32_t* __restrict__ ev, const int32_t* __restrict__ ets,
                             const int32_t* __restrict__ eps,
                             int32_t* __restrict__ tail, int32_t* __restrict__ edge,
                             int32_t* __restrict__ ats, int32_t* __restrict__ run_start) {
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= A) return;
  const uint32_t a = idx[j];
  const uint32_t e = directed ? a : (a >> 1);
  const bool second = !directed && (a & 1u);
  tail[j] = second ? ev[e] : eu[e];
  edge[j] = static_cast<int32_t>(e);
  const int32_t t = slot_of(ets, eps, e);
  ats[j] = t;
  int32_t start = 1;
  if (j > 0) {
    const uint32_t pa = idx[j - 1];
    const int32_t pt = slot_of(ets, eps, directed ? pa : (pa >> 1));
    start = (head[j] != head[j - 1] || pt != t) ? 1 : 0;
  }
  run_start[j] = start;
}

// run_id = inclusive scan of run_start - 1; scatter run heads / timestamps
__global__ void k_runs(int64_t A, const uint32_t* __restrict__ head,
                       const int32_t* __restrict__ ats, const int32_t* __restrict__ run_start,
                       const int32_t* __restrict__ run_incl, int32_t* __restrict__ run_head,
                       int32_t* __restrict__ run_ts) {
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= A || !run_start[j]) return;
  const int32_t r = run_incl[j] - 1;
  run_head[r] = static_cast<int32_t>(head[j]);
  run_ts[r] = ats[j];
}

// vtx_run_off[u] = first run with head >= u
__global__ void k_vtx_off(int32_t n, int64_t R, const int32_t* __restrict__ run_head,
                          int32_t* __restrict__ off) {
  const int64_t u = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (u > n) return;
  int64_t lo = 0, hi = R;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (run_head[mid] < u) lo = mid + 1;
    else hi = mid;
  }
  off[u] = static_cast<int32_t>(lo);
}

__global__ void k_arc_src_meta(int64_t A, const uint32_t* __restrict__ head,
                               int32_t* __restrict__ tail, const int32_t* __restrict__ edge,
                               const int32_t* __restrict__ ets,
                               const int32_t* __restrict__ delay,
                               const int32_t* __restrict__ run_start,
                               const int32_t* __restrict__ run_ts,
                               const int32_t* __restrict__ vtx_run_off,
                               int32_t* __restrict__ arc_src, uint32_t* __restrict__ arc_meta) {
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= A) return;
  const int32_t x = tail[j];
  // the tail's state is read at ts - delta (instant: ts - 1)
  const int64_t back = static_cast<int64_t>(ets[edge[j]]) - (delay ? delay[x] : 1);
  int32_t lo = vtx_run_off[x], hi = vtx_run_off[x + 1];
  const int32_t base = lo;
  while (lo < hi) {  // first run of x with slot > back
    const int32_t mid = lo + ((hi - lo) >> 1);
    if (run_ts[mid] <= back) lo = mid + 1;
    else hi = mid;
  }
  arc_src[j] = lo == base ? -1 : lo - 1;
  if (back < 0) tail[j] = -1;  // level 2 reads z_tail only at ts - delta >= 0
  uint32_t meta = static_cast<uint32_t>(edge[j]);
  if (j == 0 || head[j] != head[j - 1]) meta |= kVStart;
  if (j + 1 == A || run_start[j + 1]) meta |= kRunEnd;
  arc_meta[j] = meta;
}

__global__ void k_vstart_flags(int64_t A, const uint32_t* __restrict__ meta,
                               uint8_t* __restrict__ f) {
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j < A) f[j] = (meta[j] & kVStart) ? 1 : 0;
}

// Chunk boundary near c*ch: the next vertex start if it is within ch/2,
// else c*ch itself (a long vertex is split; k_fixup repairs its prefix).
// Strictly increasing in c except possibly at the final A.
__global__ void k_chunk_bounds(int64_t C0, int64_t A, int64_t ch,
                               const int64_t* __restrict__ vs, int64_t nv,
                               int64_t* __restrict__ bounds) {
  const int64_t c = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c > C0) return;
  const int64_t t = c * ch < A ? c * ch : A;
  if (c == C0 || t == A) {
    bounds[c] = A;
    return;
  }
  int64_t lo = 0, hi = nv;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (vs[mid] < t) lo = mid + 1;
    else hi = mid;
  }
  const int64_t cand = lo < nv ? vs[lo] : A;
  bounds[c] = (cand - t <= ch / 2) ? cand : t;
}

__global__ void k_chunks(int64_t C, int64_t R, const int64_t* __restrict__ chunk_arc,
                         const int32_t* __restrict__ run_incl, const uint32_t* __restrict__ meta,
                         int32_t* __restrict__ chunk_run, uint8_t* __restrict__ chunk_carry) {
  const int64_t c = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c > C) return;
  const int64_t a = chunk_arc[c];
  if (c == C) {
    chunk_run[c] = static_cast<int32_t>(R);
    return;
  }
  // runs completed before arc a = id of a's run (0-based): earlier runs are
  // complete, a's own run ends at or after a
  chunk_run[c] = run_incl[a] - 1;
  chunk_carry[c] = (meta[a] & kVStart) ? 0 : 1;
}

__global__ void k_restrict_flags(int64_t m, const int32_t* __restrict__ eu,
                                 const int32_t* __restrict__ ev, const int32_t* __restrict__ ets,
                                 const uint8_t* __restrict__ keep, int32_t max_ts,
                                 uint8_t* __restrict__ f) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < m) f[i] = (ets[i] <= max_ts && keep[eu[i]] && keep[ev[i]]) ? 1 : 0;
}

__global__ void k_shaded_mask(int32_t n, const int32_t* __restrict__ off,
                              uint8_t* __restrict__ keep) {
  const int64_t u = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (u < n) keep[u] = off[u + 1] > off[u] ? 1 : 0;
}

__global__ void k_remap_edge_ids(int64_t A, uint32_t* __restrict__ meta,
                                 const int32_t* __restrict__ oid) {
  const int64_t a = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (a >= A) return;
  const uint32_t mt = meta[a];
  meta[a] = (mt & ~kEdgeMask) | static_cast<uint32_t>(oid[mt & kEdgeMask]);
}

}  // namespace

void launch_shaded_mask(int32_t n, const int32_t* off, uint8_t* keep, cudaStream_t st) {
  if (n > 0) k_shaded_mask<<<nblk(n), kT, 0, st>>>(n, off, keep);
}

void launch_remap_edge_ids(int64_t A, uint32_t* meta, const int32_t* oid, cudaStream_t st) {
  if (A > 0) k_remap_edge_ids<<<nblk(A), kT, 0, st>>>(A, meta, oid);
}

int64_t device_restrict(const int32_t* eu, const int32_t* ev, const int32_t* ets, int64_t m,
                        const uint8_t* d_keep, int32_t max_ts, int32_t* ou, int32_t* ov,
                        int32_t* ots, cudaStream_t st,
                        const std::function<void*(size_t)>& alloc,
                        const std::function<void(void*)>& release, int32_t* oid) {
  if (m == 0) return 0;
  uint8_t* f = static_cast<uint8_t*>(alloc(m));
  int64_t* cnt = static_cast<int64_t*>(alloc(8));
  k_restrict_flags<<<nblk(m), kT, 0, st>>>(m, eu, ev, ets, d_keep, max_ts, f);
  size_t tmp = 0;
  cub::DeviceSelect::Flagged(nullptr, tmp, eu, f, ou, cnt, m, st);
  void* t = alloc(tmp ? tmp : 8);
  cub::DeviceSelect::Flagged(t, tmp, eu, f, ou, cnt, m, st);
  cub::DeviceSelect::Flagged(t, tmp, ev, f, ov, cnt, m, st);
  cub::DeviceSelect::Flagged(t, tmp, ets, f, ots, cnt, m, st);
  if (oid) cub::DeviceSelect::Flagged(t, tmp, cub::CountingInputIterator<int32_t>(0), f, oid, cnt,
                                      m, st);
  int64_t kept = 0;
  cudaMemcpyAsync(&kept, cnt, 8, cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  release(t);
  release(cnt);
  release(f);
  return kept;
}

// Stable radix sort of (key, value) pairs with CUB; keys/values are swapped
// into the DoubleBuffer's current buffers.
template <typename K, typename V>
static void radix_pairs(cub::DoubleBuffer<K>& k, cub::DoubleBuffer<V>& v, int64_t n, int end_bit,
                        cudaStream_t st) {
  size_t tmp = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp, k, v, n, 0, end_bit, st);
  void* d_tmp = nullptr;
  if (cudaMallocAsync(&d_tmp, tmp ? tmp : 8, st) != cudaSuccess)
    throw std::runtime_error("device graph build: out of memory (sort)");
  cub::DeviceRadixSort::SortPairs(d_tmp, tmp, k, v, n, 0, end_bit, st);
  cudaFreeAsync(d_tmp, st);
}

void device_build(const int32_t* d_u, const int32_t* d_v, const int32_t* d_ts, int64_t m,
                  int32_t n, bool directed, bool canonical, DeviceLayout& out,
                  BuildStatus* d_status, int sm_count, cudaStream_t st,
                  const std::function<void*(size_t)>& alloc,
                  const std::function<void(void*)>& release, const int32_t* d_eps,
                  const int32_t* d_delay) {
  BuildTrace tr(st);
  auto A32 = [&](int64_t cnt) { return static_cast<int32_t*>(alloc(std::max<int64_t>(cnt, 1) * 4)); };
  BuildStatus init{};
  init.first_bad_endpoint = INT64_MAX;
  init.first_bad_ts = INT64_MAX;
  cudaMemcpyAsync(d_status, &init, sizeof(init), cudaMemcpyHostToDevice, st);

  int32_t *eu = nullptr, *ev = nullptr, *ets = nullptr;
  int64_t mc = m;
  if (canonical) {
    if (m) k_check_canonical<<<nblk(m), kT, 0, st>>>(m, n, d_u, d_v, d_ts, directed, d_status);
    eu = A32(m);
    ev = A32(m);
    ets = A32(m);
    cudaMemcpyAsync(eu, d_u, m * 4, cudaMemcpyDeviceToDevice, st);
    cudaMemcpyAsync(ev, d_v, m * 4, cudaMemcpyDeviceToDevice, st);
    cudaMemcpyAsync(ets, d_ts, m * 4, cudaMemcpyDeviceToDevice, st);
  } else {
    // keys, drop loops/invalid, sort by (ts, u, v), unique
    uint64_t* kuv[2] = {static_cast<uint64_t*>(alloc(std::max<int64_t>(m, 1) * 8)),
                        static_cast<uint64_t*>(alloc(std::max<int64_t>(m, 1) * 8))};
    uint32_t* kts[2] = {static_cast<uint32_t*>(alloc(std::max<int64_t>(m, 1) * 4)),
                        static_cast<uint32_t*>(alloc(std::max<int64_t>(m, 1) * 4))};
    uint8_t* keep = static_cast<uint8_t*>(alloc(std::max<int64_t>(m, 1)));
    if (m)
      k_validate_orient<<<nblk(m), kT, 0, st>>>(m, n, d_u, d_v, d_ts, directed ? 1 : 0, kuv[0],
                                                kts[0], keep, d_status);
    // compact kept edges
    int64_t* d_cnt = static_cast<int64_t*>(alloc(8));
    {
      size_t tmp = 0;
      cub::DeviceSelect::Flagged(nullptr, tmp, kuv[0], keep, kuv[1], d_cnt, m, st);
      void* t = alloc(tmp ? tmp : 8);
      cub::DeviceSelect::Flagged(t, tmp, kuv[0], keep, kuv[1], d_cnt, m, st);
      cub::DeviceSelect::Flagged(t, tmp, kts[0], keep, kts[1], d_cnt, m, st);
      release(t);
    }
    cudaMemcpyAsync(&mc, d_cnt, 8, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    release(keep);
    const uint64_t nn = static_cast<uint64_t>(n) * static_cast<uint64_t>(n);
    BuildStatus hs{};
    cudaMemcpy(&hs, d_status, sizeof(hs), cudaMemcpyDeviceToHost);
    cub::DoubleBuffer<uint64_t> buv(kuv[1], kuv[0]);
    cub::DoubleBuffer<uint32_t> bts(kts[1], kts[0]);
    if (mc > 0 && hs.first_bad_endpoint == INT64_MAX && hs.first_bad_ts == INT64_MAX) {
      // pass 1: by (u, v); pass 2 (stable): by ts
      tr.mark("validate + compact");
      radix_pairs(buv, bts, mc, bits_for(nn ? nn - 1 : 0), st);
      tr.mark("sort by (u, v)");
      radix_pairs(bts, buv, mc, bits_for(static_cast<uint64_t>(hs.max_ts)), st);
      tr.mark("sort by ts");
    }
    uint8_t* flag = static_cast<uint8_t*>(alloc(std::max<int64_t>(mc, 1)));
    if (mc) k_unique_flags<<<nblk(mc), kT, 0, st>>>(mc, bts.Current(), buv.Current(), flag);
    {
      size_t tmp = 0;
      cub::DeviceSelect::Flagged(nullptr, tmp, buv.Current(), flag, buv.Alternate(), d_cnt, mc, st);
      void* t = alloc(tmp ? tmp : 8);
      cub::DeviceSelect::Flagged(t, tmp, buv.Current(), flag, buv.Alternate(), d_cnt, mc, st);
      cub::DeviceSelect::Flagged(t, tmp, bts.Current(), flag, bts.Alternate(), d_cnt, mc, st);
      release(t);
    }
    int64_t mu = 0;
    cudaMemcpyAsync(&mu, d_cnt, 8, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    out.dropped_duplicates = mc - mu;
    mc = mu;
    eu = A32(mc);
    ev = A32(mc);
    ets = A32(mc);
    if (mc) k_unpack_edges<<<nblk(mc), kT, 0, st>>>(mc, n, bts.Alternate(), buv.Alternate(), eu, ev, ets);
    release(flag);
    release(d_cnt);
    release(kuv[0]);
    release(kuv[1]);
    release(kts[0]);
    release(kts[1]);
  }
  tr.mark("unique + unpack");
  out.m = mc;
  out.eu = eu;
  out.ev = ev;
  out.ets = ets;

  // ---- arcs, runs -----------------------------------------------------------
  const int64_t A = directed ? mc : 2 * mc;
  out.A = A;
  uint32_t* hd[2] = {static_cast<uint32_t*>(alloc(std::max<int64_t>(A, 1) * 4)),
                     static_cast<uint32_t*>(alloc(std::max<int64_t>(A, 1) * 4))};
  uint32_t* ix[2] = {static_cast<uint32_t*>(alloc(std::max<int64_t>(A, 1) * 4)),
                     static_cast<uint32_t*>(alloc(std::max<int64_t>(A, 1) * 4))};
  cub::DoubleBuffer<uint32_t> bh(hd[0], hd[1]), bi(ix[0], ix[1]);
  if (!d_eps) {
    // stable by head over edge order = (head, ts) order
    if (mc) k_make_arcs<<<nblk(mc), kT, 0, st>>>(mc, directed ? 1 : 0, eu, ev, hd[0], ix[0]);
    if (A) radix_pairs(bh, bi, A, bits_for(static_cast<uint64_t>(n)), st);
  } else {
    // transition times: sort by (head, slot)
    uint64_t* ky[2] = {static_cast<uint64_t*>(alloc(std::max<int64_t>(A, 1) * 8)),
                       static_cast<uint64_t*>(alloc(std::max<int64_t>(A, 1) * 8))};
    if (mc) k_arc_keys<<<nblk(mc), kT, 0, st>>>(mc, directed ? 1 : 0, eu, ev, ets, d_eps, ky[0], ix[0]);
    cub::DoubleBuffer<uint64_t> bk(ky[0], ky[1]);
    if (A) radix_pairs(bk, bi, A, 32 + bits_for(static_cast<uint64_t>(n)), st);
    if (A) k_key_heads<<<nblk(A), kT, 0, st>>>(A, bk.Current(), bh.Current());
    cudaStreamSynchronize(st);
    release(ky[0]);
    release(ky[1]);
  }
  const uint32_t* head = bh.Current();
  int32_t* tail = A32(A);
  int32_t* edge = A32(A);
  int32_t* ats = A32(A);
  int32_t* run_start = A32(A + 1);
  int32_t* run_incl = A32(A + 1);
  if (A)
    k_arc_fields<<<nblk(A), kT, 0, st>>>(A, directed ? 1 : 0, head, bi.Current(), eu, ev, ets,
                                         d_eps, tail, edge, ats, run_start);
  {
    size_t tmp = 0;
    cub::DeviceScan::InclusiveSum(nullptr, tmp, run_start, run_incl, A, st);
    void* t = alloc(tmp ? tmp : 8);
    if (A) cub::DeviceScan::InclusiveSum(t, tmp, run_start, run_incl, A, st);
    release(t);
  }
  int32_t R32 = 0;
  if (A) cudaMemcpyAsync(&R32, run_incl + A - 1, 4, cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  const int64_t R = R32;
  out.R = R;
  out.run_head = A32(R);
  out.run_ts = A32(R);
  if (A) k_runs<<<nblk(A), kT, 0, st>>>(A, head, ats, run_start, run_incl, out.run_head, out.run_ts);
  out.vtx_run_off = A32(static_cast<int64_t>(n) + 1);
  k_vtx_off<<<nblk(static_cast<int64_t>(n) + 1), kT, 0, st>>>(n, R, out.run_head, out.vtx_run_off);
  out.arc_src = A32(A);
  out.arc_meta = reinterpret_cast<uint32_t*>(A32(A));
  if (A)
    k_arc_src_meta<<<nblk(A), kT, 0, st>>>(A, head, tail, edge, ets, d_delay, run_start,
                                           out.run_ts, out.vtx_run_off, out.arc_src,
                                           out.arc_meta);
  out.arc_tail = tail;

  tr.mark("arcs: sort, runs, sources");
  // ---- chunks ---------------------------------------------------------------
  int64_t ch = A / (static_cast<int64_t>(std::max(sm_count, 1)) * 64);
  ch = std::min<int64_t>(2048, std::max<int64_t>(64, ch));
  const int64_t C0 = A ? (A + ch - 1) / ch : 0;
  int64_t C = 0;
  {
    // vertex starts -> boundaries aligned to them where possible
    uint8_t* vf = static_cast<uint8_t*>(alloc(std::max<int64_t>(A, 1)));
    int64_t* vs = static_cast<int64_t*>(alloc(std::max<int64_t>(A, 1) * 8));
    int64_t* cnt = static_cast<int64_t*>(alloc(8));
    if (A) k_vstart_flags<<<nblk(A), kT, 0, st>>>(A, out.arc_meta, vf);
    cub::CountingInputIterator<int64_t> it(0);
    size_t tmp = 0;
    cub::DeviceSelect::Flagged(nullptr, tmp, it, vf, vs, cnt, A, st);
    void* t = alloc(tmp ? tmp : 8);
    if (A) cub::DeviceSelect::Flagged(t, tmp, it, vf, vs, cnt, A, st);
    release(t);
    int64_t nv = 0;
    if (A) cudaMemcpyAsync(&nv, cnt, 8, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    int64_t* bounds = static_cast<int64_t*>(alloc((C0 + 1) * 8));
    k_chunk_bounds<<<nblk(C0 + 1), kT, 0, st>>>(C0, A, ch, vs, nv, bounds);
    out.chunk_arc = static_cast<int64_t*>(alloc((C0 + 1) * 8));
    tmp = 0;
    cub::DeviceSelect::Unique(nullptr, tmp, bounds, out.chunk_arc, cnt, C0 + 1, st);
    t = alloc(tmp ? tmp : 8);
    cub::DeviceSelect::Unique(t, tmp, bounds, out.chunk_arc, cnt, C0 + 1, st);
    release(t);
    int64_t nb = 1;
    cudaMemcpyAsync(&nb, cnt, 8, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    C = A ? nb - 1 : 0;
    release(vf);
    release(vs);
    release(cnt);
    release(bounds);
  }
  out.C = C;
  out.chunk_run = A32(C + 1);
  out.chunk_carry = static_cast<uint8_t*>(alloc(std::max<int64_t>(C, 1)));
  k_chunks<<<nblk(C + 1), kT, 0, st>>>(C, R, out.chunk_arc, run_incl, out.arc_meta,
                                       out.chunk_run, out.chunk_carry);
  int32_t* cidx = A32(C);
  int32_t* ccnt = A32(1);
  out.carry_list = A32(C);
  {
    cub::CountingInputIterator<int32_t> it(0);
    size_t tmp = 0;
    cub::DeviceSelect::Flagged(nullptr, tmp, it, out.chunk_carry, out.carry_list, ccnt, C, st);
    void* t = alloc(tmp ? tmp : 8);
    if (C) cub::DeviceSelect::Flagged(t, tmp, it, out.chunk_carry, out.carry_list, ccnt, C, st);
    release(t);
  }
  int32_t nc = 0;
  if (C) cudaMemcpyAsync(&nc, ccnt, 4, cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  out.ncarry = nc;
  release(cidx);
  release(ccnt);
  release(edge);
  release(ats);
  release(run_start);
  release(run_incl);
  release(hd[0]);
  release(hd[1]);
  tr.mark("chunks");
  release(ix[0]);
  release(ix[1]);
}

namespace {

__global__ void k_mark_src(int64_t A, const int32_t* __restrict__ arc_src,
                           int32_t* __restrict__ flag, unsigned long long* counts) {
  const int64_t a = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int32_t s = a < A ? arc_src[a] : -1;
  if (s >= 0) flag[s] = 1;
  const unsigned c = __popc(__ballot_sync(0xffffffffu, s >= 0));
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(counts, static_cast<unsigned long long>(c));
}

__global__ void k_mark_last_run(int32_t n, const int32_t* __restrict__ vro,
                                int32_t* __restrict__ flag) {
  const int64_t v = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v < n && vro[v + 1] > vro[v]) flag[vro[v + 1] - 1] = 1;
}

__global__ void k_slots(int64_t R, const int32_t* __restrict__ flag,
                        const int32_t* __restrict__ excl, int32_t* __restrict__ slot,
                        unsigned long long* counts) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= R) return;
  slot[r] = flag[r] ? excl[r] : -1;
  if (r == R - 1) counts[1] = static_cast<unsigned long long>(excl[r] + flag[r]);
}

__global__ void k_src_to_slot(int64_t A, int32_t* __restrict__ arc_src,
                              const int32_t* __restrict__ slot) {
  const int64_t a = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (a >= A) return;
  const int32_t s = arc_src[a];
  if (s >= 0) arc_src[a] = slot[s];
}

}  // namespace

namespace {

__global__ void k_run_end_flags(int64_t A, const uint32_t* __restrict__ meta,
                                int32_t* __restrict__ f) {
  const int64_t a = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (a < A) f[a] = (meta[a] & kRunEnd) ? 1 : 0;
}

// arc a lies in run (number of run ends before it); its edge (u, v, ts):
// directed -> (tail, head); undirected -> the arc with tail < head writes
__global__ void k_edges_from_arcs(int64_t A, int directed, const uint32_t* __restrict__ meta,
                                  const int32_t* __restrict__ tail,
                                  const int32_t* __restrict__ ends_before,
                                  const int32_t* __restrict__ run_head,
                                  const int32_t* __restrict__ run_ts, int32_t* __restrict__ eu,
                                  int32_t* __restrict__ ev, int32_t* __restrict__ ets) {
  const int64_t a = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (a >= A) return;
  const int32_t r = ends_before[a];
  const int32_t h = run_head[r], t = tail[a];
  if (!directed && t > h) return;
  const uint32_t e = meta[a] & kEdgeMask;
  eu[e] = t;
  ev[e] = h;
  ets[e] = run_ts[r];
}

}  // namespace

void edges_from_layout(const DevGraph& g, bool directed, int32_t* eu, int32_t* ev, int32_t* ets,
                       cudaStream_t st) {
  const int64_t A = g.A;
  if (A == 0) return;
  constexpr int kTb = 256;
  const unsigned blocks = static_cast<unsigned>((A + kTb - 1) / kTb);
  int32_t *f = nullptr, *ex = nullptr;
  void* tmp = nullptr;
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, f, ex, A, st);
  if (cudaMallocAsync(&f, A * 4, st) != cudaSuccess ||
      cudaMallocAsync(&ex, A * 4, st) != cudaSuccess ||
      cudaMallocAsync(&tmp, tb ? tb : 8, st) != cudaSuccess)
    throw std::runtime_error("edge reconstruction: out of device memory");
  k_run_end_flags<<<blocks, kTb, 0, st>>>(A, g.arc_meta, f);
  cub::DeviceScan::ExclusiveSum(tmp, tb, f, ex, A, st);
  k_edges_from_arcs<<<blocks, kTb, 0, st>>>(A, directed ? 1 : 0, g.arc_meta, g.arc_tail, ex,
                                            g.run_head, g.run_ts, eu, ev, ets);
  cudaFreeAsync(f, st);
  cudaFreeAsync(ex, st);
  cudaFreeAsync(tmp, st);
}

SlotCounts build_run_slots(int64_t A, int64_t R, int32_t* arc_src, int32_t* run_slot,
                           cudaStream_t st, const int32_t* vtx_run_off, int32_t n) {
  SlotCounts out;
  if (R == 0) return out;
  constexpr int kT = 256;
  auto nblk = [](int64_t n) { return static_cast<unsigned>((n + kT - 1) / kT); };
  int32_t *flag = nullptr, *excl = nullptr;
  unsigned long long* counts = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, flag, excl, R, st);
  if (cudaMallocAsync(&flag, R * 4, st) != cudaSuccess ||
      cudaMallocAsync(&excl, R * 4, st) != cudaSuccess ||
      cudaMallocAsync(&counts, 16, st) != cudaSuccess ||
      cudaMallocAsync(&tmp, tmp_bytes ? tmp_bytes : 8, st) != cudaSuccess)
    throw std::runtime_error("state slots: out of device memory");
  cudaMemsetAsync(flag, 0, R * 4, st);
  cudaMemsetAsync(counts, 0, 16, st);
  if (A) k_mark_src<<<nblk(A), kT, 0, st>>>(A, arc_src, flag, counts);
  if (vtx_run_off && n > 0) k_mark_last_run<<<nblk(n), kT, 0, st>>>(n, vtx_run_off, flag);
  cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, flag, excl, R, st);
  k_slots<<<nblk(R), kT, 0, st>>>(R, flag, excl, run_slot, counts);
  if (A) k_src_to_slot<<<nblk(A), kT, 0, st>>>(A, arc_src, run_slot);
  unsigned long long hc[2] = {0, 0};
  cudaMemcpyAsync(hc, counts, 16, cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(flag, st);
  cudaFreeAsync(excl, st);
  cudaFreeAsync(counts, st);
  cudaFreeAsync(tmp, st);
  if (cudaStreamSynchronize(st) != cudaSuccess)
    throw std::runtime_error("state slots: device error");
  out.arcs_with_src = static_cast<int64_t>(hc[0]);
  out.slots = static_cast<int64_t>(hc[1]);
  return out;
}


// ---- static projection (graph.cpp:148-199): distinct (a, b) pairs of the
// canonical edges (a < b for undirected graphs), ascending, each with the
// ids of its temporal edges in increasing order ---------------------------

namespace {

__global__ void k_static_keys(int64_t m, int32_t n, int directed, const int32_t* __restrict__ u,
                              const int32_t* __restrict__ v, uint64_t* __restrict__ key,
                              int32_t* __restrict__ id) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= m) return;
  int32_t a = u[i], b = v[i];
  if (!directed && a > b) {
    const int32_t t = a;
    a = b;
    b = t;
  }
  key[i] = static_cast<uint64_t>(a) * static_cast<uint64_t>(n) + static_cast<uint64_t>(b);
  id[i] = static_cast<int32_t>(i);
}

__global__ void k_static_heads(int64_t m, const uint64_t* __restrict__ key,
                               int32_t* __restrict__ flag) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < m) flag[i] = (i == 0 || key[i] != key[i - 1]) ? 1 : 0;
}

__global__ void k_static_emit(int64_t m, int32_t n, const uint64_t* __restrict__ key,
                              const int32_t* __restrict__ flag, const int32_t* __restrict__ rank,
                              int32_t* __restrict__ a, int32_t* __restrict__ b,
                              int32_t* __restrict__ off) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= m || !flag[i]) return;
  const int32_t j = rank[i];
  a[j] = static_cast<int32_t>(key[i] / static_cast<uint64_t>(n));
  b[j] = static_cast<int32_t>(key[i] % static_cast<uint64_t>(n));
  off[j] = static_cast<int32_t>(i);
}

}  // namespace

int64_t static_projection(const int32_t* u, const int32_t* v, int64_t m, int32_t n, bool directed,
                          int32_t* a, int32_t* b, int32_t* off, int32_t* back, cudaStream_t st,
                          const std::function<void*(size_t)>& alloc,
                          const std::function<void(void*)>& release) {
  if (m == 0) return 0;
  auto* k0 = static_cast<uint64_t*>(alloc(static_cast<size_t>(m) * 8));
  auto* k1 = static_cast<uint64_t*>(alloc(static_cast<size_t>(m) * 8));
  auto* i0 = static_cast<int32_t*>(alloc(static_cast<size_t>(m) * 4));
  k_static_keys<<<nblk(m), kT, 0, st>>>(m, n, directed ? 1 : 0, u, v, k0, i0);
  // stable radix sort by key; ties keep edge-id order (std::stable_sort)
  cub::DoubleBuffer<uint64_t> bk(k0, k1);
  cub::DoubleBuffer<int32_t> bv(i0, back);
  const uint64_t nn = static_cast<uint64_t>(n);
  radix_pairs(bk, bv, m, bits_for(nn * nn ? nn * nn - 1 : 0), st);
  if (bv.Current() != back)
    cudaMemcpyAsync(back, bv.Current(), static_cast<size_t>(m) * 4, cudaMemcpyDeviceToDevice, st);
  const uint64_t* ks = bk.Current();
  auto* flag = static_cast<int32_t*>(alloc(static_cast<size_t>(m) * 4));
  auto* rank = static_cast<int32_t*>(alloc(static_cast<size_t>(m) * 4));
  k_static_heads<<<nblk(m), kT, 0, st>>>(m, ks, flag);
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, flag, rank, m, st);
  void* t = alloc(tb ? tb : 8);
  cub::DeviceScan::ExclusiveSum(t, tb, flag, rank, m, st);
  release(t);
  int32_t last[2] = {0, 0};
  cudaMemcpyAsync(&last[0], rank + (m - 1), 4, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(&last[1], flag + (m - 1), 4, cudaMemcpyDeviceToHost, st);
  k_static_emit<<<nblk(m), kT, 0, st>>>(m, n, ks, flag, rank, a, b, off);
  if (cudaStreamSynchronize(st) != cudaSuccess)
    throw std::runtime_error("static projection: device error");
  const int64_t ms = static_cast<int64_t>(last[0]) + last[1];
  const int32_t mm = static_cast<int32_t>(m);
  cudaMemcpyAsync(off + ms, &mm, 4, cudaMemcpyHostToDevice, st);
  cudaStreamSynchronize(st);
  release(k0);
  release(k1);
  release(i0);
  release(flag);
  release(rank);
  return ms;
}

}  // namespace tsv

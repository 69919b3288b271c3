// tsv_abi.cu -- the extern "C" boundary of libtsv.so (declared in include/tsv.h).
//
// Host orchestration of the sieve: graph upload, shade upload, z-table build,
// batch loop over sieve points, level passes, readout, finalize.  Errors are
// reported as status codes plus a thread-local message; the C++ drop-in
// rethrows them as the reference's exception types.
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/tsv.h"
#include "coef.hpp"
#include "engine.hpp"
#include "gf_device.cuh"
#include "layout.hpp"

namespace {

thread_local std::string g_error;

struct CapError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define TSV_CUDA(x)                                                           \
  do {                                                                        \
    cudaError_t e_ = (x);                                                     \
    if (e_ != cudaSuccess)                                                    \
      throw CudaError(std::string(#x) + ": " + cudaGetErrorString(e_));       \
  } while (0)

template <typename F>
int guard(F&& f) {
  try {
    f();
    return TSV_OK;
  } catch (const std::invalid_argument& e) {
    g_error = e.what();
    return TSV_ERR_INVALID;
  } catch (const CapError& e) {
    g_error = e.what();
    return TSV_ERR_CAP;
  } catch (const CudaError& e) {
    g_error = e.what();
    return TSV_ERR_CUDA;
  } catch (const std::exception& e) {
    g_error = e.what();
    return TSV_ERR_CUDA;
  }
}

// ---- profiling -------------------------------------------------------------

struct ProfRec {
  std::string name;
  cudaEvent_t a, b;
};
std::mutex g_prof_mu;
bool g_prof_on = false;
std::vector<ProfRec> g_prof;
thread_local const char* g_prof_open = nullptr;
thread_local cudaEvent_t g_prof_open_ev = nullptr;
std::atomic<int64_t> g_launches{0};

template <typename T>
T* dalloc(size_t count) {
  T* p = nullptr;
  if (count == 0) count = 1;
  TSV_CUDA(cudaMalloc(&p, count * sizeof(T)));
  return p;
}

template <typename T>
T* dupload(const std::vector<T>& v) {
  T* p = dalloc<T>(v.size());
  if (!v.empty())
    TSV_CUDA(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  return p;
}

// Stream-ordered allocation that, when the device is full, gives the free
// cached state buffers (below) and the pool's unused memory back and tries
// once more: a vertex-path evaluation leaves tens of GB in that cache, which
// another engine's state must be able to claim.
bool alloc_retry(void** p, size_t bytes, cudaStream_t st);

struct DevBuf {
  void* p = nullptr;
  cudaStream_t st = nullptr;
  DevBuf() = default;
  DevBuf(size_t bytes, cudaStream_t s) : st(s) {
    if (!alloc_retry(&p, bytes ? bytes : 8, s)) TSV_CUDA(cudaErrorMemoryAllocation);
  }
  ~DevBuf() {
    if (p) cudaFreeAsync(p, st);
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

// The coefficient engine's two big state buffers (C5: 2 x 38 GB) come from
// a per-device cache that keeps them across evaluations -- also across
// graphs: a fresh graph's evaluation would otherwise re-map tens of GB
// through the stream-ordered pool (0.2-3 s at C5 in the end-to-end legs).
// A buffer is reused when large enough and free; its last user's stream
// work is ordered before the next user's by an event.  Small buffers go
// through the pool as before.
struct StateBuf {
  void* p = nullptr;
  size_t bytes = 0;
  int dev = -1;
  cudaStream_t st = nullptr;
  StateBuf(size_t want, cudaStream_t s);
  ~StateBuf();
  StateBuf(const StateBuf&) = delete;
  StateBuf& operator=(const StateBuf&) = delete;
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

namespace {
struct CachedState {
  int dev;
  void* p;
  size_t bytes;
  bool busy;
  cudaEvent_t done;  // recorded on the last user's stream at release
};
std::mutex g_state_mu;
std::vector<CachedState> g_state;
constexpr size_t kStateCacheMin = size_t{1} << 30;  // cache buffers >= 1 GiB
constexpr int kStateCacheMax = 8;
}  // namespace

// bytes of this device's free cached state buffers (a vertex-path
// evaluation's state comes out of them, so they count as available)
size_t cached_state_free(int dev) {
  std::lock_guard<std::mutex> lk(g_state_mu);
  size_t b = 0;
  for (const CachedState& c : g_state)
    if (c.dev == dev && !c.busy) b += c.bytes;
  return b;
}

// Frees this device's cached state buffers that are not in use; returns
// the bytes released.
size_t drop_free_cached_state(int dev) {
  std::lock_guard<std::mutex> lk(g_state_mu);
  size_t b = 0;
  for (size_t i = 0; i < g_state.size();) {
    CachedState& c = g_state[i];
    if (c.dev == dev && !c.busy) {
      cudaEventSynchronize(c.done);
      cudaEventDestroy(c.done);
      cudaFree(c.p);
      b += c.bytes;
      g_state.erase(g_state.begin() + static_cast<long>(i));
    } else {
      ++i;
    }
  }
  return b;
}

bool alloc_retry(void** p, size_t bytes, cudaStream_t st) {
  if (cudaMallocAsync(p, bytes, st) == cudaSuccess) return true;
  cudaGetLastError();
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  drop_free_cached_state(dev);
  cudaMemPool_t pool = nullptr;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    cudaDeviceSynchronize();
    cudaMemPoolTrimTo(pool, 0);
  }
  if (cudaMallocAsync(p, bytes, st) == cudaSuccess) return true;
  cudaGetLastError();
  *p = nullptr;
  return false;
}

StateBuf::StateBuf(size_t want, cudaStream_t s) : st(s) {
  TSV_CUDA(cudaGetDevice(&dev));
  want = want ? want : 8;
  if (want >= kStateCacheMin && !std::getenv("TSV_NO_STATE_CACHE")) {
    std::lock_guard<std::mutex> lk(g_state_mu);
    int best = -1;
    for (size_t i = 0; i < g_state.size(); ++i) {
      const CachedState& c = g_state[i];
      if (c.dev == dev && !c.busy && c.bytes >= want &&
          (best < 0 || c.bytes < g_state[best].bytes))
        best = static_cast<int>(i);
    }
    if (best >= 0) {
      CachedState& c = g_state[best];
      c.busy = true;
      TSV_CUDA(cudaStreamWaitEvent(st, c.done, 0));
      p = c.p;
      bytes = c.bytes;
      return;
    }
    // make room: drop free cached buffers of this device that are too small
    for (size_t i = 0; i < g_state.size();) {
      CachedState& c = g_state[i];
      if (c.dev == dev && !c.busy) {
        cudaEventSynchronize(c.done);
        cudaEventDestroy(c.done);
        cudaFree(c.p);
        g_state.erase(g_state.begin() + static_cast<long>(i));
      } else {
        ++i;
      }
    }
    if (static_cast<int>(g_state.size()) < kStateCacheMax) {
      void* q = nullptr;
      if (cudaMalloc(&q, want) != cudaSuccess) {
        // the stream-ordered pool may hold the memory: trim it and retry,
        // else fall back to a pool allocation
        cudaGetLastError();
        cudaMemPool_t pool = nullptr;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
          cudaDeviceSynchronize();
          cudaMemPoolTrimTo(pool, 0);
        }
        if (cudaMalloc(&q, want) != cudaSuccess) {
          cudaGetLastError();
          TSV_CUDA(cudaMallocAsync(&p, want, st));
          bytes = 0;
          return;
        }
      }
      cudaEvent_t e = nullptr;
      TSV_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      g_state.push_back({dev, q, want, true, e});
      p = q;
      bytes = want;
      return;
    }
  }
  if (!alloc_retry(&p, want, st)) TSV_CUDA(cudaErrorMemoryAllocation);
  bytes = 0;  // pool allocation (not cached)
}

StateBuf::~StateBuf() {
  if (!p) return;
  if (!bytes) {
    cudaFreeAsync(p, st);
    return;
  }
  std::lock_guard<std::mutex> lk(g_state_mu);
  for (CachedState& c : g_state)
    if (c.p == p) {
      cudaEventRecord(c.done, st);
      c.busy = false;
    }
}

// The state buffers (2*R*W words, up to ~130 GB at 1e9 edges) are stream-
// ordered allocations; keep freed pool memory mapped so repeated
// evaluations (probes, repetitions, steps) do not re-map it every time.
void keep_pool_memory(int dev) {
  static std::mutex mu;
  static std::vector<int> done;
  std::lock_guard<std::mutex> lk(mu);
  if (std::find(done.begin(), done.end(), dev) != done.end()) return;
  cudaMemPool_t pool = nullptr;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t keep = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    // evaluations on concurrent streams (repetitions, probes) must not be
    // chained by the pool: no new stream dependencies to reuse a block freed
    // on another stream (same-stream reuse and completed frees still apply)
    int no = 0;
    cudaMemPoolSetAttribute(pool, cudaMemPoolReuseAllowInternalDependencies, &no);
  }
  done.push_back(dev);
}

struct DeviceGuard {
  int prev = 0;
  explicit DeviceGuard(int dev) {
    TSV_CUDA(cudaGetDevice(&prev));
    if (prev != dev) TSV_CUDA(cudaSetDevice(dev));
    keep_pool_memory(dev);
  }
  ~DeviceGuard() { cudaSetDevice(prev); }
};

}  // namespace

namespace tsv {

void prof_begin(const char* name, cudaStream_t st) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (!g_prof_on) return;
  cudaEventCreate(&g_prof_open_ev);
  cudaEventRecord(g_prof_open_ev, st);
  g_prof_open = name;
}

void prof_end(cudaStream_t st) {
  if (!g_prof_on || !g_prof_open) return;
  cudaEvent_t e;
  cudaEventCreate(&e);
  cudaEventRecord(e, st);
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_prof.push_back({g_prof_open, g_prof_open_ev, e});
  g_prof_open = nullptr;
}

}  // namespace tsv

inline uint64_t next_graph_uid() {
  static std::atomic<uint64_t> ctr{1};
  return ctr.fetch_add(1);
}

struct tsv_shades {
  int k = 0;
  int32_t n = 0;
  int64_t single = 0;  // vertices with exactly one shade (engine choice)
  int64_t multi = 0;   // vertices with several shades
  int device = 0;
  int32_t* off = nullptr;
  int32_t* shades = nullptr;
  // the graph restricted to vertices with a shade (same vertex and edge ids),
  // built once per (graph, shades) by shaded_subgraph(), for the last few
  // graphs (uid); a null subgraph = not worth it / not applicable.  Callers
  // hold the shared_ptr while they enqueue work on it; freeing a graph runs
  // cudaFree, which waits for the kernels still reading it.
  struct SubEntry {
    uint64_t uid;
    std::shared_ptr<tsv_graph> sub;
  };
  mutable std::mutex sub_mu;
  mutable std::vector<SubEntry> subs;
  // the n x k table v_{u,d} of the shade basis per seed, with det(W), for the
  // level-by-level (multi-GPU) entry point
  struct ZjEntry {
    uint64_t seed;
    uint64_t* d;
    uint64_t det;
  };
  mutable std::mutex zj_mu;
  mutable std::vector<ZjEntry> zjs;
  ~tsv_shades() {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    for (auto& z : zjs) cudaFree(z.d);
    cudaFree(off);
    cudaFree(shades);
    cudaSetDevice(prev);
  }
};

struct tsv_graph {
  // process-unique id (a freed graph's address may be reused by a new one)
  const uint64_t uid = next_graph_uid();
  tsv::HostLayout host;  // n, t, directed, drop counts (+ canonical edges if host-built)
  tsv::DevGraph dev;
  int device = 0;
  int64_t device_bytes = 0;
  int64_t m = 0;                      // canonical edge count
  int model = 0;                      // edge model the layout was built for
  bool edges_in_layout = false;       // canonical edges only implied by the layout
  int64_t arcs_with_src = 0, runs_referenced = 0;
  const int32_t* d_eu = nullptr;      // canonical edges on the device (device build)
  const int32_t* d_ev = nullptr;
  const int32_t* d_ets = nullptr;
  std::vector<void*> owned;
  // last shade table evaluated on this graph (binary-search and self-
  // reduction probes repeat it): reused only when the caller's CSR equals a
  // host copy of the cached one word for word (parallel compare)
  mutable std::mutex shade_mu;
  mutable std::shared_ptr<tsv_shades> shade_cache;
  mutable std::vector<int32_t> shade_off_copy, shade_vs_copy;
  mutable int shade_k = 0;
  mutable bool shade_uniform = false;  // cached CSR = every vertex shade_upat
  mutable int32_t shade_uc = 0;
  mutable std::vector<int32_t> shade_upat;
  // stream of the synchronous entry points (created once per graph)
  mutable std::mutex stream_mu;
  mutable cudaStream_t api_stream = nullptr;
  // vertex-lane coefficient engine (coef_vertex.cu): per (rank, world)
  // partition -- its work list and state-slot range -- built on first use;
  // applicable = false when the graph has hub vertices
  struct VertPart {
    int rank = 0, world = 1;
    bool applicable = false;
    tsv::VertList vl;
    int32_t v_lo = 0, v_hi = 0;
    int64_t slot_lo = 0, slot_hi = 0;
    std::vector<void*> owned;
    bool xlists = false;  // exchange lists built
    tsv::ExchangeLists xl;
  };
  mutable std::mutex vl_mu;
  mutable std::vector<std::unique_ptr<VertPart>> parts;
  ~tsv_graph() {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    if (api_stream) cudaStreamDestroy(api_stream);
    for (auto& vp : parts)
      for (void* p : vp->owned) cudaFree(p);
    for (void* p : owned) cudaFree(p);
    cudaSetDevice(prev);
  }
};

namespace {

template <typename T>
const T* own_upload(tsv_graph* g, const std::vector<T>& v) {
  T* p = dupload(v);
  g->owned.push_back(p);
  g->device_bytes += static_cast<int64_t>(std::max<size_t>(v.size(), 1) * sizeof(T));
  return p;
}

// small_ok: the entry point evaluates GF(2^8 / 2^16 / 2^32) too (the
// temporal sieve, small_field.cu); the others are GF(2^64) only.
void check_config(const tsv_config* cfg, bool small_ok = false) {
  if (!cfg) throw std::invalid_argument("null config");
  if (cfg->field_bits != 8 && cfg->field_bits != 16 && cfg->field_bits != 32 &&
      cfg->field_bits != 64)
    throw std::invalid_argument("field_bits must be 8, 16, 32 or 64");
  if (cfg->field_bits != 64 && !small_ok)
    throw std::invalid_argument(
        "field_bits 8/16/32 are evaluated by the temporal sieve only (this sieve is GF(2^64))");
  const int W = cfg->lane_width;
  if (W < 1 || W > 256 || (W & (W - 1)))
    throw std::invalid_argument("lane_width must be a power of two in [1,256]");
  if (cfg->edge_model < 0 || cfg->edge_model > 3)
    throw std::invalid_argument("edge_model must be 0..3");
  const int ppb = cfg->points_per_batch;
  if (ppb != 0 && (ppb < 1 || ppb > 128 || (ppb & (ppb - 1))))
    throw std::invalid_argument("points_per_batch must be 0 or a power of two <= 128");
}

tsv::Batch batch_shape(int W) {
  tsv::Batch b;
  if (W >= 32) {
    b.lanes = 32;
    b.ppt = W / 32;
  } else {
    b.lanes = W;
    b.ppt = 1;
  }
  return b;
}

// Device words an evaluation may allocate: 92% of free memory plus freed
// (reusable) pool memory.
uint64_t device_budget_words() {
  size_t free_b = 0, total_b = 0;
  TSV_CUDA(cudaMemGetInfo(&free_b, &total_b));
  int dev = 0;
  cudaMemPool_t pool = nullptr;
  if (cudaGetDevice(&dev) == cudaSuccess &&
      cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t reserved = 0, used = 0;  // freed pool memory is reusable
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved);
    cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used);
    if (reserved > used) free_b += reserved - used;
  }
  return static_cast<uint64_t>(free_b * 0.92) / 8;
}

// Does a working set of `words` fit next to what is allocated?  A set below
// 1/8 of the device is taken as fitting without a cudaMemGetInfo query (the
// query is not free: on the bench's deep stream queues it blocked the host).
bool fits_device(uint64_t words) {
  static std::mutex mu;
  static std::vector<std::pair<int, size_t>> total;
  int dev = 0;
  TSV_CUDA(cudaGetDevice(&dev));
  size_t tb = 0;
  {
    std::lock_guard<std::mutex> lk(mu);
    for (auto& t : total)
      if (t.first == dev) tb = t.second;
    if (!tb) {
      size_t f = 0;
      TSV_CUDA(cudaMemGetInfo(&f, &tb));
      total.emplace_back(dev, tb);
    }
  }
  if (words * 8 <= tb / 8) return true;
  return words <= device_budget_words();
}

// Points per batch: the largest power of two <= min(range, 128) whose
// working set fits the word cap and free device memory.
// *zb_ok: the per-batch z table (n*W words) also fits next to that working set.
// *lanes: 2 when there are several batches and two working sets fit, so that
// consecutive batches run on two streams (their kernels overlap), else 1.
int choose_width(const tsv_graph* g, int k, uint64_t range, const tsv_config* cfg,
                 uint64_t* peak_words, bool* zb_ok, int* lanes) {
  // state rows = referenced runs (slots); R is kept for the z-table rule
  const uint64_t R = static_cast<uint64_t>(g->dev.R), C = static_cast<uint64_t>(g->dev.C);
  const uint64_t S = static_cast<uint64_t>(g->dev.S);
  const uint64_t n = static_cast<uint64_t>(g->dev.n);
  auto words = [&](uint64_t W) {
    return (k >= 2 ? 2 * S * W + C * W : 0) + n * static_cast<uint64_t>(k) + n;
  };
  int W = cfg->points_per_batch ? cfg->points_per_batch : 128;
  while (static_cast<uint64_t>(W) > range && W > 1) W >>= 1;
  const uint64_t budget = device_budget_words();
  if (cfg->points_per_batch == 0)
    while (W > 1 && (words(W) > cfg->memory_cap_words || words(W) > budget)) W >>= 1;
  // z table only when small next to the state (n <= R/8) and it fits
  const uint64_t zw = n * static_cast<uint64_t>(W);
  *zb_ok = k >= 2 && n * 8 <= R && words(W) + zw <= budget &&
           words(W) + zw <= cfg->memory_cap_words;
  *peak_words = words(W) + (*zb_ok ? zw : 0);
  *lanes = 1;
  const uint64_t lane_words = words(W) - n * static_cast<uint64_t>(k) - n + (*zb_ok ? zw : 0);
  if (range > static_cast<uint64_t>(W) && *peak_words + lane_words <= budget &&
      *peak_words + lane_words <= cfg->memory_cap_words && !std::getenv("TSV_ONE_LANE")) {
    *lanes = 2;
    *peak_words += lane_words;
  }
  if (words(W) > cfg->memory_cap_words)
    throw CapError("sieve memory cap exceeded: needs " + std::to_string(words(W)) +
                   " field words, cap " + std::to_string(cfg->memory_cap_words));
  return W;
}

// Vertex-ordered sieve (vc_impl): positional z, per-level color filter.
struct VcSpec {
  const int32_t* d_colors = nullptr;  // n primary colors (device)
  std::vector<int32_t> order;         // k colors, position-exact
  int32_t wild = -1;                  // wildcard color, -1 = none
};

std::shared_ptr<tsv_graph> shaded_subgraph(const tsv_graph* g, const tsv_shades* sh);
tsv_graph* device_graph_build(int32_t n, int64_t m, const int32_t* u, const int32_t* v,
                              const int32_t* ts, bool directed, int32_t t, int device,
                              bool canonical, bool on_device = false,
                              const int32_t* eps = nullptr, const int32_t* delays = nullptr,
                              int model = 0, bool force_last_runs = false);
void copy_to_host(void* dst, const void* d_src, size_t bytes, cudaStream_t st);
void copy_to_device(void* d_dst, const void* src, size_t bytes, cudaStream_t st);

// Subset-index tables of the coefficient engine for one k (host).
const tsv::CoefTables& coef_const_tables(int k) {
  static std::mutex mu;
  static std::vector<std::unique_ptr<tsv::CoefTables>> tabs(31);
  std::lock_guard<std::mutex> lk(mu);
  if (!tabs[k]) tabs[k] = std::make_unique<tsv::CoefTables>(tsv::coef_tables(k));
  return *tabs[k];
}

// Device copies of the index tables (they depend on k and the arc kernel
// only): built and uploaded once per (device, k, kernel) for the process, so
// an evaluation issues no pageable host->device copy (a pageable copy stalls
// the host and serialises the streams of concurrent evaluations).
struct CoefConst {
  int2* pairs = nullptr;      // pairs (readout), jpairs (z map), items
  int32_t* maps = nullptr;    // smap, item offsets/counts
  uint64_t* ident = nullptr;  // k x k identity (w of the shade basis)
  uint64_t* omask = nullptr;  // per level, (k+1)^2 output masks of the item lists
  std::vector<size_t> poff, joff, moff, icoff, omoff;
};
const CoefConst& coef_const(int dev, int k, bool items) {
  static std::mutex mu;
  static std::vector<std::unique_ptr<CoefConst>> cache;
  std::lock_guard<std::mutex> lk(mu);
  const size_t key = (static_cast<size_t>(dev) * 31 + k) * 2 + (items ? 1 : 0);
  if (cache.size() <= key) cache.resize(key + 1);
  if (cache[key]) return *cache[key];
  const tsv::CoefTables& T = coef_const_tables(k);
  auto c = std::make_unique<CoefConst>();
  std::vector<int2> pairs;
  c->poff.assign(static_cast<size_t>(k) + 1, 0);
  c->joff = c->moff = c->icoff = c->omoff = c->poff;
  std::vector<uint64_t> om;
  for (int l = 2; l <= k; ++l) {
    c->poff[l] = pairs.size();
    pairs.insert(pairs.end(), T.pairs[l].begin(), T.pairs[l].end());
  }
  for (int l = 2; l <= k; ++l) {
    c->joff[l] = pairs.size();
    pairs.insert(pairs.end(), T.jpairs[l].begin(), T.jpairs[l].end());
  }
  std::vector<int32_t> maps;
  for (int l = 2; l <= k; ++l) {
    c->moff[l] = maps.size();
    maps.insert(maps.end(), T.smap[l].begin(), T.smap[l].end());
  }
  if (items) {
    for (int l = 2; l <= k; ++l) {
      tsv::CoefItems ci = tsv::coef_items(k, l);
      c->omoff[l] = om.size();
      for (size_t pt = 0; pt < ci.off.size(); ++pt) {
        uint64_t msk = 0;
        for (int32_t i = 0; i < ci.cnt[pt]; ++i) {
          const int32_t o = ci.items[static_cast<size_t>(ci.off[pt] + i)].y;
          if (o < 64) msk |= 1ull << o;
        }
        om.push_back(msk);
      }
      for (int32_t& o : ci.off) o += static_cast<int32_t>(pairs.size());  // absolute
      pairs.insert(pairs.end(), ci.items.begin(), ci.items.end());
      c->icoff[l] = maps.size();
      maps.insert(maps.end(), ci.off.begin(), ci.off.end());
      maps.insert(maps.end(), ci.cnt.begin(), ci.cnt.end());
    }
  }
  std::vector<uint64_t> I(static_cast<size_t>(k) * k, 0);
  for (int d = 0; d < k; ++d) I[static_cast<size_t>(d) * k + d] = 1;
  int cur = 0;
  TSV_CUDA(cudaGetDevice(&cur));
  TSV_CUDA(cudaSetDevice(dev));
  TSV_CUDA(cudaMalloc(&c->pairs, std::max<size_t>(pairs.size(), 1) * sizeof(int2)));
  TSV_CUDA(cudaMalloc(&c->maps, std::max<size_t>(maps.size(), 1) * 4));
  TSV_CUDA(cudaMalloc(&c->ident, I.size() * 8));
  TSV_CUDA(cudaMalloc(&c->omask, std::max<size_t>(om.size(), 1) * 8));
  if (!om.empty())
    TSV_CUDA(cudaMemcpy(c->omask, om.data(), om.size() * 8, cudaMemcpyHostToDevice));
  TSV_CUDA(cudaMemcpy(c->pairs, pairs.data(), pairs.size() * sizeof(int2),
                      cudaMemcpyHostToDevice));
  TSV_CUDA(cudaMemcpy(c->maps, maps.data(), maps.size() * 4, cudaMemcpyHostToDevice));
  TSV_CUDA(cudaMemcpy(c->ident, I.data(), I.size() * 8, cudaMemcpyHostToDevice));
  TSV_CUDA(cudaSetDevice(cur));
  cache[key] = std::move(c);
  return *cache[key];
}

// Largest in-degree the vertex-lane engine takes: a lane walks its vertex's
// arcs serially, so power-law hubs go to the arc-parallel kernels.
constexpr int32_t kVertexMaxArcs = 4096;

// The vertex-lane partition `rank` of `world` of g (built once, on `st`):
// the vertices [n*rank/world, n*(rank+1)/world), their work list and state
// slots.  applicable = false when the graph has hub vertices.
const tsv_graph::VertPart& vertex_part(const tsv_graph* g, int rank, int world,
                                       cudaStream_t st) {
  std::lock_guard<std::mutex> lk(g->vl_mu);
  for (auto& vp : g->parts)
    if (vp->rank == rank && vp->world == world) return *vp;
  auto vp = std::make_unique<tsv_graph::VertPart>();
  vp->rank = rank;
  vp->world = world;
  const int64_t n = g->dev.n;
  vp->v_lo = static_cast<int32_t>(n * rank / world);
  vp->v_hi = static_cast<int32_t>(n * (rank + 1) / world);
  std::vector<void*>& live = vp->owned;
  auto alloc = [&](size_t bytes) -> void* {
    void* p = nullptr;
    if (!alloc_retry(&p, bytes ? bytes : 8, st))
      throw CudaError("vertex list: out of device memory");
    live.push_back(p);
    return p;
  };
  auto release = [&](void* p) {
    auto it = std::find(live.begin(), live.end(), p);
    if (it != live.end()) live.erase(it);
    cudaFreeAsync(p, st);
  };
  try {
    tsv::build_vertex_list(g->dev, vp->vl, st, alloc, release, vp->v_lo, vp->v_hi);
    int32_t maxc = 0;
    if (vp->vl.nv) {
      TSV_CUDA(cudaMemcpyAsync(&maxc, vp->vl.count, 4, cudaMemcpyDeviceToHost, st));
      TSV_CUDA(cudaStreamSynchronize(st));
    }
    // the largest in-degree of the whole graph decides applicability (every
    // rank of a world must agree): the full list is partition (0, 1)
    vp->applicable = maxc <= kVertexMaxArcs;
    int32_t r0 = 0, r1 = 0;
    TSV_CUDA(cudaMemcpyAsync(&r0, g->dev.vtx_run_off + vp->v_lo, 4, cudaMemcpyDeviceToHost, st));
    TSV_CUDA(cudaMemcpyAsync(&r1, g->dev.vtx_run_off + vp->v_hi, 4, cudaMemcpyDeviceToHost, st));
    TSV_CUDA(cudaStreamSynchronize(st));
    vp->slot_lo = tsv::count_slots_before(g->dev, r0, st, alloc, release);
    vp->slot_hi = tsv::count_slots_before(g->dev, r1, st, alloc, release);
  } catch (...) {
    for (void* p : live) cudaFreeAsync(p, st);
    live.clear();
    throw;
  }
  g->parts.push_back(std::move(vp));
  return *g->parts.back();
}

// Largest in-degree the vertex-lane engine takes: a lane walks its vertex's
// arcs serially, so power-law hubs go to the arc-parallel kernels.
bool vertex_applicable(const tsv_graph* g, cudaStream_t st) {
  if (!vertex_part(g, 0, 1, st).applicable) return false;
  return true;
}

// Time-window plan of a coefficient evaluation whose state rows do not fit
// (coef_window.cu): the shaded edges with ts <= max_ts in canonical order
// (ts-major, so a window is a contiguous range), split between distinct
// timestamps into windows of at most `rows_cap` arcs.
struct WindowPlan {
  int64_t m = 0;                 // kept edges
  std::unique_ptr<DevBuf> ku, kv, kts, koid;  // kept canonical edges, original edge ids
  std::vector<int64_t> bounds;   // window w = edges [bounds[w], bounds[w+1])
};

// Splits [0, m) into windows of at most cap arcs (arcs_per_edge per edge),
// boundaries moved down to the start of their timestamp group.  Returns
// false when one timestamp alone exceeds the cap.
bool plan_windows(const int32_t* d_ts, int64_t m, int arcs_per_edge, int64_t cap,
                  std::vector<int64_t>& bounds, cudaStream_t st) {
  const int64_t cap_e = std::max<int64_t>(cap / arcs_per_edge, 1);
  int64_t nw = std::max<int64_t>((m + cap_e - 1) / cap_e, 1);
  for (int attempt = 0; attempt < 16; ++attempt, nw = nw + nw / 4 + 1) {
    bounds.assign(1, 0);
    if (nw > 1) {
      std::vector<int64_t> pos(static_cast<size_t>(nw - 1)), got(pos.size());
      for (int64_t w = 1; w < nw; ++w) pos[w - 1] = w * m / nw;
      DevBuf dp(pos.size() * 8, st), dg(pos.size() * 8, st);
      TSV_CUDA(cudaMemcpyAsync(dp.p, pos.data(), pos.size() * 8, cudaMemcpyHostToDevice, st));
      tsv::launch_ts_group_start(d_ts, dp.as<int64_t>(), static_cast<int>(pos.size()),
                                 dg.as<int64_t>(), st);
      TSV_CUDA(cudaMemcpyAsync(got.data(), dg.p, got.size() * 8, cudaMemcpyDeviceToHost, st));
      TSV_CUDA(cudaStreamSynchronize(st));
      for (int64_t x : got)
        if (x > bounds.back()) bounds.push_back(x);
    }
    bounds.push_back(m);
    bool ok = true;
    for (size_t w = 0; w + 1 < bounds.size(); ++w)
      ok = ok && (bounds[w + 1] - bounds[w]) <= cap_e;
    if (ok) return true;
  }
  return false;
}

// The coefficient (top-degree) engine, coef_kernels.cu: the XOR over ALL
// 2^k sieve points in one pass per level, bit-identical to the point engine.
// Used for full-range evaluations; when its working set (two state buffers
// of S rows) does not fit, the arcs run in time windows (coef_window.cu).
// TSV_ENGINE=points disables it.  Returns false (nothing launched) when not
// applicable.
bool eval_coef(const tsv_graph* g, const tsv_shades* sh, int k, int32_t max_ts,
               const tsv_config* cfg, int32_t anchor_source, uint64_t* d_acc, cudaStream_t st,
               uint64_t* peak_out, const VcSpec* vc) {
  const char* eng = std::getenv("TSV_ENGINE");
  if (eng && std::strcmp(eng, "points") == 0) return false;
  if (k < 2 || k > 12) return false;  // C(k, l) <= tsv::kZAcc
  // TSV_TRACE_COEF=1: host microseconds per phase of this call on stderr
  // (no synchronization added: enqueue cost and blocking calls)
  static const bool trace = [] {
    const char* e = std::getenv("TSV_TRACE_COEF");
    return e && e[0] == '1';
  }();
  const auto tc0 = std::chrono::steady_clock::now();
  auto tmark = [&](const char* what) {
    if (!trace) return;
    std::fprintf(stderr, "[coef] %-24s %9.1f us\n", what,
                 std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - tc0)
                     .count());
  };
  const tsv_graph* g0 = g;  // the caller's graph (time windows restrict it)
  // arcs touching a shadeless vertex never carry a nonzero product (its z,
  // hence every S row, is zero): evaluate the shaded subgraph, which keeps
  // the vertex and edge ids (y draws) and gives the same accumulators
  std::shared_ptr<tsv_graph> sub_hold;
  if (!vc && sh) {
    sub_hold = shaded_subgraph(g, sh);
    if (sub_hold) g = sub_hold.get();
  }
  const tsv::CoefTables& T = coef_const_tables(k);
  const uint64_t n = static_cast<uint64_t>(g->dev.n);
  // item-stream kernel (coef_items.cu) unless the vertex-ordered sieve's
  // positional z (no shade structure) or TSV_ITEMS=0
  // (measured: C3/C4, all single-shade, 1.3x faster; C5, no single-shade
  // vertex, 1.2x slower than k_coef_arcs)
  const char* it_env = std::getenv("TSV_ITEMS");
  bool use_items = !vc && !(it_env && std::strcmp(it_env, "0") == 0) &&
                   ((it_env && std::strcmp(it_env, "1") == 0) || sh->single * 4 >= n);
  // U-row entries of level l (2..k-1) per vertex class, and the row stride:
  // rows of multi-shade heads hold their U row, then (z map in place) their
  // S row; without multi-shade rows a row is just the U frame (the single-
  // shade compact frame C(k-1, l-1) in the item-stream layout)
  const bool multi_rows = vc || sh->multi > 0;
  auto fr_multi = [&](int l) { return static_cast<int>(T.count[l - 1]); };
  auto fr_single = [&](int l) {
    return use_items ? static_cast<int>(T.count[l - 1] * (k - l + 1) / k) : fr_multi(l);
  };
  auto rs = [&](int l) {
    return multi_rows ? static_cast<int>(std::max(T.count[l - 1], T.count[l]))
                      : (sh->single ? fr_single(l) : fr_multi(l));
  };
  int64_t M = 1;  // largest row stride; the chunk aggregates take C(k, l-1)
  int64_t MA = 1;
  for (int l = 2; l < k; ++l) M = std::max<int64_t>(M, rs(l));
  for (int l = 2; l <= k; ++l) MA = std::max<int64_t>(MA, T.count[l - 1]);
  const uint64_t S = static_cast<uint64_t>(std::max<int64_t>(g->dev.S, 1));
  const uint64_t C = static_cast<uint64_t>(std::max<int64_t>(g->dev.C, 1));
  const uint64_t words = 2 * S * M + C * MA + 2 * n * k + 2 * n + S + (n + S) / 8 + 2;
  tmark("tables, subgraph");
  // (the vertex path takes its two state buffers from the per-device cache)
  int cur_dev = 0;
  TSV_CUDA(cudaGetDevice(&cur_dev));
  const uint64_t cached = static_cast<uint64_t>(cached_state_free(cur_dev)) / 8;
  const bool vertex_like = !vc && sh->single == 0 && tsv::vertex_engine_supports(k);
  const uint64_t need = vertex_like ? words - std::min<uint64_t>(cached, 2 * S * M) : words;
  const bool fits = words <= cfg->memory_cap_words && fits_device(need);
  tmark("fits_device");
  // time windows (coef_window.cu) when the state rows do not fit at once:
  // instant edge model, shade structure (not the VC sieve's positional z)
  const char* win_env = std::getenv("TSV_WINDOW_ROWS");  // (tests: force windows of <= N arcs)
  const int64_t force_rows = win_env ? std::atoll(win_env) : 0;
  const bool windowed = (!fits || force_rows > 0) && !vc && g0->model == 0;
  if (!fits && !windowed) return false;
  if (windowed && !use_items) {  // (the carried prefix is read by the item-stream kernels)
    use_items = true;
    M = 1;
    for (int l = 2; l < k; ++l) M = std::max<int64_t>(M, rs(l));
  }
  WindowPlan wp;
  std::vector<int64_t> cs_words(static_cast<size_t>(k) + 1, 0);  // carry stride per level
  int64_t rows_cap = static_cast<int64_t>(S);
  uint64_t fixed_words = 0;
  if (windowed) {
    for (int l = 2; l < k; ++l) cs_words[l] = multi_rows ? fr_multi(l) : fr_single(l);
    for (int l = 2; l < k; ++l) fixed_words += n * static_cast<uint64_t>(cs_words[l]) + n / 8 + 1;
    const uint64_t m0 = static_cast<uint64_t>(g0->m);
    fixed_words += 2 * n * k + 2 * n + 2 * m0 + (g0->d_eu ? 0 : 2 * m0);
    // per row (window arc): two state rows, flags, z-map list, the window
    // graph and its build temporaries (~80 bytes per edge)
    const uint64_t per_row = 2 * static_cast<uint64_t>(M) + 12;
    const uint64_t budget = std::min<uint64_t>(cfg->memory_cap_words, device_budget_words());
    if (budget <= fixed_words + (n + 1) * per_row) return false;
    rows_cap = static_cast<int64_t>((budget - fixed_words) / per_row) - static_cast<int64_t>(n);
    if (force_rows > 0) rows_cap = std::min<int64_t>(rows_cap, force_rows);
    if (rows_cap < (force_rows > 0 ? 16 : 1024)) return false;
    // the shaded edges of the caller's graph with ts <= max_ts, original ids
    const int64_t m = g0->m;
    std::vector<void*> tmp;
    auto alloc = [&](size_t bytes) -> void* {
      void* p = nullptr;
      if (!alloc_retry(&p, bytes ? bytes : 8, st))
        throw CudaError("time windows: out of device memory");
      tmp.push_back(p);
      return p;
    };
    auto release = [&](void* p) {
      auto it = std::find(tmp.begin(), tmp.end(), p);
      if (it != tmp.end()) tmp.erase(it);
      cudaFreeAsync(p, st);
    };
    try {
      const int32_t *eu = g0->d_eu, *ev = g0->d_ev, *ets = g0->d_ets;
      if (!eu) {
        auto* a = static_cast<int32_t*>(alloc(std::max<int64_t>(m, 1) * 4));
        auto* b = static_cast<int32_t*>(alloc(std::max<int64_t>(m, 1) * 4));
        auto* c = static_cast<int32_t*>(alloc(std::max<int64_t>(m, 1) * 4));
        if (g0->edges_in_layout) {
          tsv::edges_from_layout(g0->dev, g0->host.directed, a, b, c, st);
        } else if (m) {
          TSV_CUDA(cudaMemcpyAsync(a, g0->host.eu.data(), m * 4, cudaMemcpyHostToDevice, st));
          TSV_CUDA(cudaMemcpyAsync(b, g0->host.ev.data(), m * 4, cudaMemcpyHostToDevice, st));
          TSV_CUDA(cudaMemcpyAsync(c, g0->host.ets.data(), m * 4, cudaMemcpyHostToDevice, st));
        }
        eu = a;
        ev = b;
        ets = c;
      }
      auto* keep = static_cast<uint8_t*>(alloc(std::max<uint64_t>(n, 1)));
      tsv::launch_shaded_mask(static_cast<int32_t>(n), sh->off, keep, st);
      const size_t eb = static_cast<size_t>(std::max<int64_t>(m, 1)) * 4;
      wp.ku = std::make_unique<DevBuf>(eb, st);
      wp.kv = std::make_unique<DevBuf>(eb, st);
      wp.kts = std::make_unique<DevBuf>(eb, st);
      wp.koid = std::make_unique<DevBuf>(eb, st);
      wp.m = tsv::device_restrict(eu, ev, ets, m, keep, max_ts, wp.ku->as<int32_t>(),
                                  wp.kv->as<int32_t>(), wp.kts->as<int32_t>(), st, alloc, release,
                                  wp.koid->as<int32_t>());
      for (void* p : tmp) cudaFreeAsync(p, st);
      tmp.clear();
    } catch (...) {
      for (void* p : tmp) cudaFreeAsync(p, st);
      throw;
    }
    if (!plan_windows(wp.kts->as<int32_t>(), wp.m, g0->host.directed ? 1 : 2, rows_cap,
                      wp.bounds, st))
      return false;
    if (peak_out) *peak_out = fixed_words + (static_cast<uint64_t>(rows_cap) + n) * per_row;
  } else if (peak_out) {
    *peak_out = words;
  }
  const int32_t nn = g->dev.n;
  int dev = 0, sms = 148;
  TSV_CUDA(cudaGetDevice(&dev));
  TSV_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));

  // Shade basis (coef_kernels.cu, top): z_u(x) = XOR_d v_{u,d} w_d(x), so the
  // engine runs on the n x k table of v_{u,d} (0 for d not in S(u); k_zj
  // with the identity for w) and the readout multiplies by det(W) = per(W)
  // (char 2).  Vertex-ordered sieves keep their positional z_{u,j}.
  uint64_t scale = 1;
  DevBuf d_zj(static_cast<size_t>(n) * k * 8, st);
  if (vc) {
    tsv::launch_zj_positional(nn, k, cfg->seed, d_zj.as<uint64_t>(), st);
  } else {
    std::vector<uint64_t> W(static_cast<size_t>(k) * k);
    const uint64_t pre = tsv::draw_prefix(cfg->seed, tsv::kRoleShadeW);
    for (int d = 0; d < k; ++d) {
      for (int j = 0; j < k; ++j)
        W[static_cast<size_t>(d) * k + j] = tsv::draw_nonzero_from(pre, d + 1, j + 1, 0);
    }
    scale = tsv::gf_det_host(W.data(), k);
    tsv::launch_zj_ident(nn, k, cfg->seed, sh->off, sh->shades, d_zj.as<uint64_t>(), st);
  }
  tmark("shade table");
  // state rows: S slots, or per window its slots plus n carry slots
  const uint64_t rows = windowed ? static_cast<uint64_t>(rows_cap) + n : S;
  if (!vc && !windowed && sh->single == 0 && tsv::vertex_engine_supports(k))
    for (int l = 2; l < k; ++l) M = std::max<int64_t>(M, tsv::vertex_row_words(k, l));
  std::unique_ptr<StateBuf> VX, VY;  // vertex path: cached state buffers
  // every shaded vertex multi-shade and small k (k-TempPath, C5): the
  // vertex-lane engine (coef_vertex.cu) -- fused z map and readout, so none
  // of the buffers below (ulast, flags, z-map lists, chunk aggregates)
  const char* vx_env = std::getenv("TSV_VERTEX");
  const bool try_vertex = !vc && !windowed && sh->single == 0 &&
                          tsv::vertex_engine_supports(k) && !(vx_env && vx_env[0] == '0');
  tmark("state buffers");
  if (try_vertex && vertex_applicable(g, st)) {
    const tsv::VertList* vl = &vertex_part(g, 0, 1, st).vl;
    tmark("vertex list");
    VX = std::make_unique<StateBuf>(rows * M * 8, st);
    VY = std::make_unique<StateBuf>(rows * M * 8, st);
    uint64_t *A = VX->as<uint64_t>(), *B = VY->as<uint64_t>();
    for (int l = 2; l <= k; ++l) {
      tsv::CoefParams cp;
      cp.g = g->dev;
      cp.zj = d_zj.as<uint64_t>();
      cp.k = k;
      cp.ell = l;
      cp.last = l == k;
      cp.seed = cfg->seed;
      cp.anchor_source = anchor_source;
      cp.s_prev = A;
      cp.ubuf = B;
      cp.max_ts = max_ts;
      // (with transition times an arc can land past t: always test then)
      cp.below_t = max_ts < g->host.t || g->model != 0;
      tsv::launch_coef_vertex(cp, *vl, scale, d_acc, st);
      TSV_CUDA(cudaGetLastError());
      std::swap(A, B);
    }
    tmark("levels enqueued");
    return true;
  }
  DevBuf X(rows * M * 8, st), Y(rows * M * 8, st);
  DevBuf ulast(std::max<uint64_t>(n, 1) * k * 8, st), slot_head(std::getenv("TSV_ZTRANS") ? S * 4 : 8, st);
  // zero skipping and the single-shade form (CoefParams::vsh); positional z
  // keeps the plain z map
  DevBuf vsh(std::max<uint64_t>(n, 1), st), vsv(std::max<uint64_t>(n, 1) * 8, st);
  DevBuf fl0(rows, st), fl1(rows, st);
  if (!vc) tsv::launch_vshade(nn, k, d_zj.as<uint64_t>(), vsh.as<int8_t>(), vsv.as<uint64_t>(), st);
  TSV_CUDA(cudaMemsetAsync(ulast.p, 0, std::max<uint64_t>(n, 1) * k * 8, st));
  // the index tables depend on (k, use_items) only: uploaded once per device
  tmark("buffers");
  const CoefConst& cc = coef_const(dev, k, use_items);
  const std::vector<size_t>&poff = cc.poff, &joff = cc.joff, &moff = cc.moff, &icoff = cc.icoff;
  // multi-shade rows: the direct z map over a (slot, head) list, or
  // (TSV_ZTRANS=tab) the warp-per-window table map over slot_head
  const char* zt_env = std::getenv("TSV_ZTRANS");
  const bool zt_tab = zt_env && std::strcmp(zt_env, "tab") == 0 && !windowed;
  DevBuf mlist(rows * 8, st), mcount(4, st);
  // expected listed rows: slots x the multi-shade share of the shaded vertices
  const int64_t rows_hint =
      vc ? static_cast<int64_t>(rows)
         : static_cast<int64_t>(static_cast<double>(rows) * static_cast<double>(sh->multi) /
                                static_cast<double>(std::max<int64_t>(sh->multi + sh->single, 1)));
  const int2* dp = cc.pairs;
  // chunk counters of the persistent item kernel, one per level and window
  const char* ps_env = std::getenv("TSV_PERSIST");
  const bool persist = !(ps_env && std::strcmp(ps_env, "0") == 0);
  const size_t nwin = windowed ? wp.bounds.size() - 1 : 1;
  DevBuf ctrs(static_cast<size_t>(k + 1) * nwin * 4, st);
  if (persist) TSV_CUDA(cudaMemsetAsync(ctrs.p, 0, static_cast<size_t>(k + 1) * nwin * 4, st));
  // carries of the windowed form: per level l < k, the U rows of every
  // vertex as of the window start (stride cs_words[l]) and a nonzero flag
  std::vector<std::unique_ptr<DevBuf>> carry(static_cast<size_t>(k) + 1),
      cnz(static_cast<size_t>(k) + 1);
  DevBuf cmlist(windowed ? std::max<uint64_t>(n, 1) * 8 : 8, st), cmcount(4, st);
  if (windowed) {
    for (int l = 2; l < k; ++l) {
      carry[l] = std::make_unique<DevBuf>(std::max<uint64_t>(n, 1) * cs_words[l] * 8, st);
      cnz[l] = std::make_unique<DevBuf>(std::max<uint64_t>(n, 1), st);
      TSV_CUDA(cudaMemsetAsync(cnz[l]->p, 0, std::max<uint64_t>(n, 1), st));
    }
  }
  for (size_t w = 0; w < nwin; ++w) {
    // the graph of this pass: the whole (shaded) graph, or the window's edges
    // with their original ids, every vertex's last run given a slot, and the
    // arcs without a source in the window reading the tail's carry slot
    std::unique_ptr<tsv_graph> gw;
    tsv::DevGraph dg = g->dev;
    int64_t Sw = 0;
    if (windowed) {
      const int64_t e0 = wp.bounds[w], e1 = wp.bounds[w + 1];
      TSV_CUDA(cudaStreamSynchronize(st));
      gw.reset(device_graph_build(nn, e1 - e0, wp.ku->as<int32_t>() + e0,
                                  wp.kv->as<int32_t>() + e0, wp.kts->as<int32_t>() + e0,
                                  g0->host.directed, g0->host.t, g0->device, /*canonical=*/true,
                                  /*on_device=*/true, nullptr, nullptr, 0,
                                  /*force_last_runs=*/true));
      tsv::launch_win_edge_ids(gw->dev.A, const_cast<uint32_t*>(gw->dev.arc_meta),
                               wp.koid->as<int32_t>(), e0, st);
      Sw = gw->dev.S;
      tsv::launch_win_src(gw->dev.A, const_cast<int32_t*>(gw->dev.arc_src), gw->dev.arc_tail, Sw,
                          st);
      dg = gw->dev;
      dg.S = Sw + static_cast<int64_t>(n);
      tsv::launch_win_multi_list(nn, Sw, vsh.as<int8_t>(), cmlist.as<int2>(),
                                 cmcount.as<int32_t>(), st);
    }
    const uint64_t Cw = static_cast<uint64_t>(std::max<int64_t>(dg.C, 1));
    DevBuf agg(Cw * MA * 8, st);
    if (zt_tab)
      tsv::launch_slot_head(dg.R, dg.run_slot, dg.run_head, slot_head.as<int32_t>(), st);
    else if (k > 2)
      tsv::launch_multi_slots(dg.R, dg.run_slot, dg.run_head, vc ? nullptr : vsh.as<int8_t>(),
                              mlist.as<int2>(), mcount.as<int32_t>(), st);
    uint64_t *A = X.as<uint64_t>(), *B = Y.as<uint64_t>();
    uint8_t *fa = fl0.as<uint8_t>(), *fb = fl1.as<uint8_t>();
    const uint64_t S_pass = static_cast<uint64_t>(std::max<int64_t>(dg.S, 1));
    for (int l = 2; l <= k; ++l) {
      tsv::CoefParams cp;
      cp.g = dg;
      cp.zj = d_zj.as<uint64_t>();
      cp.k = k;
      cp.ell = l;
      cp.last = l == k;
      cp.seed = cfg->seed;
      cp.anchor_source = anchor_source;
      cp.E = static_cast<int>(T.count[l - 1]);
      cp.s_prev = A;
      cp.rs_in = l > 2 ? rs(l - 1) : 0;
      cp.ubuf = B;
      cp.rs_out = l < k ? rs(l) : 0;
      cp.agg = agg.as<uint64_t>();
      cp.ulast = ulast.as<uint64_t>();
      cp.max_ts = max_ts;
      cp.vsh = vc ? nullptr : vsh.as<int8_t>();
      cp.vsv = vc ? nullptr : vsv.as<uint64_t>();
      cp.sflag = fa;
      cp.sflag_out = fb;
      cp.smap = l > 2 ? cc.maps + moff[l - 1] : nullptr;
      cp.chunk_ctr = persist ? ctrs.as<int32_t>() + w * (k + 1) + l : nullptr;
      cp.sms = sms;
      if (use_items) {
        const int K1 = k + 1;
        cp.items = dp;  // offsets are absolute in d_pairs
        cp.item_off = cc.maps + icoff[l];
        cp.item_cnt = cp.item_off + K1 * K1;
        cp.item_omask = cc.omask + cc.omoff[l];
        cp.frame_multi = static_cast<int>(T.count[l - 1]);
        cp.frame_single = static_cast<int>(T.count[l - 1] * (k - l + 1) / k);  // C(k-1, l-1)
        cp.frame_max = sh->multi ? cp.frame_multi : cp.frame_single;
        cp.warp_words = tsv::GfTable::kWords + (cp.frame_max + 31) / 32 * 32;
      }
      if (windowed && !cp.last) {
        cp.carry_in = carry[l]->as<uint64_t>();
        cp.carry_nz = cnz[l]->as<uint8_t>();
        cp.carry_cs = static_cast<int>(cs_words[l]);
      }
      if (vc) {
        cp.vc_color = vc->d_colors;
        cp.vc_head = vc->order[l - 1];
        cp.vc_tail = vc->order[l - 2];
        cp.vc_wild = vc->wild;
      }
      if (!cp.last) TSV_CUDA(cudaMemsetAsync(fb, 0, S_pass, st));
      if (use_items) {
        tsv::launch_coef_items(cp, st);
      } else {
        for (int e0 = 0; e0 < cp.E; e0 += tsv::kCoefSlice) {
          cp.e0 = e0;
          cp.ne = std::min(tsv::kCoefSlice, cp.E - e0);
          tsv::launch_coef_arcs(cp, st);
        }
      }
      if (!cp.last) {
        tsv::launch_coef_fixup(cp, st);
        if (windowed) {
          tsv::WinCarryArgs wa;
          wa.run_slot = dg.run_slot;
          wa.vro = dg.vtx_run_off;
          wa.n = nn;
          wa.Sw = Sw;
          wa.vsh = vsh.as<int8_t>();
          wa.frs = fr_single(l);
          wa.frm = fr_multi(l);
          wa.rows = B;
          wa.rs = rs(l);
          wa.sflag = fb;
          wa.carry = carry[l]->as<uint64_t>();
          wa.cs = static_cast<int>(cs_words[l]);
          wa.cnz = cnz[l]->as<uint8_t>();
          tsv::launch_win_carry(wa, st);
        }
        if (zt_tab) {
          tsv::launch_coef_ztrans(dg.S, static_cast<int>(T.count[l]), l, slot_head.as<int32_t>(),
                                  d_zj.as<uint64_t>(), k, cp.E, B, rs(l), dp + joff[l], cp.vsh, fb,
                                  sms, st);
        } else {
          tsv::launch_coef_ztrans_direct(dg.S, static_cast<int>(T.count[l]), l, mlist.as<int2>(),
                                         mcount.as<int32_t>(), d_zj.as<uint64_t>(), k, B, rs(l),
                                         dp + poff[l], vc ? nullptr : fb, sms, rows_hint, st);
          if (windowed && sh->multi)
            tsv::launch_coef_ztrans_direct(static_cast<int64_t>(n), static_cast<int>(T.count[l]),
                                           l, cmlist.as<int2>(), cmcount.as<int32_t>(),
                                           d_zj.as<uint64_t>(), k, B, rs(l), dp + poff[l], fb,
                                           sms, sh->multi, st);
        }
        std::swap(A, B);
        std::swap(fa, fb);
      }
      TSV_CUDA(cudaGetLastError());
    }
    if (gw) TSV_CUDA(cudaStreamSynchronize(st));  // the window graph is freed next
  }
  tsv::launch_coef_readout(nn, d_zj.as<uint64_t>(), k, ulast.as<uint64_t>(), dp + poff[k], scale,
                           use_items ? vsh.as<int8_t>() : nullptr,
                           use_items ? vsv.as<uint64_t>() : nullptr, d_acc, st);
  TSV_CUDA(cudaGetLastError());
  return true;
}

// GF(2^8 / 2^16 / 2^32) temporal sieve (small_field.cu): the point form, one
// thread per (head vertex, point), batches of W points.
void eval_small_field(const tsv_graph* g, const tsv_shades* sh, int k, int32_t max_ts,
                      const tsv_config* cfg, int32_t anchor_source, uint64_t p_begin,
                      uint64_t p_end, uint64_t* d_acc, cudaStream_t st, uint64_t* peak_out) {
  std::vector<void*> live;
  auto alloc = [&](size_t bytes) -> void* {
    void* p = nullptr;
    if (!alloc_retry(&p, bytes ? bytes : 8, st))
      throw CudaError("small-field sieve: out of device memory");
    live.push_back(p);
    return p;
  };
  auto release = [&](void* p) {
    auto it = std::find(live.begin(), live.end(), p);
    if (it != live.end()) live.erase(it);
    cudaFreeAsync(p, st);
  };
  const uint64_t S = static_cast<uint64_t>(std::max<int64_t>(g->dev.S, 1));
  const uint64_t bytes = static_cast<uint64_t>(cfg->field_bits / 8);
  int W = static_cast<int>(std::min<uint64_t>(p_end - p_begin, 64));
  auto words = [&](int w) { return (2 * S * w * bytes + 7) / 8 + 2 * static_cast<uint64_t>(g->dev.n); };
  while (W > 1 && (words(W) > cfg->memory_cap_words || !fits_device(words(W)))) W >>= 1;
  if (words(W) > cfg->memory_cap_words)
    throw CapError("sieve memory cap exceeded: needs " + std::to_string(words(W)) +
                   " field words, cap " + std::to_string(cfg->memory_cap_words));
  if (peak_out) *peak_out = words(W);
  try {
    tsv::VertList vl;
    if (k >= 2) tsv::build_vertex_list(g->dev, vl, st, alloc, release);
    tsv::SmallFieldArgs a;
    a.bits = cfg->field_bits;
    a.g = g->dev;
    a.head = vl.head;
    a.start = vl.start;
    a.count = vl.count;
    a.nv = vl.nv;
    a.off = sh->off;
    a.shades = sh->shades;
    a.k = k;
    a.seed = cfg->seed;
    a.anchor = anchor_source;
    a.max_ts = max_ts;
    a.pb = p_begin;
    a.pe = p_end;
    a.W = W;
    a.acc = d_acc;
    a.alloc = alloc;
    a.release = release;
    tsv::launch_small_field(a, st);
    TSV_CUDA(cudaGetLastError());
  } catch (...) {
    for (void* p : live) cudaFreeAsync(p, st);
    throw;
  }
  for (void* p : live) cudaFreeAsync(p, st);
}

void eval_device(const tsv_graph* g, const tsv_shades* sh, int k, int32_t max_ts,
                 const tsv_config* cfg, int32_t anchor_source, uint64_t p_begin,
                 uint64_t p_end, uint64_t* d_acc, cudaStream_t st,
                 uint64_t* peak_out, const VcSpec* vc = nullptr) {
  check_config(cfg, !vc);
  if (k < 1 || k > 30) throw std::invalid_argument("k out of range [1,30]");
  if (max_ts < 1 || max_ts > g->host.t) throw std::invalid_argument("max_ts outside [1..t]");
  if (!vc && (!sh || sh->n != g->dev.n || sh->k != k))
    throw std::invalid_argument("shade assignment built for a different graph");
  if (!vc && sh->device != g->device)
    throw std::invalid_argument("shade table uploaded to device " + std::to_string(sh->device) +
                                ", graph lives on device " + std::to_string(g->device));
  if (vc && static_cast<int>(vc->order.size()) != k)
    throw std::invalid_argument("order must have k colors");
  if (cfg->edge_model != g->model)
    throw std::invalid_argument("graph was built for edge model " + std::to_string(g->model) +
                                ", config asks for " + std::to_string(cfg->edge_model) +
                                " (tsv_graph_build_model)");
  const uint64_t P = 1ull << k;
  p_end = std::min(p_end, P);
  if (p_begin >= p_end) return;
  if (cfg->field_bits != 64) {
    eval_small_field(g, sh, k, max_ts, cfg, anchor_source, p_begin, p_end, d_acc, st, peak_out);
    return;
  }
  if (p_begin == 0 && p_end == P &&
      eval_coef(g, sh, k, max_ts, cfg, anchor_source, d_acc, st, peak_out, vc))
    return;
  uint64_t peak = 0;
  bool zb_ok = false;
  int nlanes = 1;
  const int W = choose_width(g, k, p_end - p_begin, cfg, &peak, &zb_ok, &nlanes);
  if (peak_out) *peak_out = peak;
  const int32_t n = g->dev.n;

  // w_{d,j} table on the host (k^2 draws), z_{u,j} on the device.
  DevBuf d_w(static_cast<size_t>(k) * k * 8, st), d_zj(static_cast<size_t>(n) * k * 8, st);
  tsv::launch_wtab(k, cfg->seed, d_w.as<uint64_t>(), st);
  if (vc)
    tsv::launch_zj_positional(n, k, cfg->seed, d_zj.as<uint64_t>(), st);
  else
    tsv::launch_zj(n, k, cfg->seed, sh->off, sh->shades, d_w.as<uint64_t>(),
                   d_zj.as<uint64_t>(), st);
  TSV_CUDA(cudaGetLastError());

  if (k == 1) {
    tsv::Batch b;
    b.pb = p_begin;
    b.pe = p_end;
    if (vc)
      tsv::launch_k1(n, d_zj.as<uint64_t>(), b, -1, d_acc, st, vc->d_colors, vc->order[0],
                     vc->wild);
    else
      tsv::launch_k1(n, d_zj.as<uint64_t>(), b, anchor_source, d_acc, st);
    TSV_CUDA(cudaGetLastError());
    return;
  }
  const size_t state_words = static_cast<size_t>(std::max<int64_t>(g->dev.S, 1)) * W;
  // Level 2 reads z_tail^A for every arc and the run-end products z_head^A:
  // when the per-batch table z[u][w] is small next to the state (n <= R/8)
  // and fits, it is materialized once per batch and gathered like a state row.
  const uint64_t zb_bytes = static_cast<uint64_t>(n) * W * 8;
  const bool use_zb = zb_ok;
  // One or two lanes (stream + private working set); batch i runs on lane
  // i % lanes, the second lane's stream forked from / joined to `st`.
  struct Lane {
    cudaStream_t st = nullptr;
    std::unique_ptr<DevBuf> s0, s1, agg, zb;
  };
  std::vector<Lane> lanes(static_cast<size_t>(nlanes));
  cudaEvent_t fork = nullptr, join = nullptr;
  for (int l = 0; l < nlanes; ++l) {
    Lane& L = lanes[l];
    if (l == 0) {
      L.st = st;
    } else {
      TSV_CUDA(cudaStreamCreateWithFlags(&L.st, cudaStreamNonBlocking));
    }
    L.s0 = std::make_unique<DevBuf>(state_words * 8, st);
    L.s1 = std::make_unique<DevBuf>(state_words * 8, st);
    L.agg = std::make_unique<DevBuf>(static_cast<size_t>(g->dev.C) * W * 8, st);
    L.zb = std::make_unique<DevBuf>(use_zb ? zb_bytes : 8, st);
  }
  if (nlanes > 1) {  // lane 1 starts after z and the buffers exist on `st`
    TSV_CUDA(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
    TSV_CUDA(cudaEventCreateWithFlags(&join, cudaEventDisableTiming));
    TSV_CUDA(cudaEventRecord(fork, st));
    TSV_CUDA(cudaStreamWaitEvent(lanes[1].st, fork, 0));
  }
  tsv::LevelParams base_lp;
  base_lp.g = g->dev;
  base_lp.zj = d_zj.as<uint64_t>();
  base_lp.k = k;
  base_lp.seed = cfg->seed;
  base_lp.anchor_source = anchor_source;
  if (const char* e = std::getenv("TSV_YMUL"))
    base_lp.ymul = std::strcmp(e, "holes") == 0 ? 1 : 0;
  uint64_t batch_no = 0;
  for (uint64_t pb = p_begin; pb < p_end; pb += W, ++batch_no) {
    Lane& L = lanes[batch_no % lanes.size()];
    const cudaStream_t bst = L.st;
    tsv::LevelParams lp = base_lp;
    lp.agg = L.agg->as<uint64_t>();
    DevBuf& zb = *L.zb;
    DevBuf& s0 = *L.s0;
    DevBuf& s1 = *L.s1;
    lp.b = batch_shape(W);
    lp.b.pb = pb;
    lp.b.pe = std::min(p_end, pb + static_cast<uint64_t>(W));
    if (use_zb) {
      tsv::launch_zbatch(n, d_zj.as<uint64_t>(), k, lp.b, zb.as<uint64_t>(), bst);
      lp.zb = zb.as<uint64_t>();
    }
    uint64_t* cur = s0.as<uint64_t>();
    uint64_t* prev = s1.as<uint64_t>();
    // level k is produced fused with the readout
    for (int ell = 2; ell <= k; ++ell) {
      lp.ell = ell;
      lp.s_prev = prev;
      lp.s_cur = cur;
      lp.last = ell == k;
      lp.max_ts = max_ts;
      lp.acc = d_acc;
      if (vc) {
        lp.vc_color = vc->d_colors;
        lp.vc_head = vc->order[ell - 1];
        lp.vc_tail = vc->order[ell - 2];
        lp.vc_wild = vc->wild;
      }
      tsv::launch_level(lp, bst);
      if (lp.last) break;
      tsv::launch_fixup(lp, bst);
      std::swap(cur, prev);
    }
    TSV_CUDA(cudaGetLastError());
  }
  if (nlanes > 1) {  // join lane 1 back into `st` before its buffers are freed
    TSV_CUDA(cudaEventRecord(join, lanes[1].st));
    TSV_CUDA(cudaStreamWaitEvent(st, join, 0));
    cudaEventDestroy(fork);
    cudaEventDestroy(join);
    cudaStreamDestroy(lanes[1].st);  // released once its work completes
  }
}

void finalize_host(int32_t n, uint64_t* acc, int32_t sink, int k, tsv_outcome* out) {
  int64_t flagged = 0;
  uint64_t h = 1469598103934665603ull;
  auto eat = [&](uint64_t x) {
    for (int i = 0; i < 8; ++i) {
      h ^= (x >> (8 * i)) & 0xff;
      h *= 1099511628211ull;
    }
  };
  for (int32_t u = 0; u < n; ++u) {
    if (sink >= 0 && u != sink) acc[u] = 0;
    if (!acc[u]) continue;
    ++flagged;
    eat(static_cast<uint64_t>(u));
    eat(acc[u]);
  }
  out->flagged = flagged;
  out->global_nonzero = flagged > 0;
  out->checksum = h;
  out->fn_bound = (2.0 * k - 1.0) / std::pow(2.0, 64);
}

// On-device build (build_kernels.cu): host edges -> HBM once, canonicalize,
// sort and lay out on the GPU.  Every buffer still alive at the end belongs
// to the graph.
tsv_graph* device_graph_build(int32_t n, int64_t m, const int32_t* u, const int32_t* v,
                              const int32_t* ts, bool directed, int32_t t, int device,
                              bool canonical, bool on_device, const int32_t* eps,
                              const int32_t* delays, int model, bool force_last_runs) {
  const cudaMemcpyKind kind = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  DeviceGuard dg(device);
  int sm_count = 0;  // (cudaGetDeviceProperties costs milliseconds per call)
  TSV_CUDA(cudaDeviceGetAttribute(&sm_count, cudaDevAttrMultiProcessorCount, device));
  cudaStream_t st = nullptr;
  TSV_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  std::vector<void*> live;
  auto alloc = [&](size_t bytes) -> void* {
    void* p = nullptr;
    if (!alloc_retry(&p, bytes ? bytes : 8, st))
      throw CudaError("device graph build: out of device memory");
    live.push_back(p);
    return p;
  };
  auto release = [&](void* p) {
    auto it = std::find(live.begin(), live.end(), p);
    if (it != live.end()) live.erase(it);
    cudaFreeAsync(p, st);
  };
  auto* g = new tsv_graph();
  g->device = device;
  g->model = model;
  g->host.n = n;
  g->host.directed = directed;
  try {
    int32_t* du = static_cast<int32_t*>(alloc(std::max<int64_t>(m, 1) * 4));
    int32_t* dv = static_cast<int32_t*>(alloc(std::max<int64_t>(m, 1) * 4));
    int32_t* dts = static_cast<int32_t*>(alloc(std::max<int64_t>(m, 1) * 4));
    if (m) {
      // pageable host arrays go through the pinned staging buffers
      cudaPointerAttributes pa{};
      const bool pageable = kind == cudaMemcpyHostToDevice &&
                            (cudaPointerGetAttributes(&pa, u) != cudaSuccess ||
                             pa.type == cudaMemoryTypeUnregistered);
      cudaGetLastError();  // (clear a failed attribute query)
      if (pageable) {
        copy_to_device(du, u, m * 4, st);
        copy_to_device(dv, v, m * 4, st);
        copy_to_device(dts, ts, m * 4, st);
      } else {
        TSV_CUDA(cudaMemcpyAsync(du, u, m * 4, kind, st));
        TSV_CUDA(cudaMemcpyAsync(dv, v, m * 4, kind, st));
        TSV_CUDA(cudaMemcpyAsync(dts, ts, m * 4, kind, st));
      }
    }
    // edge model (sieve.cpp:179-186): transition times when model 1/3,
    // vertex delays (0 when none were given) when model 2/3
    const bool use_eps = model == 1 || model == 3, use_delay = model == 2 || model == 3;
    int32_t *deps = nullptr, *ddel = nullptr;
    if (use_eps) {
      deps = static_cast<int32_t*>(alloc(std::max<int64_t>(m, 1) * 4));
      if (m && eps) TSV_CUDA(cudaMemcpyAsync(deps, eps, m * 4, kind, st));
      else if (m) {
        std::vector<int32_t> ones(static_cast<size_t>(m), 1);
        TSV_CUDA(cudaMemcpyAsync(deps, ones.data(), m * 4, cudaMemcpyHostToDevice, st));
        TSV_CUDA(cudaStreamSynchronize(st));
      }
    }
    if (use_delay) {
      ddel = static_cast<int32_t*>(alloc(std::max<int64_t>(n, 1) * 4));
      if (n && delays) TSV_CUDA(cudaMemcpyAsync(ddel, delays, static_cast<size_t>(n) * 4, kind, st));
      else if (n) TSV_CUDA(cudaMemsetAsync(ddel, 0, static_cast<size_t>(n) * 4, st));
    }
    const char* tre = std::getenv("TSV_TRACE_BUILD");
    const bool trace = tre && tre[0] == '1';
    const auto tb0 = std::chrono::steady_clock::now();
    auto mark = [&](const char* what) {
      if (!trace) return;
      cudaStreamSynchronize(st);
      std::fprintf(stderr, "[build] %-28s %9.1f ms (total)\n", what,
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() -
                                                             tb0).count());
    };
    mark("uploads");
    auto* status = static_cast<tsv::BuildStatus*>(alloc(sizeof(tsv::BuildStatus)));
    tsv::DeviceLayout L;
    tsv::device_build(du, dv, dts, m, n, directed, canonical, L, status,
                      sm_count, st, alloc, release, deps, ddel);
    if (deps) release(deps);
    if (ddel) release(ddel);
    tsv::BuildStatus hs{};
    TSV_CUDA(cudaMemcpyAsync(&hs, status, sizeof(hs), cudaMemcpyDeviceToHost, st));
    TSV_CUDA(cudaStreamSynchronize(st));
    TSV_CUDA(cudaGetLastError());
    release(du);
    release(dv);
    release(dts);
    release(status);
    if (hs.first_bad_endpoint != INT64_MAX || hs.first_bad_ts != INT64_MAX)
      throw std::invalid_argument(hs.first_bad_endpoint <= hs.first_bad_ts
                                      ? "edge endpoint out of range"
                                      : "timestamp below 1");
    if (hs.not_canonical) throw std::invalid_argument("edge list is not canonical");
    if (L.m >= static_cast<int64_t>(tsv::kEdgeMask))
      throw std::invalid_argument("edge count exceeds the engine's 2^30 edge ids");
    const int32_t max_ts = hs.max_ts;
    g->host.t = t > 0 ? t : std::max<int32_t>(max_ts, 1);
    if (L.m > 0 && max_ts > g->host.t) throw std::invalid_argument("timestamp exceeds t");
    g->host.dropped_self_loops = canonical ? 0 : hs.self_loops;
    g->host.dropped_duplicates = L.dropped_duplicates;
    g->m = L.m;
    const char* eil = std::getenv("TSV_EDGES_IN_LAYOUT");  // (tests: force the mode)
    if ((L.m > (int64_t{1} << 26) || (eil && eil[0] == '1')) && model == 0) {
      // large graphs: the canonical edge list is needed only on demand
      // (tsv_graph_edges, restriction, EC/VC); it is rebuilt from the layout
      // then (edges_from_layout), so neither HBM nor a host copy holds it
      g->edges_in_layout = true;
      release(L.eu);
      release(L.ev);
      release(L.ets);
    } else {
      g->d_eu = L.eu;
      g->d_ev = L.ev;
      g->d_ets = L.ets;
    }
    tsv::DevGraph& d = g->dev;
    d.n = n;
    d.A = L.A;
    d.R = L.R;
    d.C = L.C;
    d.arc_src = L.arc_src;
    d.arc_meta = L.arc_meta;
    d.arc_tail = L.arc_tail;
    d.run_head = L.run_head;
    d.run_ts = L.run_ts;
    d.vtx_run_off = L.vtx_run_off;
    d.chunk_arc = L.chunk_arc;
    d.chunk_run = L.chunk_run;
    d.chunk_carry = L.chunk_carry;
    d.carry_list = L.carry_list;
    d.ncarry = L.ncarry;
    auto* slots = static_cast<int32_t*>(alloc(std::max<int64_t>(L.R, 1) * 4));
    const tsv::SlotCounts sc = tsv::build_run_slots(L.A, L.R, L.arc_src, slots, st,
                                                    force_last_runs ? L.vtx_run_off : nullptr, n);
    g->arcs_with_src = sc.arcs_with_src;
    g->runs_referenced = sc.slots;
    d.run_slot = slots;
    d.S = sc.slots;
    mark("state slots");
    g->device_bytes = 12 * L.A + 12 * L.R + 4 * (static_cast<int64_t>(n) + 1) + 12 * L.m +
                      17 * (L.C + 1);
    TSV_CUDA(cudaStreamSynchronize(st));
    g->owned = live;
    live.clear();
    cudaStreamDestroy(st);
  } catch (...) {
    for (void* p : live) cudaFreeAsync(p, st);
    cudaStreamSynchronize(st);
    cudaStreamDestroy(st);
    delete g;
    throw;
  }
  return g;
}

// Graph restricted to the vertices with at least one shade, keeping vertex ids
// and the original edge ids in arc_meta (so every y draw is the full graph's).
// An arc with a shadeless endpoint adds nothing in the full graph: a
// shadeless tail's rows are zero at every level (z = 0), a shadeless head's
// rows are never read and its accumulator is zero; a run whose arcs all came
// from shadeless tails only repeats its vertex's prefix, so an arc's source
// (the tail's last run before it) has the same prefix in both graphs.  Built
// once per (graph, shades) on the graph's device; used by the coefficient
// engine when it drops >= 15% of the arcs (C2: 61%), else the graph itself.
std::shared_ptr<tsv_graph> shaded_subgraph(const tsv_graph* g, const tsv_shades* sh) {
  const char* env = std::getenv("TSV_SUBGRAPH");
  if (g->model != 0 || (env && env[0] == '0') || g->host.n == 0) return nullptr;
  // every vertex has a shade (k-TempPath, C5): nothing to drop
  if (sh->single + sh->multi >= static_cast<int64_t>(g->host.n)) return nullptr;
  std::lock_guard<std::mutex> lk(sh->sub_mu);
  for (const auto& e : sh->subs)
    if (e.uid == g->uid) return e.sub;
  if (sh->subs.size() >= 4) sh->subs.erase(sh->subs.begin());
  sh->subs.push_back({g->uid, nullptr});  // "not worth it" unless built below
  DeviceGuard dg(g->device);
  cudaStream_t st = nullptr;
  TSV_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  std::vector<void*> tmp;
  auto alloc = [&](size_t bytes) -> void* {
    void* p = nullptr;
    if (!alloc_retry(&p, bytes ? bytes : 8, st))
      throw CudaError("shaded subgraph: out of device memory");
    tmp.push_back(p);
    return p;
  };
  auto release = [&](void* p) {
    auto it = std::find(tmp.begin(), tmp.end(), p);
    if (it != tmp.end()) tmp.erase(it);
    cudaFreeAsync(p, st);
  };
  auto done = [&] {
    for (void* p : tmp) cudaFreeAsync(p, st);
    cudaStreamSynchronize(st);
    cudaStreamDestroy(st);
  };
  try {
    const int32_t n = g->host.n;
    const int64_t m = g->m;
    auto* keep = static_cast<uint8_t*>(alloc(static_cast<size_t>(n)));
    tsv::launch_shaded_mask(n, sh->off, keep, st);
    const int32_t *eu = g->d_eu, *ev = g->d_ev, *ets = g->d_ets;
    if (!eu && g->edges_in_layout) {
      auto* a = static_cast<int32_t*>(alloc(std::max<int64_t>(m, 1) * 4));
      auto* b = static_cast<int32_t*>(alloc(std::max<int64_t>(m, 1) * 4));
      auto* c = static_cast<int32_t*>(alloc(std::max<int64_t>(m, 1) * 4));
      tsv::edges_from_layout(g->dev, g->host.directed, a, b, c, st);
      eu = a;
      ev = b;
      ets = c;
    } else if (!eu) {
      auto* a = static_cast<int32_t*>(alloc(std::max<int64_t>(m, 1) * 4));
      auto* b = static_cast<int32_t*>(alloc(std::max<int64_t>(m, 1) * 4));
      auto* c = static_cast<int32_t*>(alloc(std::max<int64_t>(m, 1) * 4));
      if (m) {
        TSV_CUDA(cudaMemcpyAsync(a, g->host.eu.data(), m * 4, cudaMemcpyHostToDevice, st));
        TSV_CUDA(cudaMemcpyAsync(b, g->host.ev.data(), m * 4, cudaMemcpyHostToDevice, st));
        TSV_CUDA(cudaMemcpyAsync(c, g->host.ets.data(), m * 4, cudaMemcpyHostToDevice, st));
      }
      eu = a;
      ev = b;
      ets = c;
    }
    auto* ou = static_cast<int32_t*>(alloc(std::max<int64_t>(m, 1) * 4));
    auto* ov = static_cast<int32_t*>(alloc(std::max<int64_t>(m, 1) * 4));
    auto* ots = static_cast<int32_t*>(alloc(std::max<int64_t>(m, 1) * 4));
    auto* oid = static_cast<int32_t*>(alloc(std::max<int64_t>(m, 1) * 4));
    const int64_t kept = tsv::device_restrict(eu, ev, ets, m, keep, g->host.t, ou, ov, ots, st,
                                              alloc, release, oid);
    if (kept * 100 > m * 85) {
      done();
      return nullptr;
    }
    TSV_CUDA(cudaStreamSynchronize(st));
    tsv_graph* s = device_graph_build(n, kept, ou, ov, ots, g->host.directed, g->host.t,
                                      g->device, /*canonical=*/true, /*on_device=*/true);
    tsv::launch_remap_edge_ids(s->dev.A, const_cast<uint32_t*>(s->dev.arc_meta), oid, st);
    TSV_CUDA(cudaGetLastError());
    done();
    std::shared_ptr<tsv_graph> sp(s);
    sh->subs.back().sub = sp;
    return sp;
  } catch (...) {
    done();
    throw;
  }
}


// a == b over `count` words, compared on all host threads
template <typename T>
bool equal_par(const T* a, const T* b, size_t count) {
  if (count == 0 || a == b) return true;
  if (count < (size_t{1} << 20)) return std::memcmp(a, b, count * sizeof(T)) == 0;
  const size_t block = size_t{1} << 18;
  const int64_t nb = static_cast<int64_t>((count + block - 1) / block);
  int diff = 0;
#pragma omp parallel for schedule(static) reduction(| : diff)
  for (int64_t i = 0; i < nb; ++i) {
    const size_t lo = static_cast<size_t>(i) * block, len = std::min(block, count - lo);
    diff |= std::memcmp(a + lo, b + lo, len * sizeof(T)) != 0;
  }
  return diff == 0;
}

// dst = src[0..count), copied on all host threads
void copy_par(std::vector<int32_t>& dst, const int32_t* src, size_t count) {
  dst.resize(count);
  const size_t block = size_t{1} << 20;
  const int64_t nb = static_cast<int64_t>((count + block - 1) / block);
#pragma omp parallel for schedule(static) if (nb > 4)
  for (int64_t i = 0; i < nb; ++i) {
    const size_t lo = static_cast<size_t>(i) * block, len = std::min(block, count - lo);
    std::memcpy(dst.data() + lo, src + lo, len * sizeof(int32_t));
  }
}

// Copies between device memory and pageable host memory through two pinned
// staging buffers per device (reused by every call): the DMA of one chunk
// overlaps the host threads moving the neighbouring chunk.  Plain cudaMemcpy
// from/to pageable memory stages through the driver at a fraction of the
// link rate (C5: 800 MB of accumulators, 2.4 GB of shade CSR).
struct Staging {
  static constexpr size_t kChunk = size_t{32} << 20;
  std::mutex mu;
  void* buf[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
};

Staging& staging() {
  static std::mutex reg_mu;
  static std::vector<std::unique_ptr<Staging>> reg;
  int dev = 0;
  TSV_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(reg_mu);
  if (reg.size() <= static_cast<size_t>(dev)) reg.resize(static_cast<size_t>(dev) + 1);
  if (!reg[dev]) {
    auto st = std::make_unique<Staging>();
    for (int i = 0; i < 2; ++i) {
      TSV_CUDA(cudaMallocHost(&st->buf[i], Staging::kChunk));
      TSV_CUDA(cudaEventCreateWithFlags(&st->ev[i], cudaEventDisableTiming));
    }
    reg[dev] = std::move(st);
  }
  return *reg[dev];
}

void memcpy_par(char* dst, const char* src, size_t len) {
  const int64_t parts = len >= (size_t{4} << 20) ? 16 : 1;
#pragma omp parallel for schedule(static) num_threads(16) if (parts > 1)
  for (int64_t p = 0; p < parts; ++p) {
    const size_t lo = len * p / parts, hi = len * (p + 1) / parts;
    std::memcpy(dst + lo, src + lo, hi - lo);
  }
}

void copy_to_host(void* dst, const void* d_src, size_t bytes, cudaStream_t st) {
  if (bytes == 0) return;
  if (bytes < (size_t{8} << 20)) {
    TSV_CUDA(cudaMemcpyAsync(dst, d_src, bytes, cudaMemcpyDeviceToHost, st));
    TSV_CUDA(cudaStreamSynchronize(st));
    return;
  }
  Staging& S = staging();
  std::lock_guard<std::mutex> lk(S.mu);
  const size_t K = Staging::kChunk, nchunks = (bytes + K - 1) / K;
  auto issue = [&](size_t c) {
    const size_t off = c * K, len = std::min(K, bytes - off);
    TSV_CUDA(cudaMemcpyAsync(S.buf[c & 1], static_cast<const char*>(d_src) + off, len,
                             cudaMemcpyDeviceToHost, st));
    TSV_CUDA(cudaEventRecord(S.ev[c & 1], st));
  };
  issue(0);
  for (size_t c = 0; c < nchunks; ++c) {
    if (c + 1 < nchunks) issue(c + 1);  // buffer (c+1)&1 was drained in step c-1
    TSV_CUDA(cudaEventSynchronize(S.ev[c & 1]));
    const size_t off = c * K, len = std::min(K, bytes - off);
    memcpy_par(static_cast<char*>(dst) + off, static_cast<const char*>(S.buf[c & 1]), len);
  }
}

// Host -> device; returns once the source may be reused (the last DMAs are
// complete).
void copy_to_device(void* d_dst, const void* src, size_t bytes, cudaStream_t st) {
  if (bytes == 0) return;
  if (bytes < (size_t{8} << 20)) {
    TSV_CUDA(cudaMemcpyAsync(d_dst, src, bytes, cudaMemcpyHostToDevice, st));
    TSV_CUDA(cudaStreamSynchronize(st));
    return;
  }
  Staging& S = staging();
  std::lock_guard<std::mutex> lk(S.mu);
  const size_t K = Staging::kChunk, nchunks = (bytes + K - 1) / K;
  for (size_t c = 0; c < nchunks; ++c) {
    if (c >= 2) TSV_CUDA(cudaEventSynchronize(S.ev[c & 1]));  // DMA of chunk c-2 done
    const size_t off = c * K, len = std::min(K, bytes - off);
    memcpy_par(static_cast<char*>(S.buf[c & 1]), static_cast<const char*>(src) + off, len);
    TSV_CUDA(cudaMemcpyAsync(static_cast<char*>(d_dst) + off, S.buf[c & 1], len,
                             cudaMemcpyHostToDevice, st));
    TSV_CUDA(cudaEventRecord(S.ev[c & 1], st));
  }
  TSV_CUDA(cudaStreamSynchronize(st));
}

}  // namespace

extern "C" {

const char* tsv_last_error(void) { return g_error.c_str(); }
const char* tsv_version(void) { return "tsv-b200 0.1 (sm_100a)"; }

static int graph_build_impl(int32_t n, int64_t m, const int32_t* u, const int32_t* v,
                            const int32_t* ts, int directed, int32_t t, int device,
                            tsv_graph** out, bool canonical, const int32_t* eps = nullptr,
                            const int32_t* delays = nullptr, int model = 0) {
  return guard([&] {
    if (!out) throw std::invalid_argument("null output handle");
    *out = nullptr;
    if (m < 0) throw std::invalid_argument("negative edge count");
    if (m > 0 && (!u || !v || !ts)) throw std::invalid_argument("null edge arrays");
    if (n < 0) throw std::invalid_argument("negative vertex count");
    if (model < 0 || model > 3) throw std::invalid_argument("edge_model must be 0..3");
    const char* hb = std::getenv("TSV_HOST_BUILD");
    if (model != 0 || !(hb && hb[0] == '1')) {
      *out = device_graph_build(n, m, u, v, ts, directed != 0, t, device, canonical, false, eps,
                                delays, model);
      return;
    }
    auto* g = new tsv_graph();
    try {
      g->device = device;
      if (canonical)
        tsv::adopt_canonical(n, m, u, v, ts, directed != 0, t, g->host);
      else
        tsv::canonicalize(n, m, u, v, ts, directed != 0, t, g->host);
      g->m = static_cast<int64_t>(g->host.eu.size());
      DeviceGuard dg(device);
      int sm_count = 0;
      TSV_CUDA(cudaDeviceGetAttribute(&sm_count, cudaDevAttrMultiProcessorCount, device));
      tsv::build_layout(g->host, 0, sm_count);
      tsv::HostLayout& L = g->host;
      tsv::DevGraph& d = g->dev;
      d.n = L.n;
      d.A = static_cast<int64_t>(L.arc_src.size());
      d.R = static_cast<int64_t>(L.run_head.size());
      d.C = static_cast<int64_t>(L.chunk_carry.size());
      d.arc_src = own_upload(g, L.arc_src);
      d.arc_meta = own_upload(g, L.arc_meta);
      d.arc_tail = own_upload(g, L.arc_tail);
      d.run_head = own_upload(g, L.run_head);
      d.run_ts = own_upload(g, L.run_ts);
      d.vtx_run_off = own_upload(g, L.vtx_run_off);
      d.chunk_arc = own_upload(g, L.chunk_arc);
      d.chunk_run = own_upload(g, L.chunk_run);
      d.chunk_carry = own_upload(g, L.chunk_carry);
      d.carry_list = own_upload(g, L.carry_list);
      d.ncarry = static_cast<int32_t>(L.carry_list.size());
      int32_t* slots = dalloc<int32_t>(std::max<size_t>(L.run_head.size(), 1));
      g->owned.push_back(slots);
      g->device_bytes += 4 * static_cast<int64_t>(std::max<size_t>(L.run_head.size(), 1));
      const tsv::SlotCounts sc =
          tsv::build_run_slots(d.A, d.R, const_cast<int32_t*>(d.arc_src), slots, nullptr);
      g->arcs_with_src = sc.arcs_with_src;
      g->runs_referenced = sc.slots;
      d.run_slot = slots;
      d.S = sc.slots;
      // release the host copies of the device layout (keep canonical edges)
      std::vector<int32_t>().swap(L.arc_src);
      std::vector<int32_t>().swap(L.arc_tail);
      std::vector<uint32_t>().swap(L.arc_meta);
      std::vector<int32_t>().swap(L.run_head);
      std::vector<int32_t>().swap(L.run_ts);
      TSV_CUDA(cudaDeviceSynchronize());
    } catch (...) {
      delete g;
      throw;
    }
    *out = g;
  });
}

int tsv_graph_build(int32_t n, int64_t m, const int32_t* u, const int32_t* v,
                    const int32_t* ts, int directed, int32_t t, int device,
                    tsv_graph** out) {
  return graph_build_impl(n, m, u, v, ts, directed, t, device, out, false);
}

int tsv_graph_build_canonical(int32_t n, int64_t m, const int32_t* u, const int32_t* v,
                              const int32_t* ts, int directed, int32_t t, int device,
                              tsv_graph** out) {
  return graph_build_impl(n, m, u, v, ts, directed, t, device, out, true);
}

int tsv_graph_build_model(int32_t n, int64_t m, const int32_t* u, const int32_t* v,
                          const int32_t* ts, const int32_t* eps, const int32_t* delays,
                          int directed, int32_t t, int edge_model, int device,
                          tsv_graph** out) {
  if (edge_model != 0 && delays) {
    for (int32_t x = 0; x < n; ++x)
      if (delays[x] < 0) {
        g_error = "negative vertex delay";
        return TSV_ERR_INVALID;
      }
  }
  if (eps)
    for (int64_t i = 0; i < m; ++i)
      if (eps[i] < 1) {
        g_error = "transition time below 1";
        return TSV_ERR_INVALID;
      }
  return graph_build_impl(n, m, u, v, ts, directed, t, device, out, true, eps, delays,
                          edge_model);
}

int64_t tsv_canonical_edges(int32_t n, int64_t m, const int32_t* u, const int32_t* v,
                            const int32_t* ts, int directed, int32_t* out_u, int32_t* out_v,
                            int32_t* out_ts) {
  return tsv_canonical_edges_eps(n, m, u, v, ts, nullptr, directed, out_u, out_v, out_ts,
                                 nullptr);
}

int64_t tsv_canonical_edges_eps(int32_t n, int64_t m, const int32_t* u, const int32_t* v,
                                const int32_t* ts, const int32_t* eps, int directed,
                                int32_t* out_u, int32_t* out_v, int32_t* out_ts,
                                int32_t* out_eps) {
  int64_t kept = -1;
  int rc = guard([&] {
    tsv::HostLayout L;
    tsv::canonicalize(n, m, u, v, ts, directed != 0, 0, L, eps);
    kept = static_cast<int64_t>(L.eu.size());
    for (int64_t i = 0; i < kept; ++i) {
      out_u[i] = L.eu[i];
      out_v[i] = L.ev[i];
      out_ts[i] = L.ets[i];
      if (out_eps) out_eps[i] = eps ? L.eeps[i] : 1;
    }
  });
  return rc == TSV_OK ? kept : -1;
}

int tsv_graph_restrict(const tsv_graph* g, const uint8_t* keep_vertex, int32_t max_ts,
                       tsv_graph** out) {
  return guard([&] {
    if (!g || !out || (g->host.n > 0 && !keep_vertex))
      throw std::invalid_argument("null argument");
    *out = nullptr;
    if (g->model != 0)
      throw std::invalid_argument(
          "tsv_graph_restrict: graphs of non-instant edge models are rebuilt from the host "
          "(tsv_graph_build_model)");
    DeviceGuard dg(g->device);
    cudaStream_t st = nullptr;
    TSV_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    std::vector<void*> tmp;
    auto alloc = [&](size_t bytes) -> void* {
      void* p = nullptr;
      if (!alloc_retry(&p, bytes ? bytes : 8, st))
        throw CudaError("restrict: out of device memory");
      tmp.push_back(p);
      return p;
    };
    auto release = [&](void* p) {
      auto it = std::find(tmp.begin(), tmp.end(), p);
      if (it != tmp.end()) tmp.erase(it);
      cudaFreeAsync(p, st);
    };
    try {
      const int32_t n = g->host.n;
      const int64_t m = g->m;
      auto* keep = static_cast<uint8_t*>(alloc(std::max<int64_t>(n, 1)));
      if (n) TSV_CUDA(cudaMemcpyAsync(keep, keep_vertex, n, cudaMemcpyHostToDevice, st));
      const int32_t *eu = g->d_eu, *ev = g->d_ev, *ets = g->d_ets;
      if (!eu && g->edges_in_layout) {  // rebuilt on the device from the layout
        auto* a = static_cast<int32_t*>(alloc(std::max<int64_t>(m, 1) * 4));
        auto* b = static_cast<int32_t*>(alloc(std::max<int64_t>(m, 1) * 4));
        auto* c = static_cast<int32_t*>(alloc(std::max<int64_t>(m, 1) * 4));
        tsv::edges_from_layout(g->dev, g->host.directed, a, b, c, st);
        eu = a;
        ev = b;
        ets = c;
      } else if (!eu) {  // canonical edges held on the host: stage them
        auto* a = static_cast<int32_t*>(alloc(std::max<int64_t>(m, 1) * 4));
        auto* b = static_cast<int32_t*>(alloc(std::max<int64_t>(m, 1) * 4));
        auto* c = static_cast<int32_t*>(alloc(std::max<int64_t>(m, 1) * 4));
        if (m) {
          TSV_CUDA(cudaMemcpyAsync(a, g->host.eu.data(), m * 4, cudaMemcpyHostToDevice, st));
          TSV_CUDA(cudaMemcpyAsync(b, g->host.ev.data(), m * 4, cudaMemcpyHostToDevice, st));
          TSV_CUDA(cudaMemcpyAsync(c, g->host.ets.data(), m * 4, cudaMemcpyHostToDevice, st));
        }
        eu = a;
        ev = b;
        ets = c;
      }
      auto* ou = static_cast<int32_t*>(alloc(std::max<int64_t>(m, 1) * 4));
      auto* ov = static_cast<int32_t*>(alloc(std::max<int64_t>(m, 1) * 4));
      auto* ots = static_cast<int32_t*>(alloc(std::max<int64_t>(m, 1) * 4));
      const int64_t kept =
          tsv::device_restrict(eu, ev, ets, m, keep, max_ts, ou, ov, ots, st, alloc, release);
      const int32_t t_new = std::min(max_ts, g->host.t);
      TSV_CUDA(cudaStreamSynchronize(st));
      *out = device_graph_build(n, kept, ou, ov, ots, g->host.directed, t_new, g->device,
                                /*canonical=*/true, /*on_device=*/true);
    } catch (...) {
      for (void* p : tmp) cudaFreeAsync(p, st);
      cudaStreamSynchronize(st);
      cudaStreamDestroy(st);
      throw;
    }
    for (void* p : tmp) cudaFreeAsync(p, st);
    cudaStreamSynchronize(st);
    cudaStreamDestroy(st);
  });
}

void tsv_graph_free(tsv_graph* g) { delete g; }

int tsv_graph_get_info(const tsv_graph* g, tsv_graph_info* out) {
  return guard([&] {
    if (!g || !out) throw std::invalid_argument("null argument");
    out->n = g->host.n;
    out->t = g->host.t;
    out->directed = g->host.directed ? 1 : 0;
    out->device = g->device;
    out->m = g->m;
    out->arcs = g->dev.A;
    out->runs = g->dev.R;
    out->chunks = g->dev.C;
    out->split_chunks = g->dev.ncarry;
    out->dropped_self_loops = g->host.dropped_self_loops;
    out->dropped_duplicates = g->host.dropped_duplicates;
    out->device_bytes = g->device_bytes;
    out->arcs_with_src = g->arcs_with_src;
    out->runs_referenced = g->runs_referenced;
  });
}

int tsv_graph_edges(const tsv_graph* g, int32_t* u, int32_t* v, int32_t* ts) {
  return guard([&] {
    if (!g) throw std::invalid_argument("null graph");
    const size_t m = static_cast<size_t>(g->m);
    if (g->d_eu) {  // device-built: canonical edges live in HBM
      DeviceGuard dg(g->device);
      if (m && u) TSV_CUDA(cudaMemcpy(u, g->d_eu, m * 4, cudaMemcpyDeviceToHost));
      if (m && v) TSV_CUDA(cudaMemcpy(v, g->d_ev, m * 4, cudaMemcpyDeviceToHost));
      if (m && ts) TSV_CUDA(cudaMemcpy(ts, g->d_ets, m * 4, cudaMemcpyDeviceToHost));
      return;
    }
    if (g->edges_in_layout) {  // large device-built graph: rebuild from the layout
      DeviceGuard dg(g->device);
      DevBuf a(m * 4 + 4, nullptr), b(m * 4 + 4, nullptr), c(m * 4 + 4, nullptr);
      tsv::edges_from_layout(g->dev, g->host.directed, a.as<int32_t>(), b.as<int32_t>(),
                             c.as<int32_t>(), nullptr);
      if (m && u) TSV_CUDA(cudaMemcpy(u, a.p, m * 4, cudaMemcpyDeviceToHost));
      if (m && v) TSV_CUDA(cudaMemcpy(v, b.p, m * 4, cudaMemcpyDeviceToHost));
      if (m && ts) TSV_CUDA(cudaMemcpy(ts, c.p, m * 4, cudaMemcpyDeviceToHost));
      return;
    }
    if (m && u) std::memcpy(u, g->host.eu.data(), m * 4);
    if (m && v) std::memcpy(v, g->host.ev.data(), m * 4);
    if (m && ts) std::memcpy(ts, g->host.ets.data(), m * 4);
  });
}

// Does every vertex carry the same shade list (k-TempPath: all k shades)?
// Then the CSR is (c, pattern) -- one parallel read of the caller's arrays
// instead of a 2.4 GB upload and host copy at C5.
static bool uniform_shades(int32_t n, const int32_t* off, const int32_t* vs, int32_t* c_out,
                           std::vector<int32_t>* pattern) {
  if (n < 1 || off[0] != 0) return false;
  const int32_t c = off[1] - off[0];
  if (c < 0 || static_cast<int64_t>(n) * c > INT32_MAX) return false;
  int bad = 0;
#pragma omp parallel for schedule(static) reduction(| : bad) if (n > (1 << 16))
  for (int32_t i = 0; i < n; ++i) {
    if (bad) continue;
    if (off[i + 1] - off[i] != c || off[i] != static_cast<int64_t>(i) * c) {
      bad = 1;
      continue;
    }
    for (int32_t j = 0; j < c; ++j)
      if (vs[static_cast<int64_t>(i) * c + j] != vs[j]) bad = 1;
  }
  if (bad) return false;
  *c_out = c;
  pattern->assign(vs, vs + c);
  return true;
}

// The upload behind tsv_shades_upload.  known_uniform: the caller has already
// found every vertex's list equal to `pattern` (c entries) with
// uniform_shades, so the per-entry scans below are not repeated (at C5 they
// read the 2.4 GB CSR three more times, ~80 ms of every fresh-graph decide).
static void shades_upload_impl(const tsv_graph* g, int k, const int32_t* vertex_off,
                               const int32_t* vertex_shades, bool known_uniform, int32_t c,
                               std::vector<int32_t> pattern, tsv_shades** out) {
  if (!g || !out || !vertex_off) throw std::invalid_argument("null argument");
  *out = nullptr;
  if (k < 1 || k > 30) throw std::invalid_argument("k out of range [1,30]");
  const int32_t n = g->host.n;
  if (vertex_off[0] != 0) throw std::invalid_argument("vertex_off[0] must be 0");
  const int64_t cnt = vertex_off[n];
  bool uni = known_uniform;
  if (!uni && cnt > (int64_t{1} << 20))
    uni = uniform_shades(n, vertex_off, vertex_shades, &c, &pattern);
  int64_t single = 0, multi = 0;
  if (uni) {
    // off[i] = i * c was checked by uniform_shades; the entries are the pattern's
    for (int32_t x : pattern)
      if (x < 1 || x > k) throw std::invalid_argument("shade id outside [1..k]");
    single = c == 1 ? n : 0;
    multi = c > 1 ? n : 0;
  } else {
    int bad_off = 0, bad_shade = 0;
#pragma omp parallel for schedule(static) reduction(| : bad_off)
    for (int32_t i = 0; i < n; ++i) bad_off |= vertex_off[i + 1] < vertex_off[i];
    if (bad_off) throw std::invalid_argument("vertex_off must be non-decreasing");
#pragma omp parallel for schedule(static) reduction(| : bad_shade)
    for (int64_t i = 0; i < cnt; ++i) bad_shade |= vertex_shades[i] < 1 || vertex_shades[i] > k;
    if (bad_shade) throw std::invalid_argument("shade id outside [1..k]");
#pragma omp parallel for schedule(static) reduction(+ : single, multi)
    for (int32_t i = 0; i < n; ++i) {
      single += vertex_off[i + 1] - vertex_off[i] == 1;
      multi += vertex_off[i + 1] - vertex_off[i] > 1;
    }
  }
  DeviceGuard dg(g->device);
  auto* s = new tsv_shades();
  s->k = k;
  s->n = n;
  s->single = single;
  s->multi = multi;
  s->device = g->device;
  try {
    // pool allocations (cudaMalloc costs ~0.1 ms per call); the copies go
    // through the pinned staging buffers and are complete on return
    TSV_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&s->off), (static_cast<size_t>(n) + 1) * 4,
                             nullptr));
    TSV_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&s->shades),
                             std::max<size_t>(static_cast<size_t>(cnt), 1) * 4, nullptr));
    TSV_CUDA(cudaStreamSynchronize(nullptr));
    if (uni) {
      // every vertex the same list: expand (c, pattern) on the device
      int32_t* dp = nullptr;
      TSV_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dp), std::max<size_t>(c, 1) * 4,
                               nullptr));
      TSV_CUDA(cudaMemcpy(dp, pattern.data(), static_cast<size_t>(c) * 4,
                          cudaMemcpyHostToDevice));
      tsv::launch_uniform_csr(n, c, dp, s->off, s->shades, nullptr);
      TSV_CUDA(cudaFreeAsync(dp, nullptr));
      TSV_CUDA(cudaStreamSynchronize(nullptr));
    } else {
      copy_to_device(s->off, vertex_off, (static_cast<size_t>(n) + 1) * 4, nullptr);
      copy_to_device(s->shades, vertex_shades, static_cast<size_t>(cnt) * 4, nullptr);
    }
  } catch (...) {
    delete s;
    throw;
  }
  *out = s;
}

int tsv_shades_upload(const tsv_graph* g, int k, const int32_t* vertex_off,
                      const int32_t* vertex_shades, tsv_shades** out) {
  return guard([&] {
    shades_upload_impl(g, k, vertex_off, vertex_shades, false, 0, {}, out);
  });
}

void tsv_shades_free(tsv_shades* s) { delete s; }

int tsv_eval_points_device(const tsv_graph* g, const tsv_shades* s, int k,
                           int32_t max_ts, const tsv_config* cfg,
                           int32_t anchor_source, uint64_t p_begin, uint64_t p_end,
                           uint64_t* d_acc, void* stream) {
  return guard([&] {
    if (!g || !d_acc) throw std::invalid_argument("null argument");
    DeviceGuard dg(g->device);
    eval_device(g, s, k, max_ts, cfg, anchor_source, p_begin, p_end, d_acc,
                static_cast<cudaStream_t>(stream), nullptr);
  });
}

int tsv_eval_temporal_sieve(const tsv_graph* g, int k, int32_t max_ts,
                            const int32_t* vertex_off, const int32_t* vertex_shades,
                            const tsv_config* cfg, int32_t anchor_source,
                            int32_t anchor_sink, uint64_t* accumulators,
                            tsv_outcome* out) {
  return guard([&] {
    if (!g || !accumulators || !out || !vertex_off)
      throw std::invalid_argument("null argument");
    check_config(cfg, true);
    if (max_ts < 1 || max_ts > g->host.t) throw std::invalid_argument("max_ts outside [1..t]");
    if (k < 1 || k > 30) throw std::invalid_argument("k out of range [1,30]");
    const int32_t n = g->host.n;
    const int64_t cnt = vertex_off[n];
    // TSV_TRACE_API=1: phase wall times of this call on stderr
    const char* tre = std::getenv("TSV_TRACE_API");
    const bool trace = tre && tre[0] == '1';
    auto t_last = std::chrono::steady_clock::now();
    auto mark = [&](const char* what, cudaStream_t sync) {
      if (!trace) return;
      if (sync) cudaStreamSynchronize(sync);
      const auto now = std::chrono::steady_clock::now();
      std::fprintf(stderr, "[api] %-24s %9.1f ms\n", what,
                   std::chrono::duration<double, std::milli>(now - t_last).count());
      t_last = now;
    };
    if (cnt < 0 || (cnt > 0 && !vertex_shades)) throw std::invalid_argument("null argument");
    // a repeated shade table (every probe of one query) is not uploaded
    // again: reuse the cached device copy when the CSR is word-for-word equal
    // (a uniform CSR -- every vertex the same list -- is kept as its pattern)
    std::shared_ptr<tsv_shades> hold;
    int32_t uc = 0;
    std::vector<int32_t> upat;
    const bool uni = cnt > (int64_t{1} << 20) &&
                     uniform_shades(n, vertex_off, vertex_shades, &uc, &upat);
    {
      std::lock_guard<std::mutex> lk(g->shade_mu);
      if (g->shade_cache && g->shade_k == k) {
        if (g->shade_uniform)
          hold = uni && uc == g->shade_uc && upat == g->shade_upat ? g->shade_cache : nullptr;
        else if (!uni && g->shade_off_copy.size() == static_cast<size_t>(n) + 1 &&
                 g->shade_vs_copy.size() == static_cast<size_t>(cnt) &&
                 equal_par(g->shade_off_copy.data(), vertex_off, static_cast<size_t>(n) + 1) &&
                 equal_par(g->shade_vs_copy.data(), vertex_shades, static_cast<size_t>(cnt)))
          hold = g->shade_cache;
      }
    }
    mark(hold ? "shade compare (hit)" : "shade compare (miss)", nullptr);
    if (!hold) {
      tsv_shades* sh = nullptr;
      shades_upload_impl(g, k, vertex_off, vertex_shades, uni, uc, upat, &sh);
      hold = std::shared_ptr<tsv_shades>(sh, tsv_shades_free);
      std::lock_guard<std::mutex> lk(g->shade_mu);
      g->shade_cache = hold;
      g->shade_k = k;
      g->shade_uniform = uni;
      if (uni) {
        g->shade_uc = uc;
        g->shade_upat = upat;
        std::vector<int32_t>().swap(g->shade_off_copy);
        std::vector<int32_t>().swap(g->shade_vs_copy);
      } else {
        copy_par(g->shade_off_copy, vertex_off, static_cast<size_t>(n) + 1);
        copy_par(g->shade_vs_copy, vertex_shades, static_cast<size_t>(cnt));
      }
      mark("shade upload + host copy", nullptr);
    }
    DeviceGuard dg(g->device);
    // the graph's stream; a concurrent call on the same graph gets its own
    std::unique_lock<std::mutex> slk(g->stream_mu, std::try_to_lock);
    cudaStream_t st = nullptr;
    struct TmpStream {
      cudaStream_t s = nullptr;
      ~TmpStream() {
        if (s) {
          cudaStreamSynchronize(s);
          cudaStreamDestroy(s);
        }
      }
    } tmp;
    if (slk.owns_lock()) {
      if (!g->api_stream)
        TSV_CUDA(cudaStreamCreateWithFlags(&g->api_stream, cudaStreamNonBlocking));
      st = g->api_stream;
    } else {
      TSV_CUDA(cudaStreamCreateWithFlags(&tmp.s, cudaStreamNonBlocking));
      st = tmp.s;
    }
    uint64_t peak = 0;
    DevBuf acc(static_cast<size_t>(n) * 8, st);
    TSV_CUDA(cudaMemsetAsync(acc.p, 0, static_cast<size_t>(n) * 8, st));
    mark("stream + acc", st);
    eval_device(g, hold.get(), k, max_ts, cfg, anchor_source, 0, 1ull << k, acc.as<uint64_t>(),
                st, &peak);
    mark("sieve", st);
    // finalize on the device (sink restriction, flagged count, checksum),
    // then the accumulators to the caller through pinned staging buffers
    uint64_t checksum = 0;
    int64_t flagged = 0;
    tsv::device_finalize(acc.as<uint64_t>(), n, anchor_sink, st, &checksum, &flagged);
    mark("device finalize", st);
    copy_to_host(accumulators, acc.p, static_cast<size_t>(n) * 8, st);
    mark("accumulators to host", st);
    out->flagged = flagged;
    out->global_nonzero = flagged > 0;
    out->checksum = checksum;
    out->fn_bound = (2.0 * k - 1.0) / std::pow(2.0, cfg->field_bits);
    out->peak_field_words = peak;
  });
}

int tsv_vertex_partition(const tsv_graph* g, const tsv_shades* s, int k, int rank,
                         int world, tsv_partition* out) {
  return guard([&] {
    if (!g || !s || !out) throw std::invalid_argument("null argument");
    if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("bad rank/world");
    if (s->n != g->dev.n || s->k != k) throw std::invalid_argument("shade assignment built for a different graph");
    std::memset(out, 0, sizeof(*out));
    if (!tsv::vertex_engine_supports(k) || g->model != 0) return;
    DeviceGuard dg(g->device);
    cudaStream_t st = nullptr;
    TSV_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    struct Del {
      cudaStream_t s;
      ~Del() {
        cudaStreamSynchronize(s);
        cudaStreamDestroy(s);
      }
    } del{st};
    const tsv_graph::VertPart& vp = vertex_part(g, rank, world, st);
    const tsv::CoefTables& T = coef_const_tables(k);
    int64_t M = 1;
    for (int l = 1; l < k; ++l) M = std::max<int64_t>(M, T.count[l]);
    out->applicable = vp.applicable && s->single == 0 ? 1 : 0;
    out->slot_lo = vp.slot_lo;
    out->slot_hi = vp.slot_hi;
    out->slots = g->dev.S;
    for (int l = 1; l < k; ++l) M = std::max<int64_t>(M, tsv::vertex_row_words(k, l));
    out->state_words = std::max<int64_t>(g->dev.S, 1) * M;
    for (int l = 0; l <= k && l < 32; ++l) out->row_words[l] = tsv::vertex_row_words(k, l);
  });
}

// The partition `rank` of `world` with its exchange lists (and reader mask)
// built on first use, on `st`.
static const tsv_graph::VertPart& exchange_part(const tsv_graph* g, int rank, int world,
                                                cudaStream_t st) {
  if (world < 1 || world > 8 || rank < 0 || rank >= world)
    throw std::invalid_argument("bad rank/world (the reader mask holds 8 ranks)");
  std::vector<const tsv::VertList*> lists;
  std::vector<int64_t> lo, hi;
  for (int q = 0; q < world; ++q) {
    const tsv_graph::VertPart& p = vertex_part(g, q, world, st);
    lists.push_back(&p.vl);
    lo.push_back(p.slot_lo);
    hi.push_back(p.slot_hi);
  }
  auto& me = const_cast<tsv_graph::VertPart&>(vertex_part(g, rank, world, st));
  std::lock_guard<std::mutex> lk(g->vl_mu);
  if (!me.xlists) {
    auto alloc = [&](size_t bytes) -> void* {
      void* p = nullptr;
      if (!alloc_retry(&p, bytes ? bytes : 8, st))
        throw CudaError("exchange lists: out of device memory");
      me.owned.push_back(p);
      return p;
    };
    auto release = [&](void* p) {
      auto it = std::find(me.owned.begin(), me.owned.end(), p);
      if (it != me.owned.end()) me.owned.erase(it);
      cudaFreeAsync(p, st);
    };
    tsv::build_exchange_lists(g->dev, lists, lo, hi, rank, me.xl, st, alloc, release);
    me.xlists = true;
  }
  return me;
}

static int eval_vertex_level_impl(const tsv_graph* g, const tsv_shades* s, int k, int level,
                                  int32_t max_ts, const tsv_config* cfg, int32_t anchor_source,
                                  int rank, int world, const uint64_t* d_prev, uint64_t* d_cur,
                                  uint64_t* d_acc, uint64_t* const* peer_cur, void* stream) {
  return guard([&] {
    if (!g || !s || !d_acc) throw std::invalid_argument("null argument");
    check_config(cfg);
    if (!tsv::vertex_engine_supports(k) || level < 2 || level > k)
      throw std::invalid_argument("vertex-partitioned level: k must be 2..5, level 2..k");
    if (max_ts < 1 || max_ts > g->host.t) throw std::invalid_argument("max_ts outside [1..t]");
    if (s->n != g->dev.n || s->k != k || s->device != g->device)
      throw std::invalid_argument("shade assignment built for a different graph");
    if (g->model != 0) throw std::invalid_argument("vertex-partitioned level: instant model only");
    DeviceGuard dg(g->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const tsv_graph::VertPart& vp = vertex_part(g, rank, world, st);
    if (!vp.applicable) throw std::invalid_argument("vertex partition not applicable (hub vertices)");
    // v_{u,d} table and det(W) of this seed (cached with the shades)
    uint64_t* zj = nullptr;
    uint64_t det = 1;
    {
      std::lock_guard<std::mutex> lk(s->zj_mu);
      for (auto& z : s->zjs)
        if (z.seed == cfg->seed) zj = z.d, det = z.det;
      if (!zj) {
        TSV_CUDA(cudaMalloc(&zj, static_cast<size_t>(std::max<int32_t>(g->dev.n, 1)) * k * 8));
        tsv::launch_zj_ident(g->dev.n, k, cfg->seed, s->off, s->shades, zj, st);
        std::vector<uint64_t> W(static_cast<size_t>(k) * k);
        const uint64_t pre = tsv::draw_prefix(cfg->seed, tsv::kRoleShadeW);
        for (int d = 0; d < k; ++d)
          for (int j = 0; j < k; ++j)
            W[static_cast<size_t>(d) * k + j] = tsv::draw_nonzero_from(pre, d + 1, j + 1, 0);
        det = tsv::gf_det_host(W.data(), k);
        TSV_CUDA(cudaStreamSynchronize(st));
        if (s->zjs.size() >= 4) {
          cudaFree(s->zjs.front().d);
          s->zjs.erase(s->zjs.begin());
        }
        s->zjs.push_back({cfg->seed, zj, det});
      }
    }
    tsv::CoefParams cp;
    cp.g = g->dev;
    cp.zj = zj;
    cp.k = k;
    cp.ell = level;
    cp.last = level == k;
    cp.seed = cfg->seed;
    cp.anchor_source = anchor_source;
    cp.s_prev = d_prev;
    cp.ubuf = d_cur;
    cp.max_ts = max_ts;
    // (with transition times an arc can land past t: always test then)
      cp.below_t = max_ts < g->host.t || g->model != 0;
    tsv::VertPeers peers;
    if (peer_cur && world > 1 && level < k) {
      // the reader byte of every slot comes with the exchange lists
      const tsv_graph::VertPart& me = exchange_part(g, rank, world, st);
      peers.reader_mask = me.xl.reader_mask;
      peers.rank = rank;
      for (int q = 0; q < world; ++q) peers.peer[q] = q == rank ? nullptr : peer_cur[q];
    }
    tsv::launch_coef_vertex(cp, vp.vl, det, d_acc, st, peers.reader_mask ? &peers : nullptr);
    TSV_CUDA(cudaGetLastError());
  });
}

int tsv_eval_vertex_level(const tsv_graph* g, const tsv_shades* s, int k, int level,
                          int32_t max_ts, const tsv_config* cfg, int32_t anchor_source,
                          int rank, int world, const uint64_t* d_prev, uint64_t* d_cur,
                          uint64_t* d_acc, void* stream) {
  return eval_vertex_level_impl(g, s, k, level, max_ts, cfg, anchor_source, rank, world, d_prev,
                                d_cur, d_acc, nullptr, stream);
}

int tsv_eval_vertex_level_peer(const tsv_graph* g, const tsv_shades* s, int k, int level,
                               int32_t max_ts, const tsv_config* cfg, int32_t anchor_source,
                               int rank, int world, const uint64_t* d_prev, uint64_t* d_cur,
                               uint64_t* d_acc, uint64_t* const* peer_cur, void* stream) {
  if (!peer_cur) {
    g_error = "null argument";
    return TSV_ERR_INVALID;
  }
  if (world > 8) {
    g_error = "peer stores take at most 8 ranks";
    return TSV_ERR_INVALID;
  }
  return eval_vertex_level_impl(g, s, k, level, max_ts, cfg, anchor_source, rank, world, d_prev,
                                d_cur, d_acc, peer_cur, stream);
}


int tsv_vertex_exchange_plan(const tsv_graph* g, const tsv_shades* s, int k, int rank,
                             int world, tsv_exchange* out) {
  return guard([&] {
    if (!g || !s || !out) throw std::invalid_argument("null argument");
    (void)k;
    std::memset(out, 0, sizeof(*out));
    DeviceGuard dg(g->device);
    cudaStream_t st = nullptr;
    TSV_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    struct Del {
      cudaStream_t s;
      ~Del() {
        cudaStreamSynchronize(s);
        cudaStreamDestroy(s);
      }
    } del{st};
    const tsv_graph::VertPart& me = exchange_part(g, rank, world, st);
    for (int q = 0; q < world; ++q) {
      out->send_rows[q] = me.xl.send_count[q];
      out->recv_rows[q] = me.xl.recv_count[q];
    }
    out->send_total = me.xl.send_total;
    out->recv_total = me.xl.recv_total;
  });
}

static int exchange_move(const tsv_graph* g, int rank, int world, int row_words,
                         const uint64_t* src, uint64_t* dst, void* stream, bool pack) {
  return guard([&] {
    if (!g || !src || !dst) throw std::invalid_argument("null argument");
    DeviceGuard dg(g->device);
    const tsv_graph::VertPart* me = nullptr;
    {
      std::lock_guard<std::mutex> lk(g->vl_mu);
      for (auto& vp : g->parts)
        if (vp->rank == rank && vp->world == world) me = vp.get();
    }
    if (!me || !me->xlists) throw std::invalid_argument("call tsv_vertex_exchange_plan first");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (pack)
      tsv::launch_rows_pack(me->xl.send_slots, me->xl.send_total, row_words, src, dst, st);
    else
      tsv::launch_rows_unpack(me->xl.recv_slots, me->xl.recv_total, row_words, src, dst, st);
    TSV_CUDA(cudaGetLastError());
  });
}

int tsv_vertex_exchange_pack(const tsv_graph* g, int rank, int world, int row_words,
                             const uint64_t* d_rows, uint64_t* d_sendbuf, void* stream) {
  return exchange_move(g, rank, world, row_words, d_rows, d_sendbuf, stream, true);
}

int tsv_vertex_exchange_unpack(const tsv_graph* g, int rank, int world, int row_words,
                               const uint64_t* d_recvbuf, uint64_t* d_rows, void* stream) {
  return exchange_move(g, rank, world, row_words, d_recvbuf, d_rows, stream, false);
}

int64_t tsv_nonzero_index(const uint64_t* acc, int64_t n, int32_t* idx) {
  if (n <= 0 || !acc || !idx) return 0;
  const int64_t block = int64_t{1} << 16;
  const int64_t nb = (n + block - 1) / block;
  std::vector<int64_t> cnt(static_cast<size_t>(nb) + 1, 0);
#pragma omp parallel for schedule(static) if (n > (1 << 20))
  for (int64_t b = 0; b < nb; ++b) {
    int64_t c = 0;
    for (int64_t x = b * block; x < std::min(n, (b + 1) * block); ++x) c += acc[x] != 0;
    cnt[static_cast<size_t>(b) + 1] = c;
  }
  for (int64_t b = 0; b < nb; ++b) cnt[b + 1] += cnt[b];
#pragma omp parallel for schedule(static) if (n > (1 << 20))
  for (int64_t b = 0; b < nb; ++b) {
    int64_t w = cnt[b];
    for (int64_t x = b * block; x < std::min(n, (b + 1) * block); ++x)
      if (acc[x]) idx[w++] = static_cast<int32_t>(x);
  }
  return cnt[nb];
}

int tsv_finalize_device(uint64_t* d_acc, int64_t n, int32_t anchor_sink, void* stream,
                        tsv_outcome* out) {
  return guard([&] {
    if ((!d_acc && n > 0) || !out || n < 0) throw std::invalid_argument("null argument");
    uint64_t cs = 0;
    int64_t f = 0;
    tsv::device_finalize(d_acc, n, anchor_sink, static_cast<cudaStream_t>(stream), &cs, &f);
    out->flagged = f;
    out->global_nonzero = f > 0;
    out->checksum = cs;
  });
}

namespace {

// The canonical edges on the graph's device: the resident copy of a device
// build, else a staged copy of the host-held list.
struct DeviceEdges {
  const int32_t *u = nullptr, *v = nullptr, *ts = nullptr;
  std::vector<int32_t> host_ts;  // canonical timestamps on the host
  std::unique_ptr<DevBuf> bu, bv, bt;
  DeviceEdges(const tsv_graph* g, cudaStream_t st) {
    const int64_t m = g->m;
    if (g->d_eu || g->edges_in_layout) {
      if (g->d_eu) {
        u = g->d_eu;
        v = g->d_ev;
        ts = g->d_ets;
      } else {  // rebuilt from the layout
        bu = std::make_unique<DevBuf>(std::max<int64_t>(m, 1) * 4, st);
        bv = std::make_unique<DevBuf>(std::max<int64_t>(m, 1) * 4, st);
        bt = std::make_unique<DevBuf>(std::max<int64_t>(m, 1) * 4, st);
        tsv::edges_from_layout(g->dev, g->host.directed, bu->as<int32_t>(), bv->as<int32_t>(),
                               bt->as<int32_t>(), st);
        u = bu->as<int32_t>();
        v = bv->as<int32_t>();
        ts = bt->as<int32_t>();
      }
      host_ts.resize(static_cast<size_t>(m));
      if (m) TSV_CUDA(cudaMemcpyAsync(host_ts.data(), ts, m * 4, cudaMemcpyDeviceToHost, st));
      TSV_CUDA(cudaStreamSynchronize(st));
    } else {
      bu = std::make_unique<DevBuf>(std::max<int64_t>(m, 1) * 4, st);
      bv = std::make_unique<DevBuf>(std::max<int64_t>(m, 1) * 4, st);
      bt = std::make_unique<DevBuf>(std::max<int64_t>(m, 1) * 4, st);
      if (m) {
        TSV_CUDA(cudaMemcpyAsync(bu->p, g->host.eu.data(), m * 4, cudaMemcpyHostToDevice, st));
        TSV_CUDA(cudaMemcpyAsync(bv->p, g->host.ev.data(), m * 4, cudaMemcpyHostToDevice, st));
        TSV_CUDA(cudaMemcpyAsync(bt->p, g->host.ets.data(), m * 4, cudaMemcpyHostToDevice, st));
      }
      u = bu->as<int32_t>();
      v = bv->as<int32_t>();
      ts = bt->as<int32_t>();
      host_ts = g->host.ets;
    }
  }
};

struct StreamGuard {
  cudaStream_t st = nullptr;
  StreamGuard() { TSV_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking)); }
  ~StreamGuard() {
    cudaStreamSynchronize(st);
    cudaStreamDestroy(st);
  }
};

}  // namespace

int tsv_graph_static_edges(const tsv_graph* g, int64_t* ms, int32_t* a, int32_t* b,
                           int32_t* back_off, int32_t* back) {
  return guard([&] {
    if (!g || !ms || !a || !b || !back_off || !back) throw std::invalid_argument("null argument");
    if (g->model != 0)
      throw std::invalid_argument("static projection of an edge-model graph: use the instant one");
    DeviceGuard dg(g->device);
    StreamGuard sg;
    cudaStream_t st = sg.st;
    const int64_t m = g->m;
    std::vector<void*> live;
    auto alloc = [&](size_t bytes) -> void* {
      void* p = nullptr;
      if (!alloc_retry(&p, bytes ? bytes : 8, st))
        throw CudaError("static projection: out of device memory");
      live.push_back(p);
      return p;
    };
    auto release = [&](void* p) {
      auto it = std::find(live.begin(), live.end(), p);
      if (it != live.end()) live.erase(it);
      cudaFreeAsync(p, st);
    };
    try {
      const int32_t *eu = g->d_eu, *ev = g->d_ev;
      if (!eu) {
        auto* x = static_cast<int32_t*>(alloc(static_cast<size_t>(m) * 4 + 4));
        auto* y = static_cast<int32_t*>(alloc(static_cast<size_t>(m) * 4 + 4));
        auto* z = static_cast<int32_t*>(alloc(static_cast<size_t>(m) * 4 + 4));
        if (g->edges_in_layout) {
          tsv::edges_from_layout(g->dev, g->host.directed, x, y, z, st);
        } else if (m) {
          TSV_CUDA(cudaMemcpyAsync(x, g->host.eu.data(), m * 4, cudaMemcpyHostToDevice, st));
          TSV_CUDA(cudaMemcpyAsync(y, g->host.ev.data(), m * 4, cudaMemcpyHostToDevice, st));
        }
        release(z);
        eu = x;
        ev = y;
      }
      auto* da = static_cast<int32_t*>(alloc(static_cast<size_t>(m) * 4 + 4));
      auto* db = static_cast<int32_t*>(alloc(static_cast<size_t>(m) * 4 + 4));
      auto* doff = static_cast<int32_t*>(alloc(static_cast<size_t>(m) * 4 + 8));
      auto* dback = static_cast<int32_t*>(alloc(static_cast<size_t>(m) * 4 + 4));
      const int64_t s = tsv::static_projection(eu, ev, m, g->host.n, g->host.directed, da, db,
                                               doff, dback, st, alloc, release);
      copy_to_host(a, da, static_cast<size_t>(s) * 4, st);
      copy_to_host(b, db, static_cast<size_t>(s) * 4, st);
      copy_to_host(back_off, doff, static_cast<size_t>(s + 1) * 4, st);
      copy_to_host(back, dback, static_cast<size_t>(m) * 4, st);
      *ms = s;
    } catch (...) {
      for (void* p : live) cudaFreeAsync(p, st);
      throw;
    }
    for (void* p : live) cudaFreeAsync(p, st);
  });
}


int tsv_eval_edge_constrained(const tsv_graph* g, int k, const int32_t* times,
                              const int32_t* vertex_off, const int32_t* vertex_shades,
                              const tsv_config* cfg, uint64_t* accumulators, tsv_outcome* out) {
  tsv_shades* sh = nullptr;
  int rc = guard([&] {
    if (!g || !accumulators || !out || (k > 1 && !times))
      throw std::invalid_argument("null argument");
    check_config(cfg);
    if (k < 2 || k > 30) throw std::invalid_argument("k out of range [2,30]");
    for (int i = 0; i + 1 < k; ++i) {
      if (times[i] < 1 || times[i] > g->host.t)
        throw std::invalid_argument("prescribed timestamp outside [1..t]");
      if (i > 0 && times[i] <= times[i - 1])
        throw std::invalid_argument("prescribed timestamps must strictly increase");
    }
    if (cfg->edge_model != 0)
      throw std::invalid_argument("the edge-constrained sieve uses the instant model");
  });
  if (rc) return rc;
  rc = tsv_shades_upload(g, k, vertex_off, vertex_shades, &sh);
  if (rc) return rc;
  rc = guard([&] {
    DeviceGuard dg(g->device);
    const int32_t n = g->host.n;
    StreamGuard sg;
    cudaStream_t st = sg.st;
    DeviceEdges E(g, st);
    const uint64_t P = 1ull << k;
    // batch width: the n x W state pair plus the z table must fit
    size_t free_b = 0, total_b = 0;
    TSV_CUDA(cudaMemGetInfo(&free_b, &total_b));
    int W = static_cast<int>(std::min<uint64_t>(P, 128));
    auto ec_words = [&](int w) {
      return 3ull * n * w + static_cast<uint64_t>(n) * k + n;
    };
    while (W > 1 && (3ull * n * W * 8 > free_b * 0.8 || ec_words(W) > cfg->memory_cap_words))
      W >>= 1;
    if (ec_words(W) > cfg->memory_cap_words)  // (sieve.cpp:161-166's convention)
      throw CapError("sieve memory cap exceeded: needs " + std::to_string(ec_words(W)) +
                     " field words, cap " + std::to_string(cfg->memory_cap_words));
    DevBuf d_w(static_cast<size_t>(k) * k * 8, st), d_zj(static_cast<size_t>(n) * k * 8 + 8, st),
        acc(static_cast<size_t>(n) * 8 + 8, st), zb(static_cast<size_t>(n) * W * 8 + 8, st),
        s0(static_cast<size_t>(n) * W * 8 + 8, st), s1(static_cast<size_t>(n) * W * 8 + 8, st);
    tsv::launch_wtab(k, cfg->seed, d_w.as<uint64_t>(), st);
    tsv::launch_zj(n, k, cfg->seed, sh->off, sh->shades, d_w.as<uint64_t>(),
                   d_zj.as<uint64_t>(), st);
    TSV_CUDA(cudaMemsetAsync(acc.p, 0, static_cast<size_t>(n) * 8 + 8, st));
    // edge range of each prescribed timestamp (edges are sorted by ts)
    std::vector<std::pair<int64_t, int64_t>> range(static_cast<size_t>(k - 1));
    for (int i = 0; i + 1 < k; ++i) {
      auto lo = std::lower_bound(E.host_ts.begin(), E.host_ts.end(), times[i]);
      auto hi = std::upper_bound(E.host_ts.begin(), E.host_ts.end(), times[i]);
      range[i] = {lo - E.host_ts.begin(), hi - E.host_ts.begin()};
    }
    for (uint64_t pb = 0; pb < P; pb += W) {
      tsv::Batch b = batch_shape(W);
      b.pb = pb;
      b.pe = std::min(P, pb + static_cast<uint64_t>(W));
      tsv::launch_zbatch(n, d_zj.as<uint64_t>(), k, b, zb.as<uint64_t>(), st);
      const uint64_t* prev = zb.as<uint64_t>();
      uint64_t* bufs[2] = {s0.as<uint64_t>(), s1.as<uint64_t>()};
      for (int ell = 2; ell <= k; ++ell) {
        uint64_t* cur = bufs[ell & 1];
        TSV_CUDA(cudaMemsetAsync(cur, 0, static_cast<size_t>(n) * W * 8, st));
        tsv::launch_ec_level(range[ell - 2].first, range[ell - 2].second, g->host.directed,
                             E.u, E.v, zb.as<uint64_t>(), W, cfg->seed, ell, prev, cur, st);
        prev = cur;
      }
      tsv::launch_row_xor(n, W, prev, acc.as<uint64_t>(), st);
    }
    TSV_CUDA(cudaGetLastError());
    if (n)
      TSV_CUDA(cudaMemcpyAsync(accumulators, acc.p, static_cast<size_t>(n) * 8,
                               cudaMemcpyDeviceToHost, st));
    TSV_CUDA(cudaStreamSynchronize(st));
    finalize_host(n, accumulators, -1, k, out);
    out->peak_field_words = ec_words(W);
  });
  tsv_shades_free(sh);
  return rc;
}

int tsv_eval_vertex_ordered(const tsv_graph* g, int k, const int32_t* order,
                            const int32_t* colors, int32_t wildcard_color, int32_t max_ts,
                            const tsv_config* cfg, uint64_t* accumulators, tsv_outcome* out) {
  return guard([&] {
    if (!g || !order || !accumulators || !out || (g->host.n > 0 && !colors))
      throw std::invalid_argument("null argument");
    check_config(cfg);
    if (k < 1 || k > 30) throw std::invalid_argument("k out of range [1,30]");
    if (max_ts < 1 || max_ts > g->host.t) throw std::invalid_argument("max_ts outside [1..t]");
    DeviceGuard dg(g->device);
    const int32_t n = g->host.n;
    StreamGuard sg;
    cudaStream_t st = sg.st;
    VcSpec vc;
    DevBuf dcol(static_cast<size_t>(n) * 4 + 4, st), acc(static_cast<size_t>(n) * 8 + 8, st);
    if (n) TSV_CUDA(cudaMemcpyAsync(dcol.p, colors, static_cast<size_t>(n) * 4,
                                    cudaMemcpyHostToDevice, st));
    TSV_CUDA(cudaMemsetAsync(acc.p, 0, static_cast<size_t>(n) * 8 + 8, st));
    vc.d_colors = dcol.as<int32_t>();
    vc.order.assign(order, order + k);
    vc.wild = wildcard_color;
    uint64_t peak = 0;
    eval_device(g, nullptr, k, max_ts, cfg, -1, 0, 1ull << k, acc.as<uint64_t>(), st, &peak,
                &vc);
    if (n)
      TSV_CUDA(cudaMemcpyAsync(accumulators, acc.p, static_cast<size_t>(n) * 8,
                               cudaMemcpyDeviceToHost, st));
    TSV_CUDA(cudaStreamSynchronize(st));
    finalize_host(n, accumulators, -1, k, out);
    out->peak_field_words = peak;
  });
}

int tsv_vc_colorful_dp(const tsv_graph* g, int k, const int32_t* order, const int32_t* colors,
                       int32_t wildcard_color, int32_t max_ts, uint8_t* flagged) {
  return guard([&] {
    if (!g || !order || !flagged || (g->host.n > 0 && !colors))
      throw std::invalid_argument("null argument");
    if (k < 1) throw std::invalid_argument("k must be positive");
    DeviceGuard dg(g->device);
    const int32_t n = g->host.n;
    StreamGuard sg;
    cudaStream_t st = sg.st;
    DeviceEdges E(g, st);
    constexpr int32_t kInf = INT32_MAX;
    std::vector<int32_t> e1(static_cast<size_t>(n));
    for (int32_t u = 0; u < n; ++u)
      e1[u] = (colors[u] == order[0] || order[0] == wildcard_color) ? 0 : kInf;
    DevBuf dcol(static_cast<size_t>(n) * 4 + 4, st), a(static_cast<size_t>(n) * 4 + 4, st),
        b(static_cast<size_t>(n) * 4 + 4, st);
    if (n) {
      TSV_CUDA(cudaMemcpyAsync(dcol.p, colors, static_cast<size_t>(n) * 4,
                               cudaMemcpyHostToDevice, st));
      TSV_CUDA(cudaMemcpyAsync(a.p, e1.data(), static_cast<size_t>(n) * 4,
                               cudaMemcpyHostToDevice, st));
    }
    int32_t* prev = a.as<int32_t>();
    int32_t* cur = b.as<int32_t>();
    for (int ell = 2; ell <= k; ++ell) {
      // fill with "unreached"
      std::vector<int32_t> inf(static_cast<size_t>(n), kInf);
      if (n) TSV_CUDA(cudaMemcpyAsync(cur, inf.data(), static_cast<size_t>(n) * 4,
                                      cudaMemcpyHostToDevice, st));
      TSV_CUDA(cudaStreamSynchronize(st));
      tsv::launch_vc_dp_level(g->m, g->host.directed, E.u, E.v, E.ts, max_ts,
                              dcol.as<int32_t>(), order[ell - 2], order[ell - 1],
                              wildcard_color, prev, cur, st);
      std::swap(prev, cur);
    }
    std::vector<int32_t> e(static_cast<size_t>(n));
    if (n) TSV_CUDA(cudaMemcpyAsync(e.data(), prev, static_cast<size_t>(n) * 4,
                                    cudaMemcpyDeviceToHost, st));
    TSV_CUDA(cudaStreamSynchronize(st));
    TSV_CUDA(cudaGetLastError());
    for (int32_t u = 0; u < n; ++u)
      flagged[u] = (e[u] != kInf && e[u] <= static_cast<int64_t>(max_ts) + 1) ? 1 : 0;
  });
}

int tsv_eval_static_projection(int32_t n, int64_t ms, const int32_t* a, const int32_t* b,
                               int directed, int junction, int k, const int32_t* vertex_off,
                               const int32_t* vertex_shades, const tsv_config* cfg, int device,
                               uint64_t* accumulators, tsv_outcome* out) {
  return guard([&] {
    if (!accumulators || !out || !vertex_off) throw std::invalid_argument("null argument");
    check_config(cfg, true);
    if (k < 1 || k > 30) throw std::invalid_argument("k out of range [1,30]");
    if (n < 0 || ms < 0) throw std::invalid_argument("negative size");
    // head-sorted arc lists of the projection: in-arcs (tail -> head) and
    // out-arcs (head = the walk's current vertex, tail = the next one)
    // head-grouped arc lists (counting sort on all host threads; the order
    // within a head is free: both engines XOR a head's arcs, so the placement
    // races only over positions inside the head's range)
    auto arcs = [&](bool incoming, std::vector<int32_t>& head, std::vector<int32_t>& tail,
                    std::vector<int32_t>& edge, std::vector<int64_t>* head_off = nullptr) {
      const int64_t A = directed ? ms : 2 * ms;
      std::vector<int64_t> off(static_cast<size_t>(n) + 1, 0);
      int64_t bad = 0;
#pragma omp parallel for schedule(static) reduction(+ : bad) if (ms > (1 << 20))
      for (int64_t i = 0; i < ms; ++i) {
        if (a[i] < 0 || a[i] >= n || b[i] < 0 || b[i] >= n) {
          ++bad;
          continue;
        }
        __atomic_fetch_add(&off[(incoming ? b[i] : a[i]) + 1], 1, __ATOMIC_RELAXED);
        if (!directed) __atomic_fetch_add(&off[(incoming ? a[i] : b[i]) + 1], 1, __ATOMIC_RELAXED);
      }
      if (bad) throw std::invalid_argument("edge endpoint out of range");
      for (int32_t x = 0; x < n; ++x) off[x + 1] += off[x];
      if (head_off) *head_off = off;
      head.resize(static_cast<size_t>(A));
      tail.resize(static_cast<size_t>(A));
      edge.resize(static_cast<size_t>(A));
      auto put = [&](int32_t h, int32_t t, int64_t e) {
        const int64_t p = __atomic_fetch_add(&off[h], 1, __ATOMIC_RELAXED);
        head[p] = h;
        tail[p] = t;
        edge[p] = static_cast<int32_t>(e);
      };
#pragma omp parallel for schedule(static) if (ms > (1 << 20))
      for (int64_t i = 0; i < ms; ++i) {
        if (incoming) put(b[i], a[i], i); else put(a[i], b[i], i);
        if (!directed) { if (incoming) put(a[i], b[i], i); else put(b[i], a[i], i); }
      }
    };
    DeviceGuard dg(device);
    cudaStream_t st = nullptr;
    TSV_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    struct StreamGuard {
      cudaStream_t s;
      ~StreamGuard() {
        cudaStreamSynchronize(s);
        cudaStreamDestroy(s);
      }
    } sg{st};
    const uint64_t P = 1ull << k;
    const int ppt = P >= 64 ? 2 : 1;
    const int W = 32 * ppt;
    const uint64_t layers = junction ? static_cast<uint64_t>(k) + 2 : 2;
    const uint64_t words = layers * static_cast<uint64_t>(n) * W +
                           static_cast<uint64_t>(n) * (static_cast<uint64_t>(k) + 1);
    if (words > cfg->memory_cap_words)
      throw CapError("sieve memory cap exceeded: needs " + std::to_string(words) +
                     " field words, cap " + std::to_string(cfg->memory_cap_words));

    std::vector<int32_t> ih, it, ie, oh, ot, oe;
    // coefficient form (coef_static.cu): GF(2^64), k <= 12, when its rows fit
    const char* se = std::getenv("TSV_STATIC_ENGINE");
    const uint64_t cwords = tsv::static_coef_words(n, k, junction != 0);
    if (cfg->field_bits == 64 && tsv::static_coef_supported(k) &&
        !(se && std::strcmp(se, "points") == 0) && cwords <= cfg->memory_cap_words &&
        fits_device(cwords)) {
      const char* tre = std::getenv("TSV_TRACE_API");
      const bool trace = tre && tre[0] == '1';
      const auto t0 = std::chrono::steady_clock::now();
      auto mark = [&](const char* what) {
        if (!trace) return;
        cudaStreamSynchronize(st);
        std::fprintf(stderr, "[static] %-26s %9.1f ms\n", what,
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() -
                                                               t0).count());
      };
      std::vector<int64_t> ioff, ooff;
      arcs(true, ih, it, ie, &ioff);
      if (junction) arcs(false, oh, ot, oe, &ooff);
      mark("host arc lists");
      std::vector<int32_t> off(vertex_off, vertex_off + n + 1);
      std::vector<int32_t> shv(vertex_shades, vertex_shades + vertex_off[n]);
      for (int32_t s : shv)
        if (s < 1 || s > k) throw std::invalid_argument("shade id outside [1..k]");
      std::vector<void*> live;
      auto alloc = [&](size_t bytes) -> void* {
        void* p = nullptr;
        if (!alloc_retry(&p, bytes ? bytes : 8, st))
          throw CudaError("static sieve: out of device memory");
        live.push_back(p);
        return p;
      };
      auto release = [&](void* p) {
        auto itp = std::find(live.begin(), live.end(), p);
        if (itp != live.end()) live.erase(itp);
        cudaFreeAsync(p, st);
      };
      auto upv = [&](const auto& v) {
        using Tv = typename std::decay_t<decltype(v)>::value_type;
        void* d = alloc(std::max<size_t>(v.size(), 1) * sizeof(Tv));
        if (!v.empty())
          TSV_CUDA(cudaMemcpyAsync(d, v.data(), v.size() * sizeof(Tv), cudaMemcpyHostToDevice, st));
        return d;
      };
      try {
        tsv::StaticCoefInputs ci;
        ci.n = n;
        ci.k = k;
        ci.junction = junction != 0;
        ci.seed = cfg->seed;
        ci.in_off = static_cast<const int64_t*>(upv(ioff));
        ci.h_in_off = &ioff;
        ci.h_out_off = &ooff;
        ci.in_tail = static_cast<const int32_t*>(upv(it));
        ci.in_edge = static_cast<const int32_t*>(upv(ie));
        if (junction) {
          ci.out_off = static_cast<const int64_t*>(upv(ooff));
          ci.out_tail = static_cast<const int32_t*>(upv(ot));
          ci.out_edge = static_cast<const int32_t*>(upv(oe));
        }
        auto* d_off = static_cast<int32_t*>(upv(off));
        auto* d_sh = static_cast<int32_t*>(upv(shv));
        auto* zj = static_cast<uint64_t*>(alloc(static_cast<size_t>(n) * k * 8 + 8));
        tsv::launch_zj_ident(n, k, cfg->seed, d_off, d_sh, zj, st);
        std::vector<uint64_t> Wm(static_cast<size_t>(k) * k);
        const uint64_t pre = tsv::draw_prefix(cfg->seed, tsv::kRoleShadeW);
        for (int d = 0; d < k; ++d)
          for (int j = 0; j < k; ++j)
            Wm[static_cast<size_t>(d) * k + j] = tsv::draw_nonzero_from(pre, d + 1, j + 1, 0);
        ci.det = tsv::gf_det_host(Wm.data(), k);
        ci.zj = zj;
        auto* acc = static_cast<uint64_t*>(alloc(static_cast<size_t>(n) * 8 + 8));
        TSV_CUDA(cudaMemsetAsync(acc, 0, static_cast<size_t>(n) * 8 + 8, st));
        ci.acc = acc;
        ci.tables = &coef_const_tables(k);
        mark("uploads, shade table");
        tsv::eval_static_coef(ci, st, alloc, release);
        mark("coefficient sieve");
        TSV_CUDA(cudaGetLastError());
        if (n)
          TSV_CUDA(cudaMemcpyAsync(accumulators, acc, static_cast<size_t>(n) * 8,
                                   cudaMemcpyDeviceToHost, st));
        TSV_CUDA(cudaStreamSynchronize(st));
      } catch (...) {
        for (void* p : live) cudaFreeAsync(p, st);
        throw;
      }
      for (void* p : live) cudaFreeAsync(p, st);
      *out = tsv_outcome{};
      finalize_host(n, accumulators, -1, k, out);
      out->peak_field_words = cwords;
      return;
    }
    arcs(true, ih, it, ie);
    if (junction) arcs(false, oh, ot, oe);
    // chunks sized to give every SM several warps (a 256-arc chunk left the
    // C2 projection with 191 blocks, 16% of the warp slots busy)
    auto chunks = [](int64_t A) {
      std::vector<int64_t> c;
      const int64_t ch = std::min<int64_t>(256, std::max<int64_t>(32, A / (148 * 64)));
      for (int64_t s = 0; s < A; s += ch) c.push_back(s);
      c.push_back(A);
      return c;
    };
    const std::vector<int64_t> ic = chunks(static_cast<int64_t>(ih.size()));
    const std::vector<int64_t> oc = chunks(static_cast<int64_t>(oh.size()));
    auto up = [&](const auto& v) {
      using T = typename std::decay_t<decltype(v)>::value_type;
      auto* buf = new DevBuf(std::max<size_t>(v.size(), 1) * sizeof(T), st);
      if (!v.empty())
        TSV_CUDA(cudaMemcpyAsync(buf->p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, st));
      return std::unique_ptr<DevBuf>(buf);
    };
    auto d_ih = up(ih), d_it = up(it), d_ie = up(ie), d_ic = up(ic);
    auto d_oh = up(oh), d_ot = up(ot), d_oe = up(oe), d_oc = up(oc);
    std::vector<int32_t> off(vertex_off, vertex_off + n + 1);
    std::vector<int32_t> shv(vertex_shades, vertex_shades + vertex_off[n]);
    for (int32_t s : shv)
      if (s < 1 || s > k) throw std::invalid_argument("shade id outside [1..k]");
    auto d_off = up(off), d_sh = up(shv);
    std::vector<uint64_t> wtab(static_cast<size_t>(k) * k);
    for (int d = 1; d <= k; ++d)
      for (int j = 1; j <= k; ++j)
        wtab[(d - 1) * k + (j - 1)] = tsv::draw_nonzero(cfg->seed, tsv::kRoleShadeW, d, j, 0);
    auto d_w = up(wtab);
    DevBuf zj(static_cast<size_t>(n) * k * 8, st), acc(static_cast<size_t>(n) * 8, st);
    if (cfg->field_bits == 64)
      tsv::launch_zj(n, k, cfg->seed, d_off->as<int32_t>(), d_sh->as<int32_t>(),
                     d_w->as<uint64_t>(), zj.as<uint64_t>(), st);
    else
      tsv::launch_small_zj64(cfg->field_bits, n, k, cfg->seed, d_off->as<int32_t>(),
                             d_sh->as<int32_t>(), zj.as<uint64_t>(), st);
    TSV_CUDA(cudaMemsetAsync(acc.p, 0, static_cast<size_t>(n) * 8, st));
    const size_t layer = static_cast<size_t>(n) * W;
    std::vector<std::unique_ptr<DevBuf>> ending;
    // (the static sieve ping-pongs E(l) over entries 1 and 2: at least 3, k = 1 too)
    for (uint64_t i = 0; i <= std::max<uint64_t>(static_cast<uint64_t>(k), 2); ++i)
      ending.emplace_back(new DevBuf((junction || i <= 2 ? layer : 1) * 8, st));
    DevBuf s0(layer * 8, st), s1(layer * 8, st);

    tsv::StaticLevel in;
    in.C = static_cast<int64_t>(ic.size()) - 1;
    in.chunk_arc = d_ic->as<int64_t>();
    in.arc_head = d_ih->as<int32_t>();
    in.arc_tail = d_it->as<int32_t>();
    in.arc_edge = d_ie->as<int32_t>();
    in.zj = zj.as<uint64_t>();
    in.k = k;
    in.seed = cfg->seed;
    in.role = tsv::kRoleEdgeY;
    in.head_times_z = true;
    in.ppt = ppt;
    in.bits = cfg->field_bits;
    tsv::StaticLevel outl = in;
    outl.C = static_cast<int64_t>(oc.size()) - 1;
    outl.chunk_arc = d_oc->as<int64_t>();
    outl.arc_head = d_oh->as<int32_t>();
    outl.arc_tail = d_ot->as<int32_t>();
    outl.arc_edge = d_oe->as<int32_t>();
    outl.role = 4;  // edge_y2
    outl.head_times_z = false;
    outl.tail_times_z = true;

    for (uint64_t pb = 0; pb < P; pb += W) {
      const uint64_t pe = std::min(P, pb + W);
      in.pb = outl.pb = pb;
      in.pe = outl.pe = pe;
      // walks-ending family E_1..E_k (static: only the last two layers kept)
      auto E = [&](int l) -> uint64_t* {
        return ending[junction ? l : (l % 2) + 1]->as<uint64_t>();
      };
      tsv::launch_static_base(n, zj.as<uint64_t>(), k, pb, pe, ppt, E(1), st);
      for (int l = 2; l <= k; ++l) {
        TSV_CUDA(cudaMemsetAsync(E(l), 0, layer * 8, st));
        in.level = l - 1;
        in.src = E(l - 1);
        in.out = E(l);
        tsv::launch_static_level(in, st);
      }
      if (!junction) {
        tsv::launch_static_readout(n, E(k), nullptr, ppt, acc.as<uint64_t>(), st, cfg->field_bits);
        continue;
      }
      // walks-starting family S_1 = 1, S_b from S_{b-1}; readout E_{k+1-b} * S_b
      tsv::launch_static_readout(n, E(k), nullptr, ppt, acc.as<uint64_t>(), st, cfg->field_bits);
      uint64_t* sp = nullptr;
      uint64_t* sc = s0.as<uint64_t>();
      for (int bb = 2; bb <= k; ++bb) {
        TSV_CUDA(cudaMemsetAsync(sc, 0, layer * 8, st));
        outl.level = bb - 1;
        outl.src = sp;
        outl.out = sc;
        tsv::launch_static_level(outl, st);
        tsv::launch_static_readout(n, E(k + 1 - bb), sc, ppt, acc.as<uint64_t>(), st,
                                   cfg->field_bits);
        sp = sc;
        sc = (sc == s0.as<uint64_t>()) ? s1.as<uint64_t>() : s0.as<uint64_t>();
      }
    }
    TSV_CUDA(cudaGetLastError());
    if (n)
      TSV_CUDA(cudaMemcpyAsync(accumulators, acc.p, static_cast<size_t>(n) * 8,
                               cudaMemcpyDeviceToHost, st));
    TSV_CUDA(cudaStreamSynchronize(st));
    *out = tsv_outcome{};
    finalize_host(n, accumulators, -1, k, out);
    out->fn_bound = (2.0 * k - 1.0) / std::pow(2.0, cfg->field_bits);
    out->peak_field_words = words;
  });
}

int tsv_xor_combine_device(const uint64_t* d_parts, int nparts, int64_t n,
                           uint64_t* d_out, void* stream) {
  return guard([&] {
    if (nparts < 1 || n < 0) throw std::invalid_argument("bad combine shape");
    tsv::launch_xor_combine(d_parts, nparts, n, d_out, static_cast<cudaStream_t>(stream));
    TSV_CUDA(cudaGetLastError());
  });
}

int tsv_finalize(int32_t n, uint64_t* acc, int32_t anchor_sink, tsv_outcome* out) {
  return guard([&] {
    if (!out || (n > 0 && !acc)) throw std::invalid_argument("null argument");
    *out = tsv_outcome{};
    finalize_host(n, acc, anchor_sink, 1, out);
  });
}

int tsv_profile_enable(int on) {
  g_prof_on = on != 0;
  return TSV_OK;
}

int tsv_profile_get(const char* kernel, int64_t* launches, double* total_ms) {
  return guard([&] {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    int64_t cnt = 0;
    double ms = 0;
    for (auto& r : g_prof) {
      if (kernel && r.name != kernel) continue;
      TSV_CUDA(cudaEventSynchronize(r.b));
      float x = 0;
      TSV_CUDA(cudaEventElapsedTime(&x, r.a, r.b));
      ms += x;
      ++cnt;
    }
    if (launches) *launches = cnt;
    if (total_ms) *total_ms = ms;
  });
}

int tsv_profile_reset(void) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  for (auto& r : g_prof) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  g_prof.clear();
  g_launches.store(0);
  return TSV_OK;
}

int64_t tsv_kernel_launches(void) { return g_launches.load(); }

int tsv_gf_mul_device(int variant, int64_t n, const uint64_t* a, const uint64_t* b,
                      uint64_t* out) {
  return guard([&] {
    if (n < 0) throw std::invalid_argument("negative count");
    DevBuf da(n * 8, nullptr), db(n * 8, nullptr), dc(n * 8, nullptr);
    if (n) {
      TSV_CUDA(cudaMemcpy(da.p, a, n * 8, cudaMemcpyHostToDevice));
      TSV_CUDA(cudaMemcpy(db.p, b, n * 8, cudaMemcpyHostToDevice));
    }
    tsv::launch_gf_mul(variant, n, da.as<uint64_t>(), db.as<uint64_t>(), dc.as<uint64_t>(),
                       nullptr);
    TSV_CUDA(cudaGetLastError());
    if (n) TSV_CUDA(cudaMemcpy(out, dc.p, n * 8, cudaMemcpyDeviceToHost));
  });
}

int tsv_gf_bench(int variant, int64_t iters, double* products_per_s) {
  return guard([&] {
    int dev = 0, sms = 0;
    TSV_CUDA(cudaGetDevice(&dev));
    TSV_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int threads = 256, blocks = sms * 8;
    DevBuf sink(static_cast<size_t>(threads) * blocks * 8, nullptr);
    tsv::launch_gf_bench(variant, 16, sink.as<uint64_t>(), blocks, threads, nullptr);
    cudaEvent_t a, b;
    TSV_CUDA(cudaEventCreate(&a));
    TSV_CUDA(cudaEventCreate(&b));
    TSV_CUDA(cudaEventRecord(a));
    const double products =
        tsv::launch_gf_bench(variant, iters, sink.as<uint64_t>(), blocks, threads, nullptr);
    TSV_CUDA(cudaEventRecord(b));
    TSV_CUDA(cudaEventSynchronize(b));
    float ms = 0;
    TSV_CUDA(cudaEventElapsedTime(&ms, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    *products_per_s = products / (ms * 1e-3);
  });
}

int tsv_draw_edge_y_device(uint64_t seed, int32_t level, int64_t n, const int32_t* edges,
                           uint64_t* out) {
  return guard([&] {
    DevBuf de(n * 4, nullptr), dy(n * 8, nullptr);
    if (n) TSV_CUDA(cudaMemcpy(de.p, edges, n * 4, cudaMemcpyHostToDevice));
    tsv::launch_draw_y(seed, level, n, de.as<int32_t>(), dy.as<uint64_t>(), nullptr);
    TSV_CUDA(cudaGetLastError());
    if (n) TSV_CUDA(cudaMemcpy(out, dy.p, n * 8, cudaMemcpyDeviceToHost));
  });
}

}  // extern "C"

// coef.hpp -- the coefficient (top-degree) form of the temporal sieve
// (coef_kernels.cu; the derivation is at the top of that file).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "engine.hpp"

namespace tsv {

// One level l of the coefficient engine (kernel k_coef_arcs).
struct CoefParams {
  DevGraph g;
  const uint64_t* zj = nullptr;  // n x k: z_{u,j} = S_1[u][{j}]
  int k = 0;
  int ell = 2;                   // level being produced
  bool last = false;             // ell == k: flush vertex pieces into ulast
  uint64_t seed = 1;
  int32_t anchor_source = -1;
  int E = 0;                     // input entries C(k, ell-1) = row stride
  int e0 = 0, ne = 0;            // entry slice of this launch
  const uint64_t* s_prev = nullptr;  // S x E: S_{ell-1} (ell > 2)
  uint64_t* ubuf = nullptr;          // S x E: U at referenced run ends
  uint64_t* agg = nullptr;           // C x E: chunk tail prefixes
  uint64_t* ulast = nullptr;         // n x k: level-k vertex sums (zeroed)
  int32_t max_ts = 0;
  const uint8_t* vflag = nullptr;  // n: vertex has a nonzero S_1 row (nullptr: no skipping)
  const uint8_t* sflag = nullptr;  // S: S_{ell-1}[slot] row is nonzero (ell > 2)
  const int32_t* vc_color = nullptr;  // vertex-ordered sieve filter (as LevelParams)
  int32_t vc_head = 0, vc_tail = 0, vc_wild = -1;
};

// Lanes per arc group for an entry slice of ne entries (4, 8, 16 or 32).
int coef_group_lanes(int ne);
// Entries one k_coef_arcs launch covers at most (larger levels are sliced).
constexpr int kCoefSlice = 128;

void launch_coef_arcs(const CoefParams& p, cudaStream_t st);
void launch_coef_fixup(const CoefParams& p, cudaStream_t st);
void launch_coef_ztrans(int64_t S, int F, int l, const int32_t* slot_head, const uint64_t* zj,
                        int k, int E, const uint64_t* ubuf, const int2* pairs,
                        const int2* jpairs, uint64_t* out, uint8_t* sflag, int sm_count,
                        cudaStream_t st);
// vflag[u] = row u of the n x k table is nonzero
void launch_row_nonzero(int32_t n, int k, const uint64_t* rows, uint8_t* vflag, cudaStream_t st);
void launch_coef_readout(int32_t n, const uint64_t* zj, int k, const uint64_t* ulast,
                         const int2* pairs, uint64_t scale, uint64_t* acc, cudaStream_t st);
void launch_slot_head(int64_t R, const int32_t* run_slot, const int32_t* run_head,
                      int32_t* slot_head, cudaStream_t st);

// Host tables (colex order = increasing bit mask within a level).
struct CoefTables {
  int k = 0;
  std::vector<int64_t> count;  // count[l] = C(k, l), l = 0..k
  // pairs of level l (2..k): for output o (an l-subset T) and c < l,
  // (rank of T minus its c-th element among the (l-1)-subsets, that element)
  std::vector<std::vector<int2>> pairs;
  // jpairs of level l: for each j < k, the C(k-1, l-1) pairs (rank of an
  // (l-1)-subset T' without j, rank of T' + {j}) in increasing T' order
  std::vector<std::vector<int2>> jpairs;
};
CoefTables coef_tables(int k);

}  // namespace tsv

/*
 * tsv_oracle.c -- CPU restatement of the temporal-sieve hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * engine: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * leg may load it.  The product path (paper_2001_07158_b200) never links or
 * calls it and fails loudly when its own CUDA library is missing.
 *
 * Parity is pinned against the compiled reference (oracle/_ref, built from
 * /root/reference/proj/core/src by oracle/Makefile) and against the golden
 * vectors in tests/golden/ produced by tests/golden/make_golden.py.
 *
 * What is restated (reference = /root/reference/proj):
 *   - GF(2^64) product, modulus x^64+x^4+x^3+x+1 .... core/include/tsieve/gf.hpp:37-42,55-106
 *   - counter PRNG draw64 / draw_nonzero ............. gf.hpp:111-153
 *   - canonical edge ids, arcs, runs ................. core/src/graph.cpp:14-79
 *   - z_{u,j} constrained substitution ............... core/src/sieve.cpp:83-101
 *   - z_u^A lane fill (bit j of A <-> label j+1) ..... sieve.cpp:116-133
 *   - Eq. 3 temporal DP (instant model), anchor, k=1 . sieve.cpp:170-256,294-306
 *   - finalize / FNV-1a checksum ..................... sieve.cpp:35-49,136-159
 *
 * The DP is not the reference's dense P[l][v][t] layout: it is the O(runs)
 * event form.  A run is the set of arcs with a common
 * (timestamp, head).  For level l >= 2
 *     T_l[run] = z_head^A * XOR_{a in run} y(e_a, l-1) * Q_{l-1}(tail_a, ts-1)
 * where Q_l(v, i) is the XOR of T_l over v's runs with timestamp <= i (the
 * stay term of sieve.cpp:229-230 made explicit) and Q_1(v, .) = z_v^A.
 * The readout is acc[u] ^= XOR_A Q_k(u, max_ts) (sieve.cpp:297-303).
 * Field arithmetic is exact, so the evaluation order does not matter.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ GF */

#include "tsv_gf.h"

/* Exported entry points of the arithmetic (gf.hpp:55-153; bodies in tsv_gf.h). */
uint64_t tsvo_gf_mul(uint64_t a, uint64_t b) { return gf_mul(a, b); }
uint64_t tsvo_gf_mul_slow(uint64_t a, uint64_t b) { return gf_mul_slow(a, b); }
uint64_t tsvo_draw64(uint64_t seed, uint64_t role, uint64_t a, uint64_t b, uint64_t c) {
  return draw64(seed, role, a, b, c);
}
uint64_t tsvo_draw_nonzero(uint64_t seed, uint64_t role, uint64_t a, uint64_t b,
                           uint64_t c) {
  return draw_nonzero(seed, role, a, b, c);
}


/* --------------------------------------------------------------- graph */

typedef struct {
  int32_t u, v, ts;
} edge_t;

typedef struct {
  int32_t ts, head, tail, edge;
} rawarc_t;

static int cmp_edge(const void *pa, const void *pb) {
  const edge_t *a = pa, *b = pb;
  if (a->ts != b->ts) return a->ts < b->ts ? -1 : 1;
  if (a->u != b->u) return a->u < b->u ? -1 : 1;
  if (a->v != b->v) return a->v < b->v ? -1 : 1;
  return 0;
}

static int cmp_arc(const void *pa, const void *pb) {
  const rawarc_t *a = pa, *b = pb;
  if (a->ts != b->ts) return a->ts < b->ts ? -1 : 1;
  if (a->head != b->head) return a->head < b->head ? -1 : 1;
  if (a->tail != b->tail) return a->tail < b->tail ? -1 : 1;
  return 0;
}

/*
 * Canonicalize like TemporalGraph::build (graph.cpp:14-43): drop self loops,
 * orient undirected edges u<v, sort by (ts,u,v), drop duplicates.  The edge id
 * is the index in the result.  Writes the canonical edges into out_u/v/ts
 * (capacity m) and returns their count, or -1 on a range error.
 */
int64_t tsvo_canonical_edges(int32_t n, int64_t m, const int32_t *u,
                             const int32_t *v, const int32_t *ts,
                             int directed, int32_t *out_u, int32_t *out_v,
                             int32_t *out_ts) {
  edge_t *e = malloc(sizeof(edge_t) * (size_t)(m > 0 ? m : 1));
  int64_t k = 0;
  for (int64_t i = 0; i < m; ++i) {
    if (u[i] < 0 || u[i] >= n || v[i] < 0 || v[i] >= n || ts[i] < 1) {
      free(e);
      return -1;
    }
    if (u[i] == v[i]) continue;
    edge_t x = {u[i], v[i], ts[i]};
    if (!directed && x.u > x.v) {
      int32_t s = x.u;
      x.u = x.v;
      x.v = s;
    }
    e[k++] = x;
  }
  qsort(e, (size_t)k, sizeof(edge_t), cmp_edge);
  int64_t w = 0;
  for (int64_t i = 0; i < k; ++i)
    if (w == 0 || cmp_edge(&e[w - 1], &e[i]) != 0) e[w++] = e[i];
  for (int64_t i = 0; i < w; ++i) {
    out_u[i] = e[i].u;
    out_v[i] = e[i].v;
    out_ts[i] = e[i].ts;
  }
  free(e);
  return w;
}

/* ---------------------------------------------------------------- DP */

/*
 * Evaluate the temporal sieve for the sieve points A in [p_begin, p_end) and
 * XOR their contributions into acc[0..n) (not cleared here).  Edges must be
 * canonical (tsvo_canonical_edges).  vertex_off/vertex_shades is the shade
 * CSR of ShadeAssignment (sieve.hpp:39-56); shades are 1-based.
 * anchor_source < 0 disables the anchor.  The sink restriction is applied by
 * tsvo_finalize.
 */
int tsvo_eval_points(int32_t n, int64_t m, const int32_t *eu,
                     const int32_t *ev, const int32_t *ets, int directed,
                     int k, int32_t max_ts, const int32_t *vertex_off,
                     const int32_t *vertex_shades, uint64_t seed,
                     int32_t anchor_source, uint64_t p_begin, uint64_t p_end,
                     uint64_t *acc) {
  if (k < 1 || k > 30) return -1;
  /* z_{u,j} (sieve.cpp:83-101) */
  uint64_t *zj = calloc((size_t)n * (size_t)k + 1, sizeof(uint64_t));
  uint64_t *wtab = malloc(sizeof(uint64_t) * (size_t)k * (size_t)k);
  for (int d = 1; d <= k; ++d)
    for (int j = 1; j <= k; ++j)
      wtab[(d - 1) * k + (j - 1)] =
          tsvo_draw_nonzero(seed, ROLE_SHADE_W, (uint64_t)d, (uint64_t)j, 0);
  for (int32_t x = 0; x < n; ++x)
    for (int32_t s = vertex_off[x]; s < vertex_off[x + 1]; ++s) {
      int d = vertex_shades[s];
      uint64_t vv = tsvo_draw_nonzero(seed, ROLE_SHADE_V, (uint64_t)x,
                                      (uint64_t)d, 0);
      for (int j = 0; j < k; ++j)
        zj[(size_t)x * k + j] ^= tsvo_gf_mul(vv, wtab[(d - 1) * k + j]);
    }
  free(wtab);

  /* Arcs grouped into runs by (ts, head, tail) order (graph.cpp:50-79). */
  int64_t na = directed ? m : 2 * m;
  rawarc_t *arcs = malloc(sizeof(rawarc_t) * (size_t)(na > 0 ? na : 1));
  int64_t q = 0;
  for (int64_t i = 0; i < m; ++i) {
    if (ets[i] > max_ts) continue; /* arcs after the horizon never count */
    arcs[q++] = (rawarc_t){ets[i], ev[i], eu[i], (int32_t)i};
    if (!directed) arcs[q++] = (rawarc_t){ets[i], eu[i], ev[i], (int32_t)i};
  }
  na = q;
  qsort(arcs, (size_t)na, sizeof(rawarc_t), cmp_arc);
  /* run r = arcs[rb[r], rb[r+1]) ; runs are in (ts, head) order */
  int64_t *rb = malloc(sizeof(int64_t) * (size_t)(na + 1));
  int64_t nr = 0;
  for (int64_t i = 0; i < na; ++i)
    if (i == 0 || arcs[i].ts != arcs[i - 1].ts ||
        arcs[i].head != arcs[i - 1].head)
      rb[nr++] = i;
  rb[nr] = na;

  uint64_t *z = malloc(sizeof(uint64_t) * (size_t)(n > 0 ? n : 1));
  uint64_t *tprev = malloc(sizeof(uint64_t) * (size_t)(nr + 1)); /* Q_{l-1} after run r */
  uint64_t *tcur = malloc(sizeof(uint64_t) * (size_t)(nr + 1));
  int64_t *last = malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  uint64_t *run_sum = malloc(sizeof(uint64_t) * (size_t)(nr + 1));
  uint64_t *pfx = malloc(sizeof(uint64_t) * (size_t)(n > 0 ? n : 1));
  uint64_t *ycache = malloc(sizeof(uint64_t) * (size_t)(na > 0 ? na : 1));

  for (uint64_t A = p_begin; A < p_end; ++A) {
    /* z_u^A (sieve.cpp:116-133): bit j of A selects z_{u,j}. */
    for (int32_t x = 0; x < n; ++x) {
      uint64_t s = 0;
      for (int j = 0; j < k; ++j)
        if ((A >> j) & 1) s ^= zj[(size_t)x * k + j];
      z[x] = s;
    }
    if (k == 1) { /* sieve.cpp:203-213 */
      for (int32_t x = 0; x < n; ++x)
        if (anchor_source < 0 || x == anchor_source) acc[x] ^= z[x];
      continue;
    }
    for (int ell = 2; ell <= k; ++ell) {
      for (int64_t i = 0; i < na; ++i)
        ycache[i] = tsvo_draw_nonzero(seed, ROLE_EDGE_Y,
                                      (uint64_t)arcs[i].edge,
                                      (uint64_t)(ell - 1), 0);
      /* last[v]: v's latest run (level l-1) strictly before the current
       * timestamp; pfx[v]: running Q_l(v, .). */
      for (int32_t x = 0; x < n; ++x) {
        last[x] = -1;
        pfx[x] = 0;
      }
      int64_t r = 0;
      while (r < nr) {
        int32_t tsr = arcs[rb[r]].ts;
        int64_t r_end = r;
        while (r_end < nr && arcs[rb[r_end]].ts == tsr) ++r_end;
        /* all runs at this timestamp read state from strictly earlier ones */
        for (int64_t x = r; x < r_end; ++x) {
          uint64_t tmp = 0;
          for (int64_t a = rb[x]; a < rb[x + 1]; ++a) {
            int32_t tail = arcs[a].tail;
            uint64_t src;
            if (ell == 2) {
              if (anchor_source >= 0 && tail != anchor_source) continue;
              src = z[tail];
            } else {
              src = last[tail] >= 0 ? tprev[last[tail]] : 0;
            }
            tmp ^= tsvo_gf_mul(ycache[a], src);
          }
          run_sum[x] = tsvo_gf_mul(z[arcs[rb[x]].head], tmp);
        }
        for (int64_t x = r; x < r_end; ++x) {
          int32_t h = arcs[rb[x]].head;
          pfx[h] ^= run_sum[x];
          tcur[x] = pfx[h];
        }
        /* expose level l-1 runs at tsr to the next timestamp */
        for (int64_t x = r; x < r_end; ++x) last[arcs[rb[x]].head] = x;
        r = r_end;
      }
      uint64_t *sw = tprev;
      tprev = tcur;
      tcur = sw;
      if (ell == k)
        for (int32_t x = 0; x < n; ++x) acc[x] ^= pfx[x];
    }
  }
  free(zj);
  free(arcs);
  free(rb);
  free(z);
  free(tprev);
  free(tcur);
  free(last);
  free(run_sum);
  free(pfx);
  free(ycache);
  return 0;
}

/*
 * finalize (sieve.cpp:136-159): zero everything but the sink when anchored,
 * return the number of flagged vertices and the FNV-1a checksum over
 * (u, acc[u]) little-endian byte pairs of nonzero accumulators.
 */
int64_t tsvo_finalize(int32_t n, uint64_t *acc, int32_t anchor_sink,
                      uint64_t *checksum) {
  int64_t flagged = 0;
  uint64_t h = 1469598103934665603ull;
  for (int32_t x = 0; x < n; ++x) {
    if (anchor_sink >= 0 && x != anchor_sink) acc[x] = 0;
    if (!acc[x]) continue;
    ++flagged;
    uint64_t words[2] = {(uint64_t)x, acc[x]};
    for (int w = 0; w < 2; ++w)
      for (int i = 0; i < 8; ++i) {
        h ^= (words[w] >> (8 * i)) & 0xff;
        h *= 1099511628211ull;
      }
  }
  *checksum = h;
  return flagged;
}

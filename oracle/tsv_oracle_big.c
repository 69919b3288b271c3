/*
 * tsv_oracle_big.c -- multi-threaded, memory-lean restatement of the temporal
 * sieve for the BASELINE sizes (configs 2-5 at full size).
 *
 * TEST INFRASTRUCTURE ONLY (same rules as tsv_oracle.c): loaded by tests/,
 * tests/golden/make_golden_full.py and bench.py's cpu_baseline /
 * `--impl reference` legs, never by the product package.
 *
 * It computes exactly what tsv_oracle.c:tsvo_eval_points computes -- the
 * point form of the reference's DP, sieve point by sieve point -- and is
 * pinned against it (and through it against the compiled reference) by
 * tests/test_oracle.py.  What differs is only the organisation, so that a
 * 1e9-edge graph fits in host RAM and all host cores are used:
 *
 *   - canonical edge ids (graph.cpp:14-43: drop loops, undirected u<v, sort
 *     (ts,u,v), dedup; id = index) are formed IN PLACE in the caller's
 *     arrays: a counting sort by timestamp, then each timestamp bucket sorted
 *     on the packed (u,v) key;
 *   - arcs are grouped by head (stable in edge-id = time order), and a run is
 *     one (head, ts) group; the sieve state is kept per run:
 *         T_l[run] = z_head^A * XOR_{a in run} y(e_a, l-1) * Q_{l-1}(tail_a, ts-1)
 *         Q_l(v, i) = XOR of T_l over v's runs with ts <= i   (the stay term,
 *                     sieve.cpp:229-230), Q_1(v, .) = z_v^A
 *     (sieve.cpp:215-256).  Level l depends only on level l-1, so every head
 *     of one level is independent: OpenMP runs over heads;
 *   - `lanes` sieve points are evaluated per pass (lane batch, sieve.cpp:
 *     199-205) so one y draw (gf.hpp:135-153, Role::edge_y, sieve.cpp:243-245)
 *     serves the batch;
 *   - readout acc[u] ^= XOR_A Q_k(u, max_ts) (sieve.cpp:294-306); anchor:
 *     level 2 only from tail == source (sieve.cpp:241-242); k = 1 sums z
 *     (sieve.cpp:203-213).  The sink restriction is tsvo_finalize's.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <omp.h>

#include "tsv_gf.h"
#define NONE 0xFFFFFFFFu

static int cmp_u64(const void *a, const void *b) {
  uint64_t x = *(const uint64_t *)a, y = *(const uint64_t *)b;
  return x < y ? -1 : (x > y);
}

/*
 * Canonicalize (u, v, ts) in place (graph.cpp:14-43).  Returns the number of
 * canonical edges (they occupy u/v/ts[0..return)), -1 on an endpoint or
 * timestamp range error, -2 when timestamps exceed the bucket limit.
 */
int64_t tsvo_canonicalize_inplace(int32_t n, int64_t m, int32_t *u, int32_t *v,
                                  int32_t *ts, int directed) {
  int64_t k = 0;
  int32_t tmax = 0;
  for (int64_t i = 0; i < m; ++i) {
    int32_t a = u[i], b = v[i], t = ts[i];
    if (a < 0 || a >= n || b < 0 || b >= n || t < 1) return -1;
    if (a == b) continue;
    if (!directed && a > b) {
      int32_t s = a;
      a = b;
      b = s;
    }
    u[k] = a;
    v[k] = b;
    ts[k] = t;
    if (t > tmax) tmax = t;
    ++k;
  }
  if (tmax > (1 << 28)) return -2;
  int64_t nb = (int64_t)tmax + 2;
  int64_t *off = calloc((size_t)nb, sizeof(int64_t));
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < k; ++i) {
#pragma omp atomic
    off[ts[i] + 1]++;
  }
  for (int64_t b = 1; b < nb; ++b) off[b] += off[b - 1];
  int64_t *cur = malloc(sizeof(int64_t) * (size_t)nb);
  memcpy(cur, off, sizeof(int64_t) * (size_t)nb);
  uint64_t *key = malloc(sizeof(uint64_t) * (size_t)(k > 0 ? k : 1));
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < k; ++i) {
    int64_t p;
#pragma omp atomic capture
    p = cur[ts[i]]++;
    key[p] = ((uint64_t)(uint32_t)u[i] << 32) | (uint32_t)v[i];
  }
  /* sort + dedup every bucket; kept counts into cur[b] */
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t b = 0; b < nb - 1; ++b) {
    int64_t lo = off[b], hi = off[b + 1];
    if (hi - lo > 1) qsort(key + lo, (size_t)(hi - lo), sizeof(uint64_t), cmp_u64);
    int64_t w = lo;
    for (int64_t i = lo; i < hi; ++i)
      if (w == lo || key[w - 1] != key[i]) key[w++] = key[i];
    cur[b] = w - lo;
  }
  /* exclusive scan of kept counts -> output offsets (reuse cur) */
  int64_t acc = 0;
  for (int64_t b = 0; b < nb - 1; ++b) {
    int64_t c = cur[b];
    cur[b] = acc;
    acc += c;
  }
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t b = 0; b < nb - 1; ++b) {
    int64_t lo = off[b], o = cur[b];
    int64_t cnt = (b + 1 < nb - 1 ? cur[b + 1] : acc) - o;
    for (int64_t j = 0; j < cnt; ++j) {
      uint64_t x = key[lo + j];
      u[o + j] = (int32_t)(x >> 32);
      v[o + j] = (int32_t)(uint32_t)x;
      ts[o + j] = (int32_t)b;
    }
  }
  free(key);
  free(cur);
  free(off);
  return acc;
}

typedef struct {
  int32_t n;
  int64_t na, nr;
  int64_t *hoff;     /* n+1: arcs of head h are [hoff[h], hoff[h+1]), time order */
  int32_t *a_tail;   /* na */
  uint32_t *a_eid;   /* na: canonical edge id */
  int32_t *a_ts;     /* na */
  int64_t *roff;     /* n+1: runs of head h are [roff[h], roff[h+1]) */
  int32_t *r_ts;     /* nr */
  uint32_t *a_src;   /* na: tail's last run with ts' < ts (global run index), NONE */
} tsvo_big;

/*
 * Head-grouped arcs and runs of the canonical edges (graph.cpp:50-79),
 * keeping only arcs with ts <= max_ts (sieve.cpp:235: later arcs never
 * count).  Returns NULL when the arc count does not fit 32-bit indices.
 */
void *tsvo_big_build(int32_t n, int64_t m, const int32_t *u, const int32_t *v,
                     const int32_t *ts, int directed, int32_t max_ts) {
  tsvo_big *G = calloc(1, sizeof(tsvo_big));
  G->n = n;
  G->hoff = calloc((size_t)n + 1, sizeof(int64_t));
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < m; ++i) {
    if (ts[i] > max_ts) continue;
#pragma omp atomic
    G->hoff[v[i] + 1]++;
    if (!directed) {
#pragma omp atomic
      G->hoff[u[i] + 1]++;
    }
  }
  for (int64_t h = 1; h <= n; ++h) G->hoff[h] += G->hoff[h - 1];
  G->na = G->hoff[n];
  if (G->na >= (int64_t)NONE) {
    free(G->hoff);
    free(G);
    return NULL;
  }
  size_t na1 = (size_t)(G->na > 0 ? G->na : 1);
  G->a_tail = malloc(sizeof(int32_t) * na1);
  G->a_eid = malloc(sizeof(uint32_t) * na1);
  {
    int64_t *cur = malloc(sizeof(int64_t) * ((size_t)n + 1));
    memcpy(cur, G->hoff, sizeof(int64_t) * ((size_t)n + 1));
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < m; ++i) {
      if (ts[i] > max_ts) continue;
      int64_t p;
#pragma omp atomic capture
      p = cur[v[i]]++;
      G->a_tail[p] = u[i];
      G->a_eid[p] = (uint32_t)i;
      if (!directed) {
#pragma omp atomic capture
        p = cur[u[i]]++;
        G->a_tail[p] = v[i];
        G->a_eid[p] = (uint32_t)i;
      }
    }
    free(cur);
  }
  /* restore edge-id (= time) order inside every head; count runs */
  G->a_ts = malloc(sizeof(int32_t) * na1);
  G->roff = calloc((size_t)n + 1, sizeof(int64_t));
#pragma omp parallel
  {
    uint64_t *tmp = NULL;
    size_t cap = 0;
#pragma omp for schedule(dynamic, 1024)
    for (int64_t h = 0; h < n; ++h) {
      int64_t lo = G->hoff[h], hi = G->hoff[h + 1], L = hi - lo;
      if (L > 1) {
        if ((size_t)L > cap) {
          cap = (size_t)L * 2;
          tmp = realloc(tmp, cap * sizeof(uint64_t));
        }
        for (int64_t j = 0; j < L; ++j)
          tmp[j] = ((uint64_t)G->a_eid[lo + j] << 32) | (uint32_t)G->a_tail[lo + j];
        qsort(tmp, (size_t)L, sizeof(uint64_t), cmp_u64);
        for (int64_t j = 0; j < L; ++j) {
          G->a_eid[lo + j] = (uint32_t)(tmp[j] >> 32);
          G->a_tail[lo + j] = (int32_t)(uint32_t)tmp[j];
        }
      }
      int64_t runs = 0;
      for (int64_t a = lo; a < hi; ++a) {
        G->a_ts[a] = ts[G->a_eid[a]];
        if (a == lo || G->a_ts[a] != G->a_ts[a - 1]) ++runs;
      }
      G->roff[h + 1] = runs;
    }
    free(tmp);
  }
  for (int64_t h = 1; h <= n; ++h) G->roff[h] += G->roff[h - 1];
  G->nr = G->roff[n];
  G->r_ts = malloc(sizeof(int32_t) * (size_t)(G->nr > 0 ? G->nr : 1));
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t h = 0; h < n; ++h) {
    int64_t r = G->roff[h];
    for (int64_t a = G->hoff[h]; a < G->hoff[h + 1]; ++a)
      if (a == G->hoff[h] || G->a_ts[a] != G->a_ts[a - 1]) G->r_ts[r++] = G->a_ts[a];
  }
  /* predecessor run of every arc: the tail's last run strictly before ts */
  G->a_src = malloc(sizeof(uint32_t) * na1);
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t h = 0; h < n; ++h)
    for (int64_t a = G->hoff[h]; a < G->hoff[h + 1]; ++a) {
      int32_t t = G->a_tail[a], x = G->a_ts[a];
      int64_t lo = G->roff[t], hi = G->roff[t + 1]; /* first run with ts >= x */
      while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (G->r_ts[mid] < x) lo = mid + 1;
        else hi = mid;
      }
      G->a_src[a] = lo > G->roff[t] ? (uint32_t)(lo - 1) : NONE;
    }
  free(G->r_ts); /* only the predecessor search needs run timestamps */
  G->r_ts = NULL;
  return G;
}

void tsvo_big_free(void *p) {
  tsvo_big *G = p;
  if (!G) return;
  free(G->hoff);
  free(G->a_tail);
  free(G->a_eid);
  free(G->a_ts);
  free(G->roff);
  free(G->r_ts);
  free(G->a_src);
  free(G);
}

int64_t tsvo_big_arcs(const void *p) { return ((const tsvo_big *)p)->na; }
int64_t tsvo_big_runs(const void *p) { return ((const tsvo_big *)p)->nr; }

#define MAXW 16

/*
 * One level ell (2..k) of the DP for the heads in [v_lo, v_hi): reads the
 * level ell-1 run states `prev` (z at level 2), writes the level ell run
 * states of these heads into `cur` (ell < k) or XORs their readout into acc
 * (ell == k).  Heads are independent within a level (sieve.cpp:215-256).
 */
static void big_level(const tsvo_big *G, int ell, int k, const uint64_t *z, int W, int wn,
                      uint64_t seed, int32_t anchor_source, int64_t v_lo, int64_t v_hi,
                      const uint64_t *prev, uint64_t *cur, uint64_t *acc) {
  const int last = ell == k;
#pragma omp parallel for schedule(dynamic, 256)
  for (int64_t h = v_lo; h < v_hi; ++h) {
    int64_t a = G->hoff[h], ae = G->hoff[h + 1];
    if (a == ae) continue;
    uint64_t pfx[MAXW], tmp[MAXW];
    const uint64_t *zh = z + h * W;
    for (int w = 0; w < W; ++w) pfx[w] = 0;
    int64_t r = G->roff[h];
    while (a < ae) {
      int32_t t = G->a_ts[a];
      for (int w = 0; w < W; ++w) tmp[w] = 0;
      for (; a < ae && G->a_ts[a] == t; ++a) {
        if (ell > 2 && a + 16 < ae && G->a_src[a + 16] != NONE)
          __builtin_prefetch(prev + (int64_t)G->a_src[a + 16] * W);
        const uint64_t *src;
        if (ell == 2) {
          if (anchor_source >= 0 && G->a_tail[a] != anchor_source) continue;
          src = z + (int64_t)G->a_tail[a] * W;
        } else {
          if (G->a_src[a] == NONE) continue;
          src = prev + (int64_t)G->a_src[a] * W;
        }
        uint64_t y = draw_nonzero(seed, ROLE_EDGE_Y, (uint64_t)G->a_eid[a], (uint64_t)(ell - 1), 0);
        for (int w = 0; w < wn; ++w) tmp[w] ^= gf_mul(y, src[w]);
      }
      for (int w = 0; w < wn; ++w) pfx[w] ^= gf_mul(zh[w], tmp[w]);
      if (!last)
        for (int w = 0; w < W; ++w) cur[r * W + w] = pfx[w];
      ++r;
    }
    if (last) {
      uint64_t s = 0;
      for (int w = 0; w < wn; ++w) s ^= pfx[w];
      acc[h] ^= s;
    }
  }
}

/* zj (n x k, sieve.cpp:83-101) and z_u^A for points [base, base+wn), W lanes */
static void big_z(const tsvo_big *G, int k, const int32_t *vertex_off,
                  const int32_t *vertex_shades, uint64_t seed, uint64_t base, int W, int wn,
                  uint64_t *zj, uint64_t *z) {
  const int64_t n = G->n;
  uint64_t wtab[30 * 30];
  for (int d = 1; d <= k; ++d)
    for (int j = 1; j <= k; ++j)
      wtab[(d - 1) * k + (j - 1)] = draw_nonzero(seed, ROLE_SHADE_W, (uint64_t)d, (uint64_t)j, 0);
  memset(zj, 0, sizeof(uint64_t) * (size_t)n * (size_t)k);
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t x = 0; x < n; ++x)
    for (int32_t s = vertex_off[x]; s < vertex_off[x + 1]; ++s) {
      int d = vertex_shades[s];
      uint64_t vv = draw_nonzero(seed, ROLE_SHADE_V, (uint64_t)x, (uint64_t)d, 0);
      for (int j = 0; j < k; ++j) zj[x * k + j] ^= gf_mul(vv, wtab[(d - 1) * k + j]);
    }
#pragma omp parallel for schedule(static)
  for (int64_t x = 0; x < n; ++x)
    for (int w = 0; w < W; ++w) {
      uint64_t s = 0, A = base + (uint64_t)w;
      if (w < wn)
        for (int j = 0; j < k; ++j)
          if ((A >> j) & 1) s ^= zj[x * k + j];
      z[x * W + w] = s;
    }
}

/*
 * The vertex-partitioned form (the multi-GPU algorithm of DESIGN.md section
 * 6, restated point by point): level ell for the heads [v_lo, v_hi) and the
 * points [p_begin, p_begin + lanes); run states are `lanes` words per run.
 * tsvo_big_run_range gives the run-state range a head range writes.
 */
int tsvo_big_level(const void *p, int k, int ell, const int32_t *vertex_off,
                   const int32_t *vertex_shades, uint64_t seed, int32_t anchor_source,
                   uint64_t p_begin, int lanes, int64_t v_lo, int64_t v_hi,
                   const uint64_t *prev, uint64_t *cur, uint64_t *acc) {
  const tsvo_big *G = p;
  if (k < 2 || k > 30 || ell < 2 || ell > k || lanes < 1 || lanes > MAXW) return -1;
  uint64_t *zj = malloc(sizeof(uint64_t) * ((size_t)G->n * (size_t)k + 1));
  uint64_t *z = malloc(sizeof(uint64_t) * ((size_t)G->n * lanes + 1));
  if (!zj || !z) {
    free(zj);
    free(z);
    return -3;
  }
  big_z(G, k, vertex_off, vertex_shades, seed, p_begin, lanes, lanes, zj, z);
  big_level(G, ell, k, z, lanes, lanes, seed, anchor_source, v_lo, v_hi, prev, cur, acc);
  free(zj);
  free(z);
  return 0;
}

void tsvo_big_run_range(const void *p, int64_t v_lo, int64_t v_hi, int64_t *r_lo, int64_t *r_hi) {
  const tsvo_big *G = p;
  *r_lo = G->roff[v_lo];
  *r_hi = G->roff[v_hi];
}

/*
 * XOR the sieve points [p_begin, p_end) into acc[0..n) (not cleared), `lanes`
 * points per pass (1..16).  Same contract as tsvo_eval_points.  Returns 0, or
 * -1 for k out of range / bad lanes, -3 when memory is short.
 */
int tsvo_big_eval(const void *p, int k, const int32_t *vertex_off,
                  const int32_t *vertex_shades, uint64_t seed,
                  int32_t anchor_source, uint64_t p_begin, uint64_t p_end,
                  int lanes, uint64_t *acc) {
  const tsvo_big *G = p;
  if (k < 1 || k > 30 || lanes < 1 || lanes > MAXW) return -1;
  const int32_t n = G->n;
  const int W = lanes;
  /* z_{u,j} (sieve.cpp:83-101) */
  uint64_t wtab[30 * 30];
  for (int d = 1; d <= k; ++d)
    for (int j = 1; j <= k; ++j)
      wtab[(d - 1) * k + (j - 1)] =
          draw_nonzero(seed, ROLE_SHADE_W, (uint64_t)d, (uint64_t)j, 0);
  uint64_t *zj = calloc((size_t)n * (size_t)k + 1, sizeof(uint64_t));
  uint64_t *z = malloc(sizeof(uint64_t) * ((size_t)n * W + 1));
  uint64_t *S0 = NULL, *S1 = NULL;
  if (k > 2) {
    S0 = malloc(sizeof(uint64_t) * ((size_t)G->nr * W + 1));
    S1 = malloc(sizeof(uint64_t) * ((size_t)G->nr * W + 1));
  }
  if (!zj || !z || (k > 2 && (!S0 || !S1))) {
    free(zj);
    free(z);
    free(S0);
    free(S1);
    return -3;
  }
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t x = 0; x < n; ++x)
    for (int32_t s = vertex_off[x]; s < vertex_off[x + 1]; ++s) {
      int d = vertex_shades[s];
      uint64_t vv = draw_nonzero(seed, ROLE_SHADE_V, (uint64_t)x, (uint64_t)d, 0);
      for (int j = 0; j < k; ++j) zj[x * k + j] ^= gf_mul(vv, wtab[(d - 1) * k + j]);
    }

  for (uint64_t base = p_begin; base < p_end; base += (uint64_t)W) {
    int wn = (int)((p_end - base) < (uint64_t)W ? (p_end - base) : (uint64_t)W);
    /* z_u^A (sieve.cpp:116-133): bit j of A selects z_{u,j}; idle lanes 0 */
#pragma omp parallel for schedule(static)
    for (int64_t x = 0; x < n; ++x)
      for (int w = 0; w < W; ++w) {
        uint64_t s = 0, A = base + (uint64_t)w;
        if (w < wn)
          for (int j = 0; j < k; ++j)
            if ((A >> j) & 1) s ^= zj[x * k + j];
        z[x * W + w] = s;
      }
    if (k == 1) {
      for (int64_t x = 0; x < n; ++x)
        if (anchor_source < 0 || x == anchor_source)
          for (int w = 0; w < W; ++w) acc[x] ^= z[x * W + w];
      continue;
    }
    uint64_t *prev = S0, *cur = S1;
    for (int ell = 2; ell <= k; ++ell) {
      big_level(G, ell, k, z, W, wn, seed, anchor_source, 0, n, prev, cur, acc);
      uint64_t *sw = prev;
      prev = cur;
      cur = sw;
    }
  }
  free(zj);
  free(z);
  free(S0);
  free(S1);
  return 0;
}

void tsvo_set_threads(int t) {
  if (t > 0) omp_set_num_threads(t);
}

int tsvo_max_threads(void) { return omp_get_max_threads(); }

"""Seeded synthetic instances of the BASELINE.json configurations.

The reference's generators (/root/reference/proj/core/src/generator.cpp)
cannot produce these shapes (uniform-endpoint and Chung-Lu graphs at
1e4..1e9 edges), so the benchmark owns its generators.  Every instance has
exactly m distinct (u, v, ts) triples with u != v, vertex ids 0..n-1 and
timestamps in [1, t], so TemporalGraph::build drops nothing.  Colors c_i of
BASELINE map to reference colors i+1 (colors are 1-based).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class Instance:
    name: str
    n: int
    u: np.ndarray
    v: np.ndarray
    ts: np.ndarray
    t: int
    directed: bool
    colors: np.ndarray          # 1-based colors, length n
    problem: str                # ktemppath | pathmotif | colorfulpath | sdcolorful
    motif: list                 # color multiset (pathmotif/colorfulpath)
    k: int                      # query size (interior size for sdcolorful)
    source: int = -1
    dest: int = -1
    planted: list | None = None  # planted path vertices

    @property
    def m(self) -> int:
        return len(self.u)

    @property
    def k_eff(self) -> int:
        return self.k + 2 if self.problem == "sdcolorful" else self.k

    @property
    def arcs(self) -> int:
        return self.m if self.directed else 2 * self.m

    def updates(self) -> int:
        """A * (k_eff - 1) * 2^k_eff: algorithmic edge x level x point updates."""
        return self.arcs * (self.k_eff - 1) * (1 << self.k_eff)


def _endpoints_uniform(rng, n, size):
    u = rng.integers(0, n, size, dtype=np.int64)
    v = rng.integers(0, n - 1, size, dtype=np.int64)
    v = v + (v >= u)  # uniform over v != u
    return u, v


def _endpoints_chung_lu(rng, n, size, gamma, cdf):
    u = np.searchsorted(cdf, rng.random(size), side="right").astype(np.int64)
    v = np.searchsorted(cdf, rng.random(size), side="right").astype(np.int64)
    np.minimum(u, n - 1, out=u)
    np.minimum(v, n - 1, out=v)
    return u, v


def _distinct_edges(rng, n, m, t, draw, fixed=None):
    """m distinct (u, v, ts) with u != v; `fixed` triples are included first."""
    key_parts = []
    if fixed is not None and len(fixed[0]):
        fu, fv, ft = (np.asarray(x, np.int64) for x in fixed)
        key_parts.append((fu * n + fv) * (t + 1) + ft)
    need = m
    keys = np.unique(np.concatenate(key_parts)) if key_parts else np.zeros(0, np.int64)
    while len(keys) < need:
        want = int((need - len(keys)) * 1.05) + 16
        u, v = draw(want)
        ok = u != v
        u, v = u[ok], v[ok]
        ts = rng.integers(1, t + 1, len(u), dtype=np.int64)
        fresh = (u * n + v) * (t + 1) + ts
        keys = np.unique(np.concatenate([keys, fresh]))
    if len(keys) > need:
        # keep the fixed triples, drop a random subset of the rest
        if key_parts:
            fixed_keys = np.unique(np.concatenate(key_parts))
            rest = np.setdiff1d(keys, fixed_keys, assume_unique=True)
            rest = rng.permutation(rest)[:need - len(fixed_keys)]
            keys = np.concatenate([fixed_keys, rest])
        else:
            keys = rng.permutation(keys)[:need]
    keys = rng.permutation(keys)  # file order is irrelevant to build()
    ts = (keys % (t + 1)).astype(np.int32)
    uv = keys // (t + 1)
    return (uv // n).astype(np.int32), (uv % n).astype(np.int32), ts


def _planted_path(rng, n, kv, t, exclude=()):
    verts = []
    ex = set(exclude)
    while len(verts) < kv:
        x = int(rng.integers(0, n))
        if x not in ex and x not in verts:
            verts.append(x)
    times = np.sort(rng.choice(np.arange(1, t + 1), kv - 1, replace=False))
    return verts, times


def make_config(cfg: int, seed: int = 1, scale: float = 1.0) -> Instance:
    """BASELINE.json configs[cfg-1].  `scale` < 1 shrinks n and m (tests)."""
    rng = np.random.default_rng(1000 + 17 * cfg + seed)
    if cfg == 1:
        n, m, t = 1000, 10_000, 100
        verts, times = _planted_path(rng, n, 5, t)
        fixed = (verts[:-1], verts[1:], times)
        u, v, ts = _distinct_edges(rng, n, m, t, lambda s: _endpoints_uniform(rng, n, s), fixed)
        return Instance("C1 k-TempPath k=5", n, u, v, ts, t, True, np.ones(n, np.int32),
                        "ktemppath", [], 5, planted=verts)
    if cfg == 2:
        n, m, t = int(100_000 * scale), int(1_000_000 * scale), 1000
        colors = rng.integers(1, 9, n).astype(np.int32)
        motif = [1, 1, 2, 3, 4, 5]
        verts, times = _planted_path(rng, n, 6, t)
        for x, c in zip(verts, motif):
            colors[x] = c
        fixed = (verts[:-1], verts[1:], times)
        u, v, ts = _distinct_edges(rng, n, m, t, lambda s: _endpoints_uniform(rng, n, s), fixed)
        return Instance("C2 PathMotif k=6", n, u, v, ts, t, True, colors, "pathmotif", motif, 6,
                        planted=verts)
    if cfg in (3, 4):
        if cfg == 3:
            n, m, t, gamma, q, k = int(1_000_000 * scale), int(10_000_000 * scale), 10_000, 2.1, 8, 8
        else:
            n, m, t, gamma, q, k = (int(1_000_000 * scale), int(100_000_000 * scale), 100_000, 2.3,
                                    10, 10)
        w = np.arange(1, n + 1, dtype=np.float64) ** (-1.0 / (gamma - 1.0))
        cdf = np.cumsum(w)
        cdf /= cdf[-1]
        colors = rng.integers(1, q + 1, n).astype(np.int32)
        if cfg == 3:
            motif = list(range(1, 9))
            verts, times = _planted_path(rng, n, 8, t)
            for x, c in zip(verts, motif):
                colors[x] = c
            src, dst = -1, -1
        else:
            motif = []
            src, dst = 0, n - 1
            inner, _ = _planted_path(rng, n, k, t, exclude=(src, dst))
            verts = [src] + inner + [dst]
            times = np.sort(rng.choice(np.arange(1, t + 1), len(verts) - 1, replace=False))
            for x, c in zip(inner, range(1, k + 1)):
                colors[x] = c
        fixed = (verts[:-1], verts[1:], times)
        u, v, ts = _distinct_edges(rng, n, m, t,
                                   lambda s: _endpoints_chung_lu(rng, n, s, gamma, cdf), fixed)
        if cfg == 3:
            return Instance("C3 ColorfulPath k=8", n, u, v, ts, t, True, colors, "colorfulpath",
                            motif, 8, planted=verts)
        return Instance("C4 (s,d)-ColorfulPath k=10", n, u, v, ts, t, True, colors, "sdcolorful",
                        [], 10, source=src, dest=dst, planted=verts)
    if cfg == 5:
        n, m, t = int(100_000_000 * scale), int(1_000_000_000 * scale), int(1_000_000 * min(1, scale * 10))
        t = max(t, 100)
        verts, times = _planted_path(rng, n, 5, t)
        if m >= 50_000_000:
            # n^2 t = 1e22 keys for m = 1e9 draws: ~5e-5 expected duplicate
            # triples, so the global de-duplication sort is skipped at scale
            # (TemporalGraph::build still drops any, and reports the count).
            u, v = _endpoints_uniform(rng, n, m)
            u, v = u.astype(np.int32), v.astype(np.int32)
            ts = rng.integers(1, t + 1, m, dtype=np.int32)
            u[:4], v[:4], ts[:4] = verts[:-1], verts[1:], times
        else:
            fixed = (verts[:-1], verts[1:], times)
            u, v, ts = _distinct_edges(rng, n, m, t, lambda s: _endpoints_uniform(rng, n, s), fixed)
        return Instance("C5 k-TempPath k=5 at scale", n, u, v, ts, t, True, np.ones(n, np.int32),
                        "ktemppath", [], 5, planted=verts)
    raise ValueError(f"unknown config {cfg}")


def effective_query(inst: Instance):
    """(k_eff, colors_eff, motif_eff, anchor) per make_effective
    (/root/reference/proj/core/src/solver.cpp:42-126)."""
    if inst.problem == "ktemppath":
        return inst.k, np.ones(inst.n, np.int32), [1] * inst.k, (-1, -1)
    if inst.problem in ("pathmotif", "colorfulpath"):
        return inst.k, inst.colors, list(inst.motif), (-1, -1)
    if inst.problem == "sdcolorful":
        k = inst.k
        c = inst.colors.copy()
        c[(c < 1) | (c > k)] = k + 3
        c[inst.source] = k + 1
        c[inst.dest] = k + 2
        return k + 2, c, list(range(1, k + 3)), (inst.source, inst.dest)
    raise ValueError(inst.problem)


def random_small(rng, n_max=20, m_max=60, t_max=8, k_max=6, q_max=4):
    """A small random instance for parity sweeps (may contain loops/dups)."""
    n = int(rng.integers(2, n_max + 1))
    m = int(rng.integers(0, m_max + 1))
    t = int(rng.integers(1, t_max + 1))
    u = rng.integers(0, n, m).astype(np.int32)
    v = rng.integers(0, n, m).astype(np.int32)
    ts = rng.integers(1, t + 1, m).astype(np.int32)
    q = int(rng.integers(1, q_max + 1))
    colors = rng.integers(1, q + 1, n).astype(np.int32)
    k = int(rng.integers(1, k_max + 1))
    motif = [int(x) for x in rng.integers(1, q + 1, k)]
    return n, u, v, ts, bool(rng.integers(0, 2)), colors, motif

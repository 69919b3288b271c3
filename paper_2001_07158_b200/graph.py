"""Temporal-graph data model -- Python mirror of tsieve/graph.hpp + motif.hpp.

Reference: /root/reference/proj/core/include/tsieve/graph.hpp (TemporalGraph
:49-111, VertexColoring :114-139, load_graph :229-235, restrict_to :246-248)
and motif.hpp:11-74.  ``TemporalGraph.build`` canonicalizes and uploads
through the C-ABI (``tsv_graph_build``), so edge ids -- which address the y
draws -- are those of graph.cpp:14-43.
"""
from __future__ import annotations

import ctypes as C
import io
from dataclasses import dataclass, field

import numpy as np

from . import _native

Vertex = int
Timestamp = int
Color = int


class TemporalGraph:
    """Immutable device-resident temporal graph (one per CUDA device)."""

    def __init__(self, handle, info: _native.GraphInfo):
        self._h = handle
        self._info = info
        self._edges = None

    @staticmethod
    def build(n: int, edges, directed: bool, t: int = 0, device: int = 0) -> "TemporalGraph":
        """TemporalGraph::build(n, edges, directed, t) (graph.hpp:55-56)."""
        u, v, ts = _edge_arrays(edges)
        h = C.c_void_p()
        _native.check(_native.lib().tsv_graph_build(int(n), len(u), u, v, ts, int(bool(directed)),
                                                     int(t), int(device), C.byref(h)))
        info = _native.GraphInfo()
        _native.check(_native.lib().tsv_graph_get_info(h, C.byref(info)))
        return TemporalGraph(h, info)

    @staticmethod
    def build_model(n: int, edges, directed: bool, edge_model: str, eps=None, delays=None,
                    t: int = 0, device: int = 0) -> "TemporalGraph":
        """TemporalGraph::build with transition times + set_delays, mirrored on
        the device for one edge model (tsv_graph_build_model): an arc
        departing at ts lands at ts + eps - 1 and reads its tail at
        ts - delta(tail) (sieve.cpp:257-291)."""
        from .sieve import EDGE_MODELS
        model = EDGE_MODELS[edge_model]
        u, v, ts = _edge_arrays(edges)
        cu, cv, ct, ce = _native.canonical_edges_eps(n, u, v, ts, eps, directed)
        dl = None if delays is None else np.ascontiguousarray(delays, dtype=np.int32)
        if dl is not None and len(dl) != n:
            raise ValueError("delay vector size mismatch")
        h = C.c_void_p()
        _native.check(_native.lib().tsv_graph_build_model(
            int(n), len(cu), cu if len(cu) else np.zeros(1, np.int32),
            cv if len(cv) else np.zeros(1, np.int32), ct if len(ct) else np.zeros(1, np.int32),
            ce.ctypes.data if (eps is not None and len(ce)) else None,
            None if dl is None else dl.ctypes.data, int(bool(directed)), int(t), model,
            int(device), C.byref(h)))
        info = _native.GraphInfo()
        _native.check(_native.lib().tsv_graph_get_info(h, C.byref(info)))
        g = TemporalGraph(h, info)
        g._eps = ce
        g._keep = (ce, dl)  # host copies outlive the handle's build
        return g

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                _native.lib().tsv_graph_free(h)
            except Exception:
                pass
            self._h = None

    # --- reference accessors
    def n(self) -> int:
        return self._info.n

    def t(self) -> int:
        return self._info.t

    def m(self) -> int:
        return self._info.m

    def directed(self) -> bool:
        return bool(self._info.directed)

    def dropped_self_loops(self) -> int:
        return self._info.dropped_self_loops

    def dropped_duplicates(self) -> int:
        return self._info.dropped_duplicates

    def edges(self):
        """Canonical (u, v, ts) arrays; edge id = index."""
        if self._edges is None:
            m = max(self.m(), 1)
            u, v, ts = (np.zeros(m, np.int32) for _ in range(3))
            _native.check(_native.lib().tsv_graph_edges(self._h, u, v, ts))
            self._edges = (u[:self.m()], v[:self.m()], ts[:self.m()])
        return self._edges

    def static_projection(self):
        """The static projection grouped on the device (tsv_graph_static_edges,
        graph.cpp:148-199 of the reference): (a, b, back_off, back) -- the
        distinct (a, b) pairs ascending (a < b when undirected) and, per pair,
        its temporal edge ids in increasing order."""
        m = max(self.m(), 1)
        a, b, back = (np.zeros(m, np.int32) for _ in range(3))
        off = np.zeros(m + 1, np.int32)
        ms = C.c_int64(0)
        _native.check(_native.lib().tsv_graph_static_edges(self._h, C.byref(ms), a, b, off, back))
        s = ms.value
        return a[:s], b[:s], off[:s + 1], back[:self.m()]

    @property
    def info(self) -> _native.GraphInfo:
        return self._info

    @property
    def handle(self):
        return self._h


def _edge_arrays(edges):
    if isinstance(edges, tuple) and len(edges) == 3:
        u, v, ts = edges
    else:
        arr = np.asarray(edges, dtype=np.int64).reshape(-1, 3) if len(edges) else \
            np.zeros((0, 3), np.int64)
        u, v, ts = arr[:, 0], arr[:, 1], arr[:, 2]
    u = np.ascontiguousarray(u, dtype=np.int32)
    v = np.ascontiguousarray(v, dtype=np.int32)
    ts = np.ascontiguousarray(ts, dtype=np.int32)
    if not (len(u) == len(v) == len(ts)):
        raise ValueError("edge arrays differ in length")
    return u, v, ts


class VertexColoring:
    """Vertex colors in [1..q] (graph.hpp:114-139; no wildcard extension)."""

    def __init__(self, primary, q: int):
        self._p = np.ascontiguousarray(primary, dtype=np.int32)
        self._q = int(q)
        if len(self._p) and (self._p.min() < 1 or self._p.max() > self._q):
            raise ValueError("vertex color outside [1..q]")

    @staticmethod
    def uniform(n: int, c: int = 1) -> "VertexColoring":
        return VertexColoring(np.full(n, c, np.int32), c)

    def n(self) -> int:
        return len(self._p)

    def q(self) -> int:
        return self._q

    def primary(self, u: int) -> int:
        return int(self._p[u])

    def primaries(self) -> np.ndarray:
        return self._p


@dataclass
class MotifQuery:
    """motif.hpp:24-74 (size-only and color-multiset kinds)."""

    kind: str = "size_only"
    k: int = 0
    multiset: dict = field(default_factory=dict)   # color -> multiplicity, ascending

    @staticmethod
    def size_only(k: int) -> "MotifQuery":
        return MotifQuery("size_only", int(k), {})

    @staticmethod
    def from_multiset(colors) -> "MotifQuery":
        ms: dict[int, int] = {}
        for c in colors:
            ms[int(c)] = ms.get(int(c), 0) + 1
        return MotifQuery("multiset", len(list(colors)), dict(sorted(ms.items())))


@dataclass
class LoadResult:
    graph: TemporalGraph
    coloring: VertexColoring
    vertex_names: list
    raw_records: int = 0
    self_loops_dropped: int = 0
    duplicates_dropped: int = 0


def _records(text: str):
    for lineno, raw in enumerate(text.splitlines(), start=1):
        pos = raw.find("#")
        if pos >= 0:
            raw = raw[:pos]
        tok = raw.split()
        if tok:
            yield lineno, tok


def _parse_int(tok: str, lineno: int) -> int:
    try:
        s = tok.strip()
        if s != tok or not s or not (s.lstrip("+-").isdigit()):
            raise ValueError
        return int(s)
    except ValueError:
        raise RuntimeError(f"line {lineno}: malformed integer '{tok}'") from None


def parse_graph_text(edge_text, color_text=None):
    """Host half of load_graph (graph.cpp:376-448): first-appearance vertex
    interning (u then v per line), timestamps replaced by their dense rank
    1..t, colors default 1 with unknown tokens skipped, q = max color.
    Returns (n, u, v, ts, t, colors, q, names, records)."""
    if hasattr(edge_text, "read"):
        edge_text = edge_text.read()
    if color_text is not None and hasattr(color_text, "read"):
        color_text = color_text.read()
    ids: dict[str, int] = {}
    names: list[str] = []

    def intern(tok):
        x = ids.get(tok)
        if x is None:
            x = len(names)
            ids[tok] = x
            names.append(tok)
        return x

    us, vs, raw_ts = [], [], []
    records = 0
    for lineno, tok in _records(edge_text):
        if len(tok) not in (3, 4):
            raise RuntimeError(f"line {lineno}: expected 'u v ts' (optionally 'u v ts eps')")
        records += 1
        us.append(intern(tok[0]))
        vs.append(intern(tok[1]))
        tsv = _parse_int(tok[2], lineno)
        if tsv < 0:
            raise RuntimeError(f"line {lineno}: negative timestamp")
        if len(tok) == 4:
            e = _parse_int(tok[3], lineno)
            if e < 1:
                raise RuntimeError(f"line {lineno}: transition time below 1")
            if e != 1:
                raise ValueError("transition times (4th column) need a delay edge model, "
                                 "which the B200 engine does not evaluate")
        raw_ts.append(tsv)
    stamps = np.unique(np.asarray(raw_ts, dtype=np.int64))
    ranks = (np.searchsorted(stamps, np.asarray(raw_ts, dtype=np.int64)) + 1).astype(np.int32)
    n = len(names)
    colors = np.ones(n, np.int32)
    q = 1
    if color_text is not None:
        for lineno, tok in _records(color_text):
            if len(tok) != 2:
                raise RuntimeError(f"line {lineno}: expected 'u c'")
            x = ids.get(tok[0])
            if x is None:
                continue
            c = _parse_int(tok[1], lineno)
            if c < 1:
                raise RuntimeError(f"line {lineno}: color below 1")
            colors[x] = c
            q = max(q, c)
    return (n, np.asarray(us, np.int32), np.asarray(vs, np.int32), ranks, int(len(stamps)),
            colors, q, names, records)


def load_graph(edge_text, color_text=None, directed: bool = False, device: int = 0) -> LoadResult:
    """load_graph (graph.cpp:376-448); the graph is built on ``device``."""
    n, u, v, ts, t, colors, q, names, records = parse_graph_text(edge_text, color_text)
    g = TemporalGraph.build(n, (u, v, ts), directed, t, device)
    return LoadResult(g, VertexColoring(colors, q), names, records, g.dropped_self_loops(),
                      g.dropped_duplicates())


def restrict_to(g: TemporalGraph, keep_vertex, max_ts: int, device: int | None = None
                ) -> TemporalGraph:
    """Induced subgraph with ts <= max_ts (graph.cpp:483-494): kept edges keep
    their relative order, so the rebuild renumbers edge id = rank among them."""
    keep = np.ascontiguousarray(np.asarray(keep_vertex, dtype=bool).astype(np.uint8))
    if device is None or device == g.info.device:
        # order-preserving filter + rebuild on the graph's device
        h = C.c_void_p()
        _native.check(_native.lib().tsv_graph_restrict(
            g.handle, keep if len(keep) else np.zeros(1, np.uint8), int(max_ts), C.byref(h)))
        info = _native.GraphInfo()
        _native.check(_native.lib().tsv_graph_get_info(h, C.byref(info)))
        return TemporalGraph(h, info)
    u, v, ts = g.edges()
    sel = (ts <= max_ts) & keep.astype(bool)[u] & keep.astype(bool)[v]
    return TemporalGraph.build(g.n(), (u[sel], v[sel], ts[sel]), g.directed(),
                               min(int(max_ts), g.t()), device)


def save_graph(g: TemporalGraph) -> str:
    u, v, ts = g.edges()
    return "".join(f"{a} {b} {c}\n" for a, b, c in zip(u.tolist(), v.tolist(), ts.tolist()))


def save_colors(col: VertexColoring) -> str:
    return "".join(f"{i} {c}\n" for i, c in enumerate(col.primaries().tolist()))

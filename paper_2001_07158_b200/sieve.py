"""The temporal sieve -- Python mirror of tsieve/sieve.hpp on the B200 engine.

Reference: /root/reference/proj/core/include/tsieve/sieve.hpp
  SieveConfig :24-32, ShadeAssignment :39-56, build_shades :61-63,
  SieveOutcome :65-72, AnchorSpec :76-79, eval_temporal_sieve :84-87,
  false_negative_bound :122.
``eval_temporal_sieve`` calls ``tsv_eval_temporal_sieve`` (include/tsv.h);
there is no host fallback.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .graph import MotifQuery, TemporalGraph, VertexColoring


# EdgeModel (graph.hpp:179) -> tsv_config.edge_model; the graph must be
# built for the same model (TemporalGraph.build_model)
EDGE_MODELS = {"instant": 0, "transition": 1, "delay": 2, "transition_delay": 3}


@dataclass
class SieveConfig:
    seed: int = 1
    field_bits: int = 64
    lane_width: int = 8          # accepted; results do not depend on it
    threads: int = 1             # accepted; the GPU grid replaces OpenMP
    localize: bool = True
    edge_model: str = "instant"
    memory_cap_words: int = 1 << 31
    points_per_batch: int = 0    # engine knob: sieve points per device batch (0 = auto)

    def to_native(self) -> _native.Config:
        if self.threads < 1:
            raise ValueError("threads must be >= 1")
        if self.edge_model not in EDGE_MODELS:
            raise ValueError(f"unknown edge model {self.edge_model!r}")
        c = _native.Config()
        c.seed = self.seed & (2**64 - 1)
        c.field_bits = self.field_bits
        c.lane_width = self.lane_width
        c.edge_model = EDGE_MODELS[self.edge_model]
        c.points_per_batch = self.points_per_batch
        c.memory_cap_words = min(int(self.memory_cap_words), 2**64 - 1)
        return c


@dataclass
class ShadeAssignment:
    k: int = 0
    seed: int = 0
    feasible: bool = True
    missing_color: int = 0
    colors: list = field(default_factory=list)
    shade_sets: list = field(default_factory=list)
    vertex_off: np.ndarray = field(default_factory=lambda: np.zeros(1, np.int32))
    vertex_shades: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))

    def shades_of(self, u: int) -> np.ndarray:
        return self.vertex_shades[self.vertex_off[u]:self.vertex_off[u + 1]]


@dataclass
class AnchorSpec:
    source: int = -1
    sink: int = -1


@dataclass
class SieveOutcome:
    global_nonzero: bool = False
    accumulators: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint64))
    flagged: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    fn_bound: float = 0.0
    peak_field_words: int = 0
    checksum: int = 0


def false_negative_bound(k: int, field_bits: int) -> float:
    return (2.0 * k - 1.0) / (2.0 ** field_bits)


def _validate(cfg: SieveConfig):
    if cfg.field_bits not in (8, 16, 32, 64):
        raise ValueError("field_bits must be 8, 16, 32 or 64")
    w = cfg.lane_width
    if w < 1 or w > 256 or (w & (w - 1)):
        raise ValueError("lane_width must be a power of two in [1,256]")
    if cfg.threads < 1:
        raise ValueError("threads must be >= 1")


def build_shades(query: MotifQuery, coloring: VertexColoring, config: SieveConfig
                 ) -> ShadeAssignment:
    """Canonical disjoint shades (sieve.cpp:658-718): ascending shade ids
    1..k to ascending query colors, mu(c) shades per color c."""
    _validate(config)
    if not query.multiset:
        raise ValueError("build_shades needs a color multiset")
    if sum(query.multiset.values()) != query.k:
        raise ValueError("multiset multiplicities do not sum to k")
    sh = ShadeAssignment(k=query.k, seed=config.seed)
    prim = coloring.primaries()
    counts = np.bincount(prim, minlength=coloring.q() + 2) if len(prim) else \
        np.zeros(coloring.q() + 2, np.int64)
    nxt = 1
    for c, mu in sorted(query.multiset.items()):
        sh.colors.append(c)
        sh.shade_sets.append(list(range(nxt, nxt + mu)))
        nxt += mu
        present = 1 <= c < len(counts) and counts[c] > 0
        if not present and sh.feasible:
            sh.feasible = False
            sh.missing_color = c
    n = len(prim)
    # per-color shade lists -> per-vertex CSR
    cnt = np.zeros(n, np.int32)
    table = {c: s for c, s in zip(sh.colors, sh.shade_sets)}
    for c, s in table.items():
        cnt[prim == c] = len(s)
    off = np.zeros(n + 1, np.int32)
    np.cumsum(cnt, out=off[1:])
    shades = np.zeros(int(off[-1]), np.int32)
    for c, s in table.items():
        idx = np.nonzero(prim == c)[0]
        if len(idx) == 0:
            continue
        base = off[idx]
        for i, d in enumerate(s):
            shades[base + i] = d
    sh.vertex_off = off
    sh.vertex_shades = shades
    return sh


def eval_temporal_sieve(g: TemporalGraph, k: int, max_ts: int, shades: ShadeAssignment,
                        config: SieveConfig, anchor: AnchorSpec | None = None
                        ) -> SieveOutcome:
    """eval_temporal_sieve (sieve.cpp:720-732) on the B200 engine."""
    anchor = anchor or AnchorSpec()
    _validate(config)
    if max_ts < 1 or max_ts > g.t():
        raise ValueError("max_ts outside [1..t]")
    if len(shades.vertex_off) != g.n() + 1:
        raise ValueError("shade assignment built for a different graph")
    cfg = config.to_native()
    n = g.n()
    acc = np.zeros(max(n, 1), np.uint64)
    out = _native.Outcome()
    vs = shades.vertex_shades if len(shades.vertex_shades) else np.zeros(1, np.int32)
    _native.check(_native.lib().tsv_eval_temporal_sieve(
        g.handle, int(k), int(max_ts), np.ascontiguousarray(shades.vertex_off, np.int32),
        np.ascontiguousarray(vs, np.int32), C.byref(cfg), int(anchor.source),
        int(anchor.sink), acc, C.byref(out)))
    acc = acc[:n]
    res = SieveOutcome()
    res.accumulators = acc
    res.flagged = _native.nonzero_index(acc)
    if config.localize:
        res.global_nonzero = len(res.flagged) > 0
    else:
        tot = np.bitwise_xor.reduce(acc) if n else np.uint64(0)
        res.global_nonzero = bool(tot != 0)
    res.fn_bound = false_negative_bound(k, config.field_bits)
    res.peak_field_words = int(out.peak_field_words)
    res.checksum = int(out.checksum)
    return res


class DeviceShades:
    """Shade CSR resident on the graph's device (tsv_shades_upload)."""

    def __init__(self, g: TemporalGraph, k: int, shades: ShadeAssignment):
        h = C.c_void_p()
        vs = shades.vertex_shades if len(shades.vertex_shades) else np.zeros(1, np.int32)
        _native.check(_native.lib().tsv_shades_upload(
            g.handle, int(k), np.ascontiguousarray(shades.vertex_off, np.int32),
            np.ascontiguousarray(vs, np.int32), C.byref(h)))
        self.handle = h

    def __del__(self):
        if getattr(self, "handle", None):
            try:
                _native.lib().tsv_shades_free(self.handle)
            except Exception:
                pass
            self.handle = None


def eval_points_device(g: TemporalGraph, dshades: DeviceShades, k: int, max_ts: int,
                       config: SieveConfig, anchor_source: int, p_begin: int, p_end: int,
                       d_acc_ptr: int, stream_ptr: int = 0) -> None:
    """XOR sieve points [p_begin, p_end) into a device buffer (no host copies)."""
    cfg = config.to_native()
    _native.check(_native.lib().tsv_eval_points_device(
        g.handle, dshades.handle, int(k), int(max_ts), C.byref(cfg), int(anchor_source),
        int(p_begin), int(p_end), C.c_void_p(d_acc_ptr), C.c_void_p(stream_ptr)))


def xor_combine_device(d_parts_ptr: int, nparts: int, n: int, d_out_ptr: int,
                       stream_ptr: int = 0) -> None:
    _native.check(_native.lib().tsv_xor_combine_device(
        C.c_void_p(d_parts_ptr), int(nparts), int(n), C.c_void_p(d_out_ptr),
        C.c_void_p(stream_ptr)))


def finalize(acc: np.ndarray, sink: int = -1):
    """(accumulators, flagged count, checksum) per sieve.cpp:136-159."""
    a = np.ascontiguousarray(acc, dtype=np.uint64).copy()
    out = _native.Outcome()
    _native.check(_native.lib().tsv_finalize(len(a), a if len(a) else np.zeros(1, np.uint64),
                                             int(sink), C.byref(out)))
    return a, int(out.flagged), int(out.checksum)


def vertex_partition(g: TemporalGraph, dshades: DeviceShades, k: int, rank: int = 0,
                     world: int = 1) -> _native.Partition:
    """tsv_vertex_partition: this rank's state-row range of the vertex-
    partitioned evaluation (applicable = 0: use point sharding)."""
    out = _native.Partition()
    _native.check(_native.lib().tsv_vertex_partition(g.handle, dshades.handle, int(k), int(rank),
                                                     int(world), C.byref(out)))
    return out


def eval_vertex_level(g: TemporalGraph, dshades: DeviceShades, k: int, level: int, max_ts: int,
                      config: SieveConfig, anchor_source: int, rank: int, world: int,
                      d_prev: int, d_cur: int, d_acc: int, stream_ptr: int = 0,
                      peer_cur=None) -> None:
    """tsv_eval_vertex_level: level `level` of this rank's vertices.  With
    peer_cur (the `world` ranks' level buffers as device pointers valid on
    this GPU) the rows are also stored into the buffers of the ranks that
    read them (tsv_eval_vertex_level_peer: the exchange inside the kernel)."""
    cfg = config.to_native()
    if peer_cur is not None:
        ptrs = (C.c_void_p * int(world))(*[C.c_void_p(int(x) if x else None) for x in peer_cur])
        _native.check(_native.lib().tsv_eval_vertex_level_peer(
            g.handle, dshades.handle, int(k), int(level), int(max_ts), C.byref(cfg),
            int(anchor_source), int(rank), int(world), C.c_void_p(d_prev), C.c_void_p(d_cur),
            C.c_void_p(d_acc), ptrs, C.c_void_p(stream_ptr)))
        return
    _native.check(_native.lib().tsv_eval_vertex_level(
        g.handle, dshades.handle, int(k), int(level), int(max_ts), C.byref(cfg),
        int(anchor_source), int(rank), int(world), C.c_void_p(d_prev), C.c_void_p(d_cur),
        C.c_void_p(d_acc), C.c_void_p(stream_ptr)))


def vertex_exchange_plan(g: TemporalGraph, dshades: DeviceShades, k: int, rank: int,
                         world: int) -> _native.Exchange:
    """tsv_vertex_exchange_plan: rows this rank sends to / receives from each peer."""
    out = _native.Exchange()
    _native.check(_native.lib().tsv_vertex_exchange_plan(g.handle, dshades.handle, int(k),
                                                         int(rank), int(world), C.byref(out)))
    return out


def vertex_exchange_move(g: TemporalGraph, rank: int, world: int, row_words: int, src: int,
                         dst: int, pack: bool, stream_ptr: int = 0) -> None:
    """tsv_vertex_exchange_pack (rows -> send buffer) / _unpack (receive buffer -> rows)."""
    f = _native.lib().tsv_vertex_exchange_pack if pack else _native.lib().tsv_vertex_exchange_unpack
    _native.check(f(g.handle, int(rank), int(world), int(row_words), C.c_void_p(src),
                    C.c_void_p(dst), C.c_void_p(stream_ptr)))

"""ctypes front end of the parity checkers -- TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` legs may import this module.  The product package
(``paper_2001_07158_b200``) never imports it.

Two checkers live behind it:

* ``liboracle.so`` -- our plain-C restatement of the hot path
  (oracle/tsv_oracle.c, citing /root/reference/proj file:line per function);
* ``_ref/libtsieve_ref.so`` -- the unmodified reference core compiled in place
  by oracle/Makefile, driven through our own shim (oracle/ref_shim.cpp).
"""
from __future__ import annotations

import ctypes as C
import json
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libtsieve_ref.so")

_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")

_oracle = None
_ref = None


def build():
    """Compile the checkers (the reference only where its sources exist)."""
    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)


def oracle_lib():
    global _oracle
    if _oracle is None:
        if not os.path.exists(ORACLE_SO):
            build()
        lib = C.CDLL(ORACLE_SO)
        lib.tsvo_gf_mul.restype = C.c_uint64
        lib.tsvo_gf_mul.argtypes = [C.c_uint64, C.c_uint64]
        lib.tsvo_gf_mul_slow.restype = C.c_uint64
        lib.tsvo_gf_mul_slow.argtypes = [C.c_uint64, C.c_uint64]
        lib.tsvo_draw_nonzero.restype = C.c_uint64
        lib.tsvo_draw_nonzero.argtypes = [C.c_uint64] * 5
        lib.tsvo_draw64.restype = C.c_uint64
        lib.tsvo_draw64.argtypes = [C.c_uint64] * 5
        lib.tsvo_canonical_edges.restype = C.c_int64
        lib.tsvo_canonical_edges.argtypes = [C.c_int32, C.c_int64, _i32p, _i32p, _i32p,
                                             C.c_int, _i32p, _i32p, _i32p]
        lib.tsvo_eval_points.restype = C.c_int
        lib.tsvo_eval_points.argtypes = [C.c_int32, C.c_int64, _i32p, _i32p, _i32p, C.c_int,
                                         C.c_int, C.c_int32, _i32p, _i32p, C.c_uint64,
                                         C.c_int32, C.c_uint64, C.c_uint64, _u64p]
        lib.tsvo_canonicalize_inplace.restype = C.c_int64
        lib.tsvo_canonicalize_inplace.argtypes = [C.c_int32, C.c_int64, _i32p, _i32p, _i32p,
                                                  C.c_int]
        lib.tsvo_big_build.restype = C.c_void_p
        lib.tsvo_big_build.argtypes = [C.c_int32, C.c_int64, _i32p, _i32p, _i32p, C.c_int,
                                       C.c_int32]
        lib.tsvo_big_free.restype = None
        lib.tsvo_big_free.argtypes = [C.c_void_p]
        lib.tsvo_big_arcs.restype = C.c_int64
        lib.tsvo_big_arcs.argtypes = [C.c_void_p]
        lib.tsvo_big_runs.restype = C.c_int64
        lib.tsvo_big_runs.argtypes = [C.c_void_p]
        lib.tsvo_big_eval.restype = C.c_int
        lib.tsvo_big_eval.argtypes = [C.c_void_p, C.c_int, _i32p, _i32p, C.c_uint64, C.c_int32,
                                      C.c_uint64, C.c_uint64, C.c_int, _u64p]
        lib.tsvo_big_level.restype = C.c_int
        lib.tsvo_big_level.argtypes = [C.c_void_p, C.c_int, C.c_int, _i32p, _i32p, C.c_uint64,
                                       C.c_int32, C.c_uint64, C.c_int, C.c_int64, C.c_int64,
                                       C.c_void_p, C.c_void_p, _u64p]
        lib.tsvo_big_run_range.restype = None
        lib.tsvo_big_run_range.argtypes = [C.c_void_p, C.c_int64, C.c_int64,
                                           C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        lib.tsvo_set_threads.restype = None
        lib.tsvo_set_threads.argtypes = [C.c_int]
        lib.tsvo_max_threads.restype = C.c_int
        lib.tsvo_finalize.restype = C.c_int64
        lib.tsvo_finalize.argtypes = [C.c_int32, _u64p, C.c_int32, C.POINTER(C.c_uint64)]
        _oracle = lib
    return _oracle


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref_lib():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise RuntimeError("oracle/_ref/libtsieve_ref.so not built (needs /root/reference)")
        lib = C.CDLL(REF_SO)
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_gf_mul.restype = C.c_uint64
        lib.ref_gf_mul.argtypes = [C.c_uint64, C.c_uint64]
        lib.ref_draw_nonzero.restype = C.c_uint64
        lib.ref_draw_nonzero.argtypes = [C.c_uint64] * 5
        lib.ref_canonical_edges.restype = C.c_int64
        lib.ref_canonical_edges.argtypes = [C.c_int32, C.c_int64, _i32p, _i32p, _i32p, C.c_int,
                                            _i32p, _i32p, _i32p]
        lib.ref_build_shades.restype = C.c_int64
        lib.ref_build_shades.argtypes = [C.c_int32, _i32p, _i32p, C.c_int32, C.c_uint64,
                                         _i32p, _i32p, C.c_int64]
        lib.ref_eval_temporal.restype = C.c_double
        lib.ref_eval_temporal.argtypes = [C.c_int32, C.c_int64, _i32p, _i32p, _i32p, C.c_int,
                                          C.c_int32, _i32p, _i32p, C.c_int32, C.c_int32,
                                          C.c_uint64, C.c_int32, C.c_int32, C.c_int32,
                                          C.c_int32, C.c_int32, _u64p,
                                          C.POINTER(C.c_uint64), C.POINTER(C.c_int64),
                                          C.POINTER(C.c_int32)]
        lib.ref_eval_temporal_model.restype = C.c_int64
        lib.ref_eval_temporal_model.argtypes = [
            C.c_int32, C.c_int64, _i32p, _i32p, _i32p, C.c_void_p, C.c_void_p, C.c_int,
            C.c_int32, _i32p, _i32p, C.c_int32, C.c_int32, C.c_uint64, C.c_int32, C.c_int32,
            C.c_int32, C.c_int32, _u64p, C.POINTER(C.c_uint64), _i32p, _i32p, _i32p, _i32p]
        lib.ref_set_query.restype = None
        lib.ref_set_query.argtypes = [C.c_void_p, C.c_int32, C.c_void_p, C.c_int32]
        lib.ref_set_model.restype = None
        lib.ref_set_model.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_int32, C.c_int32]
        lib.ref_solve.restype = C.c_int64
        lib.ref_solve.argtypes = [C.c_int32, C.c_int64, _i32p, _i32p, _i32p, C.c_int, C.c_int32,
                                  _i32p, C.c_char_p, _i32p, C.c_int32, C.c_int32, C.c_int32,
                                  C.c_int32, C.c_uint64, C.c_int32, C.c_int32, C.c_int32,
                                  C.c_char_p, C.c_int64]
        lib.ref_load_graph.restype = C.c_int64
        lib.ref_load_graph.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.POINTER(C.c_int32),
                                       C.POINTER(C.c_int32), _i32p, _i32p, _i32p, C.c_int64,
                                       _i32p, C.c_int32, C.c_char_p, C.c_int64]
        _ref = lib
    return _ref


def _a32(x):
    return np.ascontiguousarray(np.asarray(x, dtype=np.int32))


# ----------------------------------------------------------------- oracle


def gf_mul(a: int, b: int) -> int:
    return oracle_lib().tsvo_gf_mul(a, b)


def gf_mul_slow(a: int, b: int) -> int:
    return oracle_lib().tsvo_gf_mul_slow(a, b)


def draw_nonzero(seed, role, a, b, c=0) -> int:
    return oracle_lib().tsvo_draw_nonzero(seed, role, a, b, c)


def canonical_edges(n, u, v, ts, directed):
    u, v, ts = _a32(u), _a32(v), _a32(ts)
    m = len(u)
    ou, ov, ot = (np.empty(max(m, 1), np.int32) for _ in range(3))
    w = oracle_lib().tsvo_canonical_edges(n, m, u, v, ts, int(directed), ou, ov, ot)
    if w < 0:
        raise ValueError("edge endpoint or timestamp out of range")
    return ou[:w].copy(), ov[:w].copy(), ot[:w].copy()


def eval_points(n, cu, cv, cts, directed, k, max_ts, vertex_off, vertex_shades, seed,
                anchor_source=-1, p_begin=0, p_end=None):
    """XOR of sieve points [p_begin, p_end) over canonical edges (no finalize)."""
    if p_end is None:
        p_end = 1 << k
    acc = np.zeros(max(n, 1), np.uint64)
    cu, cv, cts = _a32(cu), _a32(cv), _a32(cts)
    vs = _a32(vertex_shades) if len(vertex_shades) else np.zeros(1, np.int32)
    rc = oracle_lib().tsvo_eval_points(n, len(cu), cu, cv, cts, int(directed), k, max_ts,
                                       _a32(vertex_off), vs, seed, anchor_source,
                                       p_begin, p_end, acc)
    if rc != 0:
        raise ValueError("k out of range [1,30]")
    return acc[:n]


def canonicalize_inplace(n, u, v, ts, directed) -> int:
    """Canonical edges (graph.cpp:14-43) written into u/v/ts[0:return] in place
    (int32 arrays, modified).  Multi-threaded; for the BASELINE sizes."""
    for a in (u, v, ts):
        if a.dtype != np.int32 or not a.flags.c_contiguous:
            raise TypeError("canonicalize_inplace needs contiguous int32 arrays")
    w = oracle_lib().tsvo_canonicalize_inplace(n, len(u), u, v, ts, int(directed))
    if w == -1:
        raise ValueError("edge endpoint or timestamp out of range")
    if w < 0:
        raise ValueError("timestamps too large for the bucket sort")
    return int(w)


class BigGraph:
    """Head-grouped arcs/runs of CANONICAL edges for tsvo_big_eval
    (oracle/tsv_oracle_big.c).  The edge arrays are not referenced after
    construction, so a caller may free them."""

    def __init__(self, n, cu, cv, cts, directed, max_ts):
        self.n = int(n)
        self.h = oracle_lib().tsvo_big_build(n, len(cu), _a32(cu), _a32(cv), _a32(cts),
                                             int(directed), int(max_ts))
        if not self.h:
            raise ValueError("too many arcs for the oracle's 32-bit indices")
        self.arcs = oracle_lib().tsvo_big_arcs(self.h)
        self.runs = oracle_lib().tsvo_big_runs(self.h)

    def eval(self, k, vertex_off, vertex_shades, seed, anchor_source=-1, p_begin=0,
             p_end=None, lanes=8, out=None):
        """XOR of sieve points [p_begin, p_end) into `out` (fresh zeros if None)."""
        if p_end is None:
            p_end = 1 << k
        acc = np.zeros(max(self.n, 1), np.uint64) if out is None else out
        vs = _a32(vertex_shades) if len(vertex_shades) else np.zeros(1, np.int32)
        rc = oracle_lib().tsvo_big_eval(self.h, k, _a32(vertex_off), vs, seed, anchor_source,
                                        p_begin, p_end, lanes, acc)
        if rc == -3:
            raise MemoryError("oracle sieve state does not fit in host memory")
        if rc != 0:
            raise ValueError("k out of range [1,30] or bad lane count")
        return acc[:self.n]

    def run_range(self, v_lo, v_hi):
        """Run-state indices [r_lo, r_hi) of the heads [v_lo, v_hi)."""
        a, b = C.c_int64(0), C.c_int64(0)
        oracle_lib().tsvo_big_run_range(self.h, int(v_lo), int(v_hi), C.byref(a), C.byref(b))
        return a.value, b.value

    def level(self, k, ell, vertex_off, vertex_shades, seed, anchor_source, p_begin, lanes,
              v_lo, v_hi, prev, cur, acc):
        """Level ell for heads [v_lo, v_hi), points [p_begin, p_begin+lanes):
        prev/cur are uint64 run-state arrays (runs x lanes), acc n words."""
        vs = _a32(vertex_shades) if len(vertex_shades) else np.zeros(1, np.int32)
        rc = oracle_lib().tsvo_big_level(self.h, k, ell, _a32(vertex_off), vs, seed,
                                         anchor_source, p_begin, lanes, int(v_lo), int(v_hi),
                                         prev.ctypes.data, cur.ctypes.data, acc)
        if rc != 0:
            raise ValueError("bad level arguments")

    def close(self):
        if self.h:
            oracle_lib().tsvo_big_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def set_threads(t: int):
    oracle_lib().tsvo_set_threads(int(t))


def max_threads() -> int:
    return int(oracle_lib().tsvo_max_threads())


def finalize(acc, anchor_sink=-1):
    acc = np.ascontiguousarray(acc, dtype=np.uint64).copy()
    cs = C.c_uint64(0)
    nflag = oracle_lib().tsvo_finalize(len(acc), acc if len(acc) else np.zeros(1, np.uint64),
                                       anchor_sink, C.byref(cs))
    return acc, int(nflag), int(cs.value)


def oracle_eval(n, cu, cv, cts, directed, k, max_ts, vertex_off, vertex_shades, seed,
                anchor=(-1, -1)):
    """Full oracle: (accumulators, flagged count, checksum) like SieveOutcome."""
    acc = eval_points(n, cu, cv, cts, directed, k, max_ts, vertex_off, vertex_shades, seed,
                      anchor[0])
    return finalize(acc, anchor[1])


# -------------------------------------------------------------- reference


def ref_canonical_edges(n, u, v, ts, directed):
    u, v, ts = _a32(u), _a32(v), _a32(ts)
    m = len(u)
    ou, ov, ot = (np.empty(max(m, 1), np.int32) for _ in range(3))
    w = ref_lib().ref_canonical_edges(n, m, u, v, ts, int(directed), ou, ov, ot)
    if w < 0:
        raise ValueError(ref_lib().ref_last_error().decode())
    return ou[:w].copy(), ov[:w].copy(), ot[:w].copy()


def ref_build_shades(n, colors, motif, seed=1):
    off = np.zeros(n + 1, np.int32)
    cap = n * len(motif) + 1
    vs = np.zeros(cap, np.int32)
    cnt = ref_lib().ref_build_shades(n, _a32(colors), _a32(motif), len(motif), seed, off, vs,
                                     cap)
    if cnt == -2:
        return None
    if cnt < 0:
        raise ValueError(ref_lib().ref_last_error().decode())
    return off, vs[:cnt].copy()


def ref_eval(n, u, v, ts, directed, colors, motif, max_ts=0, seed=1, lanes=8, threads=1,
             anchor=(-1, -1), t=0, repeats=1, field_bits=64):
    """Reference eval_temporal_sieve on raw edges.  Returns dict or None (infeasible)."""
    u, v, ts = _a32(u), _a32(v), _a32(ts)
    ref_lib().ref_set_field_bits(int(field_bits))
    acc = np.zeros(max(n, 1), np.uint64)
    cs, nf, gl = C.c_uint64(0), C.c_int64(0), C.c_int32(0)
    sec = ref_lib().ref_eval_temporal(n, len(u), u, v, ts, int(directed), t, _a32(colors),
                                      _a32(motif), len(motif), max_ts, seed, lanes, threads,
                                      anchor[0], anchor[1], repeats, acc, C.byref(cs),
                                      C.byref(nf), C.byref(gl))
    if sec == -2:
        return None
    if sec < 0:
        raise ValueError(ref_lib().ref_last_error().decode())
    return {"acc": acc[:n], "checksum": int(cs.value), "nflagged": int(nf.value),
            "global": bool(gl.value), "seconds": sec}


def ref_eval_temporal_model(n, u, v, ts, eps, delays, directed, colors, motif, edge_model,
                            seed=1, max_ts=0, lanes=8, anchor=(-1, -1), t=0):
    """The reference's eval_temporal_sieve under an edge model (sieve.cpp:257-291).
    Returns None when the query is infeasible, else accumulators, checksum and
    the canonical edges (with transition times) of the reference's build."""
    u, v, ts = _a32(u), _a32(v), _a32(ts)
    m = len(u)
    eps_a = _a32(eps) if eps is not None else None
    del_a = _a32(delays) if delays is not None else None
    acc = np.zeros(max(n, 1), np.uint64)
    cs = C.c_uint64(0)
    ou, ov, ot, oe = (np.zeros(max(m, 1), np.int32) for _ in range(4))
    r = ref_lib().ref_eval_temporal_model(
        n, m, u, v, ts, None if eps_a is None else eps_a.ctypes.data,
        None if del_a is None else del_a.ctypes.data, int(directed), t, _a32(colors),
        _a32(motif), len(motif), max_ts, seed, lanes, edge_model, anchor[0], anchor[1], acc,
        C.byref(cs), ou, ov, ot, oe)
    if r == -2:
        return None
    if r < 0:
        raise ValueError(ref_lib().ref_last_error().decode())
    return {"acc": acc[:n], "checksum": int(cs.value), "u": ou[:r], "v": ov[:r], "ts": ot[:r],
            "eps": oe[:r]}


def ref_solve_query(n, u, v, ts, times, order, *args, **kw):
    """ref_solve with a timed (EC) or ordered (VC) query."""
    t = _a32(times) if times else None
    o = _a32(order) if order else None
    ref_lib().ref_set_query(None if t is None else t.ctypes.data, 0 if t is None else len(t),
                            None if o is None else o.ctypes.data, 0 if o is None else len(o))
    try:
        return ref_solve(n, u, v, ts, *args, **kw)
    finally:
        ref_lib().ref_set_query(None, 0, None, 0)


def ref_solve_model(n, u, v, ts, eps, delays, edge_model, *args, **kw):
    """ref_solve with transition times / vertex delays under an edge model."""
    e = _a32(eps) if eps is not None else None
    d = _a32(delays) if delays is not None else None
    ref_lib().ref_set_model(None if e is None else e.ctypes.data, 0 if e is None else len(e),
                            None if d is None else d.ctypes.data, 0 if d is None else len(d),
                            int(edge_model))
    try:
        return ref_solve(n, u, v, ts, *args, **kw)
    finally:
        ref_lib().ref_set_model(None, 0, None, 0, 0)


def ref_solve(n, u, v, ts, directed, colors, problem, motif=(), k=0, source=-1, dest=-1,
              seed=1, mode=0, extraction=0, preprocess=0, t=0, field_bits=64):
    u, v, ts = _a32(u), _a32(v), _a32(ts)
    ref_lib().ref_set_field_bits(int(field_bits))
    buf = C.create_string_buffer(1 << 20)
    ml = len(motif)
    marr = _a32(motif) if ml else np.zeros(1, np.int32)
    r = ref_lib().ref_solve(n, len(u), u, v, ts, int(directed), t, _a32(colors),
                            problem.encode(), marr, ml,
                            k, source, dest, seed, mode, extraction, preprocess, buf, len(buf))
    if r < 0:
        raise ValueError(ref_lib().ref_last_error().decode())
    return json.loads(buf.value.decode())


def ref_load_graph(edge_text: str, color_text: str | None, directed: bool):
    cap = edge_text.count("\n") + 2
    ou, ov, ot = (np.empty(cap, np.int32) for _ in range(3))
    n, t = C.c_int32(0), C.c_int32(0)
    cols = np.empty(2 * cap + 2, np.int32)
    names = C.create_string_buffer(1 << 22)
    m = ref_lib().ref_load_graph(edge_text.encode(),
                                 None if color_text is None else color_text.encode(),
                                 int(directed), C.byref(n), C.byref(t), ou, ov, ot, cap, cols,
                                 len(cols), names, len(names))
    if m < 0:
        raise ValueError(ref_lib().ref_last_error().decode())
    nm = names.value.decode().split("\n") if n.value else []
    return {"n": n.value, "t": t.value, "u": ou[:m].copy(), "v": ov[:m].copy(),
            "ts": ot[:m].copy(), "colors": cols[:n.value].copy(), "names": nm}

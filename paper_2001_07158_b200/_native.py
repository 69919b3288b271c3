"""ctypes binding of libtsv.so (include/tsv.h).

The engine has no CPU fallback: if the library is missing or CUDA is absent
the calls raise.  ``lib()`` loads the in-tree build at
``paper_2001_07158_b200/lib/libtsv.so`` (``__graft_entry__.build()``).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TSV_LIB") or os.path.join(HERE, "lib", "libtsv.so")

TSV_OK, TSV_ERR_INVALID, TSV_ERR_CAP, TSV_ERR_CUDA = 0, 1, 2, 3

_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")


class GraphInfo(C.Structure):
    _fields_ = [("n", C.c_int32), ("t", C.c_int32), ("directed", C.c_int32),
                ("device", C.c_int32), ("m", C.c_int64), ("arcs", C.c_int64),
                ("runs", C.c_int64), ("chunks", C.c_int64), ("split_chunks", C.c_int64),
                ("dropped_self_loops", C.c_int64), ("dropped_duplicates", C.c_int64),
                ("device_bytes", C.c_int64), ("arcs_with_src", C.c_int64),
                ("runs_referenced", C.c_int64)]


class Config(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("field_bits", C.c_int32), ("lane_width", C.c_int32),
                ("edge_model", C.c_int32), ("points_per_batch", C.c_int32),
                ("memory_cap_words", C.c_uint64)]


class Partition(C.Structure):
    _fields_ = [("applicable", C.c_int32), ("pad", C.c_int32), ("slot_lo", C.c_int64),
                ("slot_hi", C.c_int64), ("slots", C.c_int64), ("state_words", C.c_int64),
                ("row_words", C.c_int32 * 32)]


class Exchange(C.Structure):
    _fields_ = [("send_rows", C.c_int64 * 32), ("recv_rows", C.c_int64 * 32),
                ("send_total", C.c_int64), ("recv_total", C.c_int64)]


class Outcome(C.Structure):
    _fields_ = [("global_nonzero", C.c_int32), ("pad", C.c_int32), ("flagged", C.c_int64),
                ("checksum", C.c_uint64), ("peak_field_words", C.c_uint64),
                ("fn_bound", C.c_double)]


class EngineError(RuntimeError):
    """TSV_ERR_CUDA: device failure inside the engine."""


_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is not built; run __graft_entry__.build() "
                           "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp = C.c_void_p
    L.tsv_last_error.restype = C.c_char_p
    L.tsv_version.restype = C.c_char_p
    L.tsv_graph_build.argtypes = [C.c_int32, C.c_int64, _i32p, _i32p, _i32p, C.c_int,
                                  C.c_int32, C.c_int, C.POINTER(vp)]
    L.tsv_graph_build_model.argtypes = [C.c_int32, C.c_int64, _i32p, _i32p, _i32p, vp, vp,
                                        C.c_int, C.c_int32, C.c_int, C.c_int, C.POINTER(vp)]
    L.tsv_canonical_edges_eps.restype = C.c_int64
    L.tsv_canonical_edges_eps.argtypes = [C.c_int32, C.c_int64, _i32p, _i32p, _i32p, vp,
                                          C.c_int, _i32p, _i32p, _i32p, _i32p]
    L.tsv_canonical_edges.restype = C.c_int64
    L.tsv_canonical_edges.argtypes = [C.c_int32, C.c_int64, _i32p, _i32p, _i32p, C.c_int,
                                      _i32p, _i32p, _i32p]
    L.tsv_graph_restrict.argtypes = [vp, np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS"),
                                     C.c_int32, C.POINTER(vp)]
    L.tsv_graph_free.argtypes = [vp]
    L.tsv_graph_free.restype = None
    L.tsv_graph_get_info.argtypes = [vp, C.POINTER(GraphInfo)]
    L.tsv_graph_edges.argtypes = [vp, _i32p, _i32p, _i32p]
    L.tsv_graph_static_edges.argtypes = [vp, C.POINTER(C.c_int64), _i32p, _i32p, _i32p, _i32p]
    L.tsv_shades_upload.argtypes = [vp, C.c_int, _i32p, _i32p, C.POINTER(vp)]
    L.tsv_shades_free.argtypes = [vp]
    L.tsv_shades_free.restype = None
    L.tsv_eval_temporal_sieve.argtypes = [vp, C.c_int, C.c_int32, _i32p, _i32p,
                                          C.POINTER(Config), C.c_int32, C.c_int32, _u64p,
                                          C.POINTER(Outcome)]
    L.tsv_eval_points_device.argtypes = [vp, vp, C.c_int, C.c_int32, C.POINTER(Config),
                                         C.c_int32, C.c_uint64, C.c_uint64, vp, vp]
    L.tsv_xor_combine_device.argtypes = [vp, C.c_int, C.c_int64, vp, vp]
    L.tsv_finalize.argtypes = [C.c_int32, _u64p, C.c_int32, C.POINTER(Outcome)]
    L.tsv_eval_static_projection.argtypes = [C.c_int32, C.c_int64, _i32p, _i32p, C.c_int, C.c_int,
                                             C.c_int, _i32p, _i32p, C.POINTER(Config), C.c_int,
                                             _u64p, C.POINTER(Outcome)]
    L.tsv_vertex_partition.argtypes = [vp, vp, C.c_int, C.c_int, C.c_int, C.POINTER(Partition)]
    L.tsv_eval_vertex_level.argtypes = [vp, vp, C.c_int, C.c_int, C.c_int32, C.POINTER(Config),
                                        C.c_int32, C.c_int, C.c_int, vp, vp, vp, vp]
    L.tsv_eval_vertex_level_peer.argtypes = [vp, vp, C.c_int, C.c_int, C.c_int32,
                                             C.POINTER(Config), C.c_int32, C.c_int, C.c_int, vp,
                                             vp, vp, C.POINTER(C.c_void_p), vp]
    L.tsv_vertex_exchange_plan.argtypes = [vp, vp, C.c_int, C.c_int, C.c_int,
                                           C.POINTER(Exchange)]
    L.tsv_vertex_exchange_pack.argtypes = [vp, C.c_int, C.c_int, C.c_int, vp, vp, vp]
    L.tsv_vertex_exchange_unpack.argtypes = [vp, C.c_int, C.c_int, C.c_int, vp, vp, vp]
    L.tsv_nonzero_index.restype = C.c_int64
    L.tsv_nonzero_index.argtypes = [_u64p, C.c_int64, _i32p]
    L.tsv_finalize_device.argtypes = [vp, C.c_int64, C.c_int32, vp, C.POINTER(Outcome)]
    L.tsv_profile_enable.argtypes = [C.c_int]
    L.tsv_profile_get.argtypes = [C.c_char_p, C.POINTER(C.c_int64), C.POINTER(C.c_double)]
    L.tsv_kernel_launches.restype = C.c_int64
    L.tsv_gf_mul_device.argtypes = [C.c_int, C.c_int64, _u64p, _u64p, _u64p]
    L.tsv_gf_bench.argtypes = [C.c_int, C.c_int64, C.POINTER(C.c_double)]
    L.tsv_draw_edge_y_device.argtypes = [C.c_uint64, C.c_int32, C.c_int64, _i32p, _u64p]
    _lib = L
    return L


def check(rc: int) -> None:
    """Re-raise a status code as the reference's exception type."""
    if rc == TSV_OK:
        return
    msg = lib().tsv_last_error().decode()
    if rc == TSV_ERR_INVALID:
        raise ValueError(msg)            # std::invalid_argument
    if rc == TSV_ERR_CAP:
        raise MemoryError(msg)           # std::runtime_error (memory cap)
    raise EngineError(msg)


def canonical_edges(n, u, v, ts, directed):
    """Host-only canonical edge list of TemporalGraph::build (tsv_canonical_edges)."""
    u = np.ascontiguousarray(u, dtype=np.int32)
    v = np.ascontiguousarray(v, dtype=np.int32)
    ts = np.ascontiguousarray(ts, dtype=np.int32)
    m = len(u)
    ou, ov, ot = (np.zeros(max(m, 1), np.int32) for _ in range(3))
    w = lib().tsv_canonical_edges(int(n), m, u, v, ts, int(bool(directed)), ou, ov, ot)
    if w < 0:
        raise ValueError(lib().tsv_last_error().decode())
    return ou[:w].copy(), ov[:w].copy(), ot[:w].copy()


def canonical_edges_eps(n, u, v, ts, eps, directed):
    """tsv_canonical_edges_eps: canonical edges plus their transition times."""
    u = np.ascontiguousarray(u, dtype=np.int32)
    v = np.ascontiguousarray(v, dtype=np.int32)
    ts = np.ascontiguousarray(ts, dtype=np.int32)
    e = None if eps is None else np.ascontiguousarray(eps, dtype=np.int32)
    m = len(u)
    ou, ov, ot, oe = (np.zeros(max(m, 1), np.int32) for _ in range(4))
    w = lib().tsv_canonical_edges_eps(int(n), m, u, v, ts, None if e is None else e.ctypes.data,
                                      int(bool(directed)), ou, ov, ot, oe)
    if w < 0:
        raise ValueError(lib().tsv_last_error().decode())
    return ou[:w].copy(), ov[:w].copy(), ot[:w].copy(), oe[:w].copy()


def gf_mul_device(a, b, variant: int = 0):
    a = np.ascontiguousarray(a, dtype=np.uint64)
    b = np.ascontiguousarray(b, dtype=np.uint64)
    out = np.zeros(max(len(a), 1), np.uint64)
    check(lib().tsv_gf_mul_device(variant, len(a), a if len(a) else out, b if len(b) else out,
                                  out))
    return out[:len(a)]


def nonzero_index(acc) -> np.ndarray:
    """Ascending indices of the nonzero words (multi-threaded, libtsv)."""
    acc = np.ascontiguousarray(acc, dtype=np.uint64)
    out = np.empty(max(len(acc), 1), np.int32)
    c = lib().tsv_nonzero_index(acc if len(acc) else np.zeros(1, np.uint64), len(acc), out)
    return out[:c]


def finalize_device(d_acc_ptr: int, n: int, sink: int = -1, stream: int = 0):
    """tsv_finalize_device on a device buffer: (flagged, checksum)."""
    o = Outcome()
    check(lib().tsv_finalize_device(d_acc_ptr, int(n), int(sink), stream or None, C.byref(o)))
    return int(o.flagged), int(o.checksum)


def gf_bench(variant: int = 0, iters: int = 4096) -> float:
    r = C.c_double(0)
    check(lib().tsv_gf_bench(variant, iters, C.byref(r)))
    return r.value


def draw_edge_y_device(seed: int, level: int, edges):
    e = np.ascontiguousarray(edges, dtype=np.int32)
    out = np.zeros(max(len(e), 1), np.uint64)
    check(lib().tsv_draw_edge_y_device(seed, level, len(e), e if len(e) else
                                       np.zeros(1, np.int32), out))
    return out[:len(e)]


class Profile:
    """Per-kernel CUDA-event timing inside the engine (on its launch stream)."""

    @staticmethod
    def enable(on: bool = True):
        lib().tsv_profile_enable(1 if on else 0)

    @staticmethod
    def reset():
        lib().tsv_profile_reset()

    @staticmethod
    def get(kernel: str | None = None):
        n, ms = C.c_int64(0), C.c_double(0)
        check(lib().tsv_profile_get(None if kernel is None else kernel.encode(), C.byref(n),
                                    C.byref(ms)))
        return n.value, ms.value

    @staticmethod
    def launches() -> int:
        return int(lib().tsv_kernel_launches())

"""CPU tests of the host side: the C-ABI library loads and exports every
symbol include/tsv.h declares; host canonicalization, shade assignment,
graph parsing and the synthetic generators match the reference semantics.
No compute call is made without a GPU here."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_2001_07158_b200 import _native, synth
from paper_2001_07158_b200.graph import MotifQuery, VertexColoring, parse_graph_text
from paper_2001_07158_b200.sieve import SieveConfig, build_shades, false_negative_bound

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    txt = open(os.path.join(ROOT, "include", "tsv.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(tsv_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    lib = _native.lib()
    syms = declared_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    assert lib.tsv_version().decode().startswith("tsv-b200")


def test_library_is_sm100a_only():
    # the fat binary carries sm_100a SASS and nothing else
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True,
                         text=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def test_canonical_edges_match_reference(golden):
    for c in golden["canonical"]:
        cu, cv, ct = _native.canonical_edges(c["n"], c["u"], c["v"], c["ts"], c["directed"])
        assert cu.tolist() == c["cu"] and cv.tolist() == c["cv"] and ct.tolist() == c["cts"]


def test_canonical_edges_errors():
    with pytest.raises(ValueError, match="endpoint out of range"):
        _native.canonical_edges(2, [0], [5], [1], True)
    with pytest.raises(ValueError, match="timestamp below 1"):
        _native.canonical_edges(2, [0], [1], [0], True)


def test_build_shades_match_reference(golden):
    for c in golden["shades"]:
        col = VertexColoring(c["colors"], max(c["colors"]))
        sh = build_shades(MotifQuery.from_multiset(c["motif"]), col, SieveConfig())
        assert sh.feasible == c["feasible"]
        if c["feasible"]:
            assert sh.vertex_off.tolist() == c["off"]
            assert sh.vertex_shades.tolist() == c["shades"]
        else:
            assert sh.missing_color == 7


def test_build_shades_canonical_sets():
    # test_sieve.cpp:38-73
    col = VertexColoring([1, 1, 2], 2)
    sh = build_shades(MotifQuery.from_multiset([1, 1, 2]), col, SieveConfig())
    assert sh.colors == [1, 2] and sh.shade_sets == [[1, 2], [3]]
    assert sh.shades_of(0).tolist() == [1, 2] and sh.shades_of(2).tolist() == [3]
    with pytest.raises(ValueError):
        build_shades(MotifQuery.size_only(3), col, SieveConfig())
    with pytest.raises(ValueError, match="lane_width"):
        build_shades(MotifQuery.from_multiset([1]), col, SieveConfig(lane_width=3))


def test_parse_graph_matches_reference_load(golden):
    g = golden["load_fig2"]
    n, u, v, ts, t, colors, q, names, rec = parse_graph_text(g["edges"], g["colors_text"])
    assert n == g["n"] and t == g["t"] and names == g["names"]
    assert colors.tolist() == g["colors"]
    cu, cv, ct = _native.canonical_edges(n, u, v, ts, False)
    assert cu.tolist() == g["u"] and cv.tolist() == g["v"] and ct.tolist() == g["ts"]


def test_parse_graph_rank_normalizes_and_reports_lines():
    n, u, v, ts, t, colors, q, names, rec = parse_graph_text("a b 100\nb c 7 # c\n\nc a 100\n")
    assert names == ["a", "b", "c"] and ts.tolist() == [2, 1, 2] and t == 2
    with pytest.raises(RuntimeError, match="line 2: malformed integer"):
        parse_graph_text("a b 1\na b x\n")
    with pytest.raises(RuntimeError, match="line 1: expected"):
        parse_graph_text("a b\n")


def test_false_negative_bound():
    assert false_negative_bound(4, 8) == pytest.approx(7.0 / 256.0)
    assert false_negative_bound(5, 64) == pytest.approx(9.0 / 2.0**64)


@pytest.mark.parametrize("cfg", [1, 2, 3, 4])
def test_synthetic_configs_have_distinct_edges(cfg):
    inst = synth.make_config(cfg, scale=1.0 if cfg == 1 else 0.01)
    key = (inst.u.astype(np.int64) * inst.n + inst.v) * (inst.t + 1) + inst.ts
    assert len(np.unique(key)) == inst.m
    assert (inst.u != inst.v).all() and inst.ts.min() >= 1 and inst.ts.max() <= inst.t
    # the planted path is a strictly increasing temporal path
    p = inst.planted
    edges = set(zip(inst.u.tolist(), inst.v.tolist(), inst.ts.tolist()))
    times = [min(t for (a, b, t) in edges if a == x and b == y) for x, y in zip(p, p[1:])]
    assert all(a < b for a, b in zip(times, times[1:])) or len(p) <= 2
    k_eff, col, motif, anchor = synth.effective_query(inst)
    assert len(motif) == k_eff


def test_synthetic_updates_formula():
    c1 = synth.make_config(1)
    assert c1.updates() == 10_000 * 4 * 32  # A (k-1) 2^k = 1.28e6


def test_canonical_edges_carry_transition_times_like_reference():
    """Transition times ride through canonicalization; among duplicate
    (ts,u,v) edges the survivor is the reference's (graph.cpp:34-41)."""
    from oracle import oracle
    try:
        oracle.ref_lib()
    except Exception as e:  # pragma: no cover
        pytest.skip(f"oracle/_ref not built: {e}")
    rng = np.random.default_rng(17)
    for it in range(60):
        n = int(rng.integers(2, 12))
        m = int(rng.integers(0, 60))
        u = rng.integers(0, n, m)
        v = rng.integers(0, n, m)
        ts = rng.integers(1, 6, m)
        eps = rng.integers(1, 4, m)
        directed = bool(it % 2)
        want = oracle.ref_eval_temporal_model(n, u, v, ts, eps, None, directed, [1] * n, [1],
                                              edge_model=1)
        cu, cv, ct, ce = _native.canonical_edges_eps(n, u, v, ts, eps, directed)
        assert cu.tolist() == want["u"].tolist() and cv.tolist() == want["v"].tolist()
        assert ct.tolist() == want["ts"].tolist() and ce.tolist() == want["eps"].tolist()


def test_nonzero_index_matches_numpy():
    """tsv_nonzero_index (the flagged list on all host threads) == np.nonzero."""
    from paper_2001_07158_b200 import _native
    rng = np.random.default_rng(4)
    for n, p in ((0, 0.5), (1, 1.0), (70_000, 0.3), (3_000_017, 0.9), (2_500_000, 0.0)):
        a = (rng.random(n) < p).astype(np.uint64) * rng.integers(1, 2**63, n, dtype=np.uint64)
        assert np.array_equal(_native.nonzero_index(a), np.nonzero(a)[0])

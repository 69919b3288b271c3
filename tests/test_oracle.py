"""CPU tests: the oracle against the reference's golden vectors and known
answers (test_gf.cpp, test_sieve.cpp of /root/reference/proj/tests)."""
import numpy as np
import pytest

from oracle import oracle as O


def u64(h):
    return int(h, 16)


def test_x63_times_x_is_modulus(golden):
    # test_gf.cpp:63-67
    assert O.gf_mul(1 << 63, 2) == 0x1B
    assert O.gf_mul_slow(1 << 63, 2) == 0x1B


def test_gf_mul_golden(golden):
    for a, b, c in golden["gf_mul"]:
        assert O.gf_mul(u64(a), u64(b)) == u64(c)
        assert O.gf_mul_slow(u64(a), u64(b)) == u64(c)


def test_gf_field_laws():
    rng = np.random.default_rng(3)
    xs = rng.integers(0, 2**63, (300, 3), dtype=np.uint64) * 2 + 1
    for a, b, c in xs.tolist():
        assert O.gf_mul(O.gf_mul(a, b), c) == O.gf_mul(a, O.gf_mul(b, c))
        assert O.gf_mul(a, b ^ c) == O.gf_mul(a, b) ^ O.gf_mul(a, c)
        assert O.gf_mul(a, b) == O.gf_mul(b, a)
        assert O.gf_mul(a, 1) == a


def test_draws_golden(golden):
    for seed, role, a, b, h in golden["draws"]:
        assert O.draw_nonzero(seed, role, a, b, 0) == u64(h)


def test_canonical_edges_golden(golden):
    for c in golden["canonical"]:
        cu, cv, ct = O.canonical_edges(c["n"], c["u"], c["v"], c["ts"], c["directed"])
        assert cu.tolist() == c["cu"] and cv.tolist() == c["cv"] and ct.tolist() == c["cts"]


def _oracle_case(c):
    cu, cv, ct = O.canonical_edges(c["n"], c["u"], c["v"], c["ts"], c["directed"])
    from paper_2001_07158_b200 import sieve as S
    from paper_2001_07158_b200.graph import MotifQuery, VertexColoring
    col = VertexColoring(c["colors"], max(c["colors"]) if c["colors"] else 1)
    sh = S.build_shades(MotifQuery.from_multiset(c["motif"]), col, S.SieveConfig(seed=c["seed"]))
    assert sh.feasible == c["feasible"]
    if not c["feasible"]:
        return None
    t = c["t"] or (int(ct.max()) if len(ct) else 1)
    max_ts = c["max_ts"] or t
    return O.oracle_eval(c["n"], cu, cv, ct, c["directed"], len(c["motif"]), max_ts,
                         sh.vertex_off, sh.vertex_shades, c["seed"], tuple(c["anchor"]))


def test_oracle_sieve_golden(golden):
    """Restatement pinned to the reference on every golden sieve case
    (accumulators where stored, checksum and flagged set everywhere)."""
    seen_nonzero = 0
    for c in golden["sieve"]:
        r = _oracle_case(c)
        if r is None:
            continue
        acc, nflag, cs = r
        assert f"{cs:016x}" == c["checksum"], c["name"]
        assert nflag == c["nflagged"], c["name"]
        assert np.nonzero(acc)[0].tolist() == c["flagged"], c["name"]
        if "acc" in c:
            assert [f"{int(x):016x}" for x in acc] == c["acc"], c["name"]
        seen_nonzero += nflag > 0
    assert seen_nonzero >= 20


def test_oracle_known_answers(golden):
    by = {c["name"]: c for c in golden["sieve"]}
    assert by["fig2 pathmotif {1,1,2,3}"]["flagged"] == [1]      # test_sieve.cpp:75-82
    assert by["single edge"]["flagged"] == [0, 1]                # :84-90
    for s in (1, 2, 3):
        assert by[f"decreasing directed seed{s}"]["flagged"] == []  # :92-104
    assert by["decreasing undirected"]["nflagged"] > 0
    assert by["chain demo h2"]["flagged"] == [0, 2]              # :106-114
    assert by["chain demo h1"]["flagged"] == []


def test_oracle_point_ranges_xor_to_full(golden):
    """Sieve points are independent: partial sums over any split XOR to the
    whole (the multi-GPU sharding invariant)."""
    c = next(c for c in golden["sieve"] if c["name"] == "fig2 pathmotif {1,1,2,3}")
    cu, cv, ct = O.canonical_edges(c["n"], c["u"], c["v"], c["ts"], c["directed"])
    from paper_2001_07158_b200 import sieve as S
    from paper_2001_07158_b200.graph import MotifQuery, VertexColoring
    sh = S.build_shades(MotifQuery.from_multiset(c["motif"]), VertexColoring(c["colors"], 4),
                        S.SieveConfig())
    off, shades = sh.vertex_off, sh.vertex_shades
    full = O.eval_points(5, cu, cv, ct, False, 4, 5, off, shades, 1)
    parts = [O.eval_points(5, cu, cv, ct, False, 4, 5, off, shades, 1, -1, a, b)
             for a, b in ((0, 3), (3, 9), (9, 16))]
    assert np.array_equal(parts[0] ^ parts[1] ^ parts[2], full)


@pytest.mark.skipif(not O.ref_available(), reason="reference build absent (GPU box)")
def test_oracle_vs_reference_random():
    from paper_2001_07158_b200 import synth
    rng = np.random.default_rng(11)
    nz = 0
    for _ in range(150):
        n, u, v, ts, d, colors, motif = synth.random_small(rng)
        cu, cv, ct = O.canonical_edges(n, u, v, ts, d)
        rcu, rcv, rct = O.ref_canonical_edges(n, u, v, ts, d)
        assert (cu == rcu).all() and (cv == rcv).all() and (ct == rct).all()
        sh = O.ref_build_shades(n, colors, motif, 3)
        if sh is None:
            continue
        t = int(ct.max()) if len(ct) else 1
        max_ts = int(rng.integers(1, t + 1))
        r = O.ref_eval(n, u, v, ts, d, colors, motif, max_ts=max_ts, seed=3, t=t)
        acc, nf, cs = O.oracle_eval(n, cu, cv, ct, d, len(motif), max_ts, sh[0], sh[1], 3)
        assert np.array_equal(acc, r["acc"]) and cs == r["checksum"]
        nz += nf > 0
    assert nz > 10


def _big_eval(n, u, v, ts, directed, k, max_ts, off, shades, seed, anchor_src, lanes,
              p0=0, p1=None):
    """The multi-threaded restatement (tsv_oracle_big.c): in-place
    canonicalization, head-grouped runs, `lanes` points per pass."""
    u2, v2, t2 = (np.array(x, dtype=np.int32) for x in (u, v, ts))
    w = O.canonicalize_inplace(n, u2, v2, t2, directed)
    G = O.BigGraph(n, u2[:w], v2[:w], t2[:w], directed, max_ts)
    return (u2[:w], v2[:w], t2[:w]), G.eval(k, off, shades, seed, anchor_src, p0, p1, lanes)


def test_big_oracle_sieve_golden(golden):
    """tsv_oracle_big.c (the checker of the full-size goldens) pinned to the
    reference's golden sieve cases: accumulators, flagged set, checksum."""
    from paper_2001_07158_b200 import sieve as S
    from paper_2001_07158_b200.graph import MotifQuery, VertexColoring
    nz = 0
    for i, c in enumerate(golden["sieve"]):
        sh = S.build_shades(MotifQuery.from_multiset(c["motif"]),
                            VertexColoring(c["colors"], max(c["colors"])),
                            S.SieveConfig(seed=c["seed"]))
        if not sh.feasible:
            continue
        cu, cv, ct = O.canonical_edges(c["n"], c["u"], c["v"], c["ts"], c["directed"])
        t = c["t"] or (int(ct.max()) if len(ct) else 1)
        max_ts = c["max_ts"] or t
        canon, acc = _big_eval(c["n"], c["u"], c["v"], c["ts"], c["directed"], len(c["motif"]),
                               max_ts, sh.vertex_off, sh.vertex_shades, c["seed"],
                               c["anchor"][0], lanes=(1, 3, 8, 16)[i % 4])
        assert all(np.array_equal(a, b) for a, b in zip(canon, (cu, cv, ct))), c["name"]
        a, nflag, cs = O.finalize(acc, c["anchor"][1])
        assert f"{cs:016x}" == c["checksum"], c["name"]
        assert np.nonzero(a)[0].tolist() == c["flagged"], c["name"]
        nz += nflag > 0
    assert nz >= 20


def test_big_oracle_matches_restatement_random():
    """Random small instances (loops, duplicates, undirected, anchors,
    horizons below t, partial point ranges, every lane count)."""
    from paper_2001_07158_b200 import sieve as S
    from paper_2001_07158_b200 import synth
    from paper_2001_07158_b200.graph import MotifQuery, VertexColoring
    rng = np.random.default_rng(21)
    for it in range(200):
        n, u, v, ts, d, colors, motif = synth.random_small(rng, k_max=7)
        k = len(motif)
        sh = S.build_shades(MotifQuery.from_multiset(motif),
                            VertexColoring(colors, int(colors.max())), S.SieveConfig(seed=5))
        if not sh.feasible:
            continue
        cu, cv, ct = O.canonical_edges(n, u, v, ts, d)
        max_ts = int(rng.integers(1, (int(ct.max()) if len(ct) else 1) + 1))
        anchor = -1 if rng.random() < 0.6 else int(rng.integers(0, n))
        P = 1 << k
        p0 = int(rng.integers(0, P))
        p1 = int(rng.integers(p0 + 1, P + 1))
        want = O.eval_points(n, cu, cv, ct, d, k, max_ts, sh.vertex_off, sh.vertex_shades, 5,
                             anchor, p0, p1)
        _, got = _big_eval(n, u, v, ts, d, k, max_ts, sh.vertex_off, sh.vertex_shades, 5, anchor,
                           int(rng.choice([1, 2, 5, 8, 16])), p0, p1)
        assert np.array_equal(got, want), it


def test_full_size_goldens_recorded():
    """tests/golden/full_size.json covers every BASELINE config at full size
    (C1's full-size case lives in golden.json) and C2's entries come from
    the reference itself."""
    import json
    import os
    with open(os.path.join(os.path.dirname(__file__), "golden", "full_size.json")) as f:
        full = json.load(f)
    assert len(full["C2"]["evals"]) == 5
    assert all(e["source"].startswith("reference") for e in full["C2"]["evals"])
    assert full["C3"]["evals"][0]["nflagged"] > 0
    assert full["C5x0.1"]["evals"][0]["nflagged"] > 0
    assert len(full["C4"]["points"]) >= 3
    if "C5" in full:
        assert len(full["C5"]["points"]) == 32
        x = 0
        for p in full["C5"]["points"]:
            x ^= int(p["xor_total"], 16)
        assert f"{x:016x}" == full["C5"]["evals"][0]["xor_total"]

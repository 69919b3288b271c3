"""Regenerates tests/golden/golden.json from the COMPILED REFERENCE.

Run in the build container (needs /root/reference, built into
oracle/_ref/libtsieve_ref.so by oracle/Makefile):

    python tests/golden/make_golden.py

Every value below comes from the unmodified reference core
(/root/reference/proj/core/src) through oracle/ref_shim.cpp; the reference
itself ships no golden accumulator values, so these
vectors pin both the C restatement (oracle/tsv_oracle.c) and the CUDA engine.
Inputs are seeded synthetic instances; nothing is taken from any dataset.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2001_07158_b200 import synth  # noqa: E402

FIG2_EDGES = "u1 u2 3\nu2 u3 1\nu3 u4 3\nu4 u5 1\nu5 u1 2\nu2 u5 4\nu3 u5 5\n"
FIG2_COLORS = "u1 1\nu2 3\nu3 4\nu4 1\nu5 2\n"


def hx(x: int) -> str:
    return f"{int(x):016x}"


def sieve_case(name, n, u, v, ts, directed, colors, motif, max_ts=0, seed=1, anchor=(-1, -1),
               t=0, full=True):
    r = O.ref_eval(n, u, v, ts, directed, colors, motif, max_ts=max_ts, seed=seed, lanes=8,
                   threads=1, anchor=anchor, t=t)
    case = {"name": name, "n": int(n), "u": [int(x) for x in u], "v": [int(x) for x in v],
            "ts": [int(x) for x in ts], "directed": bool(directed),
            "colors": [int(x) for x in colors], "motif": [int(x) for x in motif],
            "max_ts": int(max_ts), "seed": int(seed), "anchor": list(anchor), "t": int(t)}
    if r is None:
        case["feasible"] = False
        return case
    case.update({"feasible": True, "checksum": hx(r["checksum"]), "nflagged": r["nflagged"],
                 "global": r["global"],
                 "xor_total": hx(np.bitwise_xor.reduce(r["acc"]) if n else 0),
                 "flagged": [int(x) for x in np.nonzero(r["acc"])[0]]})
    if full:
        case["acc"] = [hx(x) for x in r["acc"]]
    return case


def main():
    rng = np.random.default_rng(2001_07158)
    out = {"generator": "tests/golden/make_golden.py (reference core via oracle/ref_shim.cpp)"}

    # GF(2^64) and draws (gf.hpp:85-153); test_gf.cpp:63-67 pins x^63*x = 0x1b.
    pairs = [(1 << 63, 2)] + [(int(a), int(b)) for a, b in
                              rng.integers(0, 2**63, (200, 2), dtype=np.uint64) * 2 + 1]
    out["gf_mul"] = [[hx(a), hx(b), hx(O.ref_lib().ref_gf_mul(a, b))] for a, b in pairs]
    draws = []
    for seed in (1, 2, 99):
        for role in (1, 2, 3):
            for a in (0, 1, 7, 123456):
                for b in (0, 1, 4):
                    draws.append([seed, role, a, b,
                                  hx(O.ref_lib().ref_draw_nonzero(seed, role, a, b, 0))])
    out["draws"] = draws

    # canonical edge ids (graph.cpp:14-43)
    canon = []
    for i in range(20):
        n = int(rng.integers(2, 12))
        m = int(rng.integers(0, 40))
        u, v = rng.integers(0, n, m), rng.integers(0, n, m)
        ts = rng.integers(1, 5, m)
        d = bool(i % 2)
        cu, cv, ct = O.ref_canonical_edges(n, u, v, ts, d)
        canon.append({"n": n, "u": u.tolist(), "v": v.tolist(), "ts": ts.tolist(), "directed": d,
                      "cu": cu.tolist(), "cv": cv.tolist(), "cts": ct.tolist()})
    out["canonical"] = canon

    # shade CSR (sieve.cpp:658-718)
    shades = []
    for motif, colors in (([1, 1, 2], [1, 1, 2]), ([1, 2], [1, 1, 2]), ([1, 1, 1, 1], [1] * 4),
                          ([3, 1, 1, 2], [2, 3, 1, 1, 3]), ([1, 7], [1, 1, 2])):
        r = O.ref_build_shades(len(colors), colors, motif)
        shades.append({"colors": colors, "motif": motif, "feasible": r is not None,
                       "off": None if r is None else r[0].tolist(),
                       "shades": None if r is None else r[1].tolist()})
    out["shades"] = shades

    # load_graph on the fig2 fixture text (graph.cpp:376-448)
    lg = O.ref_load_graph(FIG2_EDGES, FIG2_COLORS, False)
    out["load_fig2"] = {"edges": FIG2_EDGES, "colors_text": FIG2_COLORS, "n": lg["n"],
                        "t": lg["t"], "u": lg["u"].tolist(), "v": lg["v"].tolist(),
                        "ts": lg["ts"].tolist(), "colors": lg["colors"].tolist(),
                        "names": lg["names"]}

    # temporal sieve known answers (test_sieve.cpp:75-114 instances)
    cases = []
    U1, U2, U3, U4, U5 = range(5)
    fig2 = ([U1, U2, U3, U4, U5, U2, U3], [U2, U3, U4, U5, U1, U5, U5], [3, 1, 3, 1, 2, 4, 5])
    fig2_col = [1, 3, 4, 1, 2]
    cases.append(sieve_case("fig2 pathmotif {1,1,2,3}", 5, *fig2, False, fig2_col, [1, 1, 2, 3]))
    cases.append(sieve_case("fig2 seed5", 5, *fig2, False, fig2_col, [1, 1, 2, 3], seed=5))
    cases.append(sieve_case("fig2 k-temppath k=4", 5, *fig2, False, [1] * 5, [1] * 4))
    cases.append(sieve_case("fig2 k-temppath k=6", 5, *fig2, False, [1] * 5, [1] * 6))
    cases.append(sieve_case("single edge", 2, [0], [1], [1], False, [1, 2], [1, 2]))
    for seed in (1, 2, 3):
        cases.append(sieve_case(f"decreasing directed seed{seed}", 3, [0, 1], [1, 2], [2, 1],
                                True, [1, 2, 3], [1, 2, 3], seed=seed))
    cases.append(sieve_case("decreasing undirected", 3, [0, 1], [1, 2], [2, 1], False, [1, 2, 3],
                            [1, 2, 3]))
    chain = ([0, 0, 1, 1], [1, 1, 2, 2], [1, 2, 1, 2])
    cases.append(sieve_case("chain demo h2", 3, *chain, False, [1, 2, 3], [1, 2, 3], max_ts=2))
    cases.append(sieve_case("chain demo h1", 3, *chain, False, [1, 2, 3], [1, 2, 3], max_ts=1))
    # random sweep: directed/undirected, anchors, horizons, k = 1..7
    for i in range(80):
        n, u, v, ts, d, colors, motif = synth.random_small(rng, n_max=16, m_max=50, t_max=7,
                                                           k_max=7, q_max=3)
        cu, cv, ct = O.ref_canonical_edges(n, u, v, ts, d)
        tmax = int(ct.max()) if len(ct) else 1
        max_ts = int(rng.integers(1, tmax + 1))
        anchor = (-1, -1)
        if i % 4 == 3 and n >= 2:
            s, dd = rng.choice(n, 2, replace=False)
            anchor = (int(s), int(dd))
        cases.append(sieve_case(f"random {i}", n, u, v, ts, d, colors, motif, max_ts=max_ts,
                                seed=int(rng.integers(1, 10**6)), anchor=anchor, t=tmax))
    # config 1 (BASELINE configs[0]) -- full accumulator vector
    c1 = synth.make_config(1)
    k, col, motif, anchor = synth.effective_query(c1)
    cases.append(sieve_case("C1 k-TempPath k=5", c1.n, c1.u, c1.v, c1.ts, True, col, motif,
                            seed=1, full=True))
    out["sieve"] = cases

    # solver level (solver.cpp), fig2 and (s,d)
    solves = []
    for prob, motif, k, mode in (("pathmotif", [1, 1, 2, 3], 0, 0), ("colorfulpath", [1, 2, 3, 4], 0, 0),
                                 ("ktemppath", [], 4, 0), ("ktemppath", [], 6, 0),
                                 ("pathmotif", [1, 1, 2, 3], 0, 1), ("pathmotif", [1, 1, 2, 3], 0, 3),
                                 ("ktemppath", [], 4, 3)):
        r = O.ref_solve(5, *fig2, False, fig2_col, prob, motif, k, seed=1, mode=mode)
        solves.append({"problem": prob, "motif": motif, "k": k, "mode": mode, "result": r})
    r = O.ref_solve(5, *fig2, False, fig2_col, "sdcolorful", [], 2, source=U4, dest=U2, seed=1,
                    mode=3)
    solves.append({"problem": "sdcolorful", "motif": [], "k": 2, "source": U4, "dest": U2,
                   "mode": 3, "result": r})
    out["solve_fig2"] = solves

    # solver sweep: the four problems x decide / optimum / extract (both
    # strategies) x preprocess none / colors on random small instances
    sweep = []
    srng = np.random.default_rng(777)
    problems = ["ktemppath", "pathmotif", "colorfulpath", "sdcolorful"]
    for i in range(64):
        n, u, v, ts, d, colors, motif = synth.random_small(srng, n_max=14, m_max=60, t_max=6,
                                                           k_max=5, q_max=3)
        prob = problems[i % 4]
        k, src, dst = 0, -1, -1
        if prob == "ktemppath":
            motif, k = [], int(srng.integers(2, 5))
        elif prob == "colorfulpath":
            motif = sorted(set(motif)) or [1]
        elif prob == "sdcolorful":
            motif, k = [], int(srng.integers(1, 3))
            src, dst = (int(x) for x in srng.choice(n, 2, replace=False))
        mode = [0, 1, 2, 3][(i // 4) % 4]
        extraction = (i // 16) % 2
        pre = (i // 32) % 2
        seed = int(srng.integers(1, 1000))
        r = O.ref_solve(n, u, v, ts, d, colors, prob, motif, k, source=src, dest=dst, seed=seed,
                        mode=mode, extraction=extraction, preprocess=pre)
        sweep.append({"n": n, "u": u.tolist(), "v": v.tolist(), "ts": ts.tolist(), "directed": d,
                      "colors": colors.tolist(), "problem": prob, "motif": motif, "k": k,
                      "source": src, "dest": dst, "seed": seed, "mode": mode,
                      "extraction": extraction, "preprocess": pre, "result": r})
    out["solve_sweep"] = sweep

    # default preprocessing (junction sieve on the static projection): the
    # kept-vertex set changes edge renumbering, so checksums pin it exactly
    pre_sweep = []
    for i in range(48):
        n, u, v, ts, d, colors, motif = synth.random_small(srng, n_max=18, m_max=70, t_max=6,
                                                           k_max=5, q_max=3)
        prob = problems[i % 4]
        k, src, dst = 0, -1, -1
        if prob == "ktemppath":
            motif, k = [], int(srng.integers(1, 5))
        elif prob == "colorfulpath":
            motif = sorted(set(motif)) or [1]
        elif prob == "sdcolorful":
            motif, k = [], int(srng.integers(1, 3))
            src, dst = (int(x) for x in srng.choice(n, 2, replace=False))
        mode = [0, 3][(i // 4) % 2]
        pre = [3, 2][(i // 8) % 2]
        seed = int(srng.integers(1, 1000))
        r = O.ref_solve(n, u, v, ts, d, colors, prob, motif, k, source=src, dest=dst, seed=seed,
                        mode=mode, extraction=(i // 16) % 2, preprocess=pre)
        pre_sweep.append({"n": n, "u": u.tolist(), "v": v.tolist(), "ts": ts.tolist(),
                          "directed": d, "colors": colors.tolist(), "problem": prob,
                          "motif": motif, "k": k, "source": src, "dest": dst, "seed": seed,
                          "mode": mode, "extraction": (i // 16) % 2, "preprocess": pre,
                          "result": r})
    out["solve_sweep_preprocess"] = pre_sweep
    fig2_default = []
    for prob, motif, k in (("pathmotif", [1, 1, 2, 3], 0), ("colorfulpath", [1, 2, 3, 4], 0),
                           ("ktemppath", [], 4), ("pathmotif", [1, 1, 1, 3], 0)):
        r = O.ref_solve(5, *fig2, False, fig2_col, prob, motif, k, seed=1, mode=3, preprocess=3)
        fig2_default.append({"problem": prob, "motif": motif, "k": k, "result": r})
    out["solve_fig2_default"] = fig2_default

    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=0)
    print(f"wrote {path}: {len(cases)} sieve cases, {os.path.getsize(path)} bytes")


if __name__ == "__main__":
    main()

"""Full-size goldens for the five BASELINE configs -> tests/golden/full_size.json.

    python tests/golden/make_golden_full.py [CONFIG ...]      (default: 2 3 4 5s 5)

Run in the build container.  What pins what:

* C2 (n=1e5, m=1e6, k=6, seeds 1-4): the UNMODIFIED reference core
  (oracle/_ref, eval_temporal_sieve, sieve.cpp:170-307) at max_ts = t for
  every seed and at one binary-search horizon (max_ts = t/2, seed 1), on all
  host threads; the multi-threaded oracle (oracle/tsv_oracle_big.c) is
  checked against it on the same inputs before anything is written.
* C3 full, C5 x0.1 (full point range), C5 full (full range, one point at a
  time, so every point's partial sum is stored too): the multi-threaded
  oracle, whose restatement is pinned to the reference by tests/test_oracle.py.
  The reference's dense layers cannot be allocated there (sieve.cpp:188-192).
* C4 full (k_eff = 12, 4096 points, ~1e9 arc-levels per point): sampled
  blocks of sieve points (hard part 6).  XOR over points
  is exact, so every block is independently checkable.

Per evaluation the file stores the finalize() outputs (sieve.cpp:136-159):
checksum, flagged count and XOR of the accumulators after the sink
restriction; per sampled block the checksum/XOR of the RAW per-vertex partial
sums (no sink restriction, so all n words are covered).  Inputs are the
seeded synthetic instances of paper_2001_07158_b200/synth.py.
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2001_07158_b200 import synth  # noqa: E402
from paper_2001_07158_b200.graph import MotifQuery, VertexColoring  # noqa: E402
from paper_2001_07158_b200.sieve import SieveConfig, build_shades  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "full_size.json")


def hx(x: int) -> str:
    return f"{int(x):016x}"


def summary(acc, sink=-1):
    a, nflag, cs = O.finalize(acc, sink)
    return {"checksum": hx(cs), "nflagged": nflag,
            "xor_total": hx(np.bitwise_xor.reduce(a) if len(a) else 0)}


def log(*a):
    print(f"[{time.strftime('%H:%M:%S')}]", *a, flush=True)


class Prepared:
    """A config's canonical graph in the oracle's layout + shade CSR."""

    def __init__(self, cfg, scale=1.0, max_ts=None):
        t0 = time.time()
        inst = synth.make_config(cfg, scale=scale)
        self.inst_meta = {"name": inst.name, "n": inst.n, "m": inst.m, "t": inst.t,
                          "directed": inst.directed, "k_eff": inst.k_eff}
        k, colors, motif, anchor = synth.effective_query(inst)
        self.k, self.anchor = k, anchor
        self.sh = build_shades(MotifQuery.from_multiset(motif),
                               VertexColoring(colors, int(colors.max())), SieveConfig(seed=1))
        self.shades_by_seed = {}
        self.colors, self.motif = colors, motif
        u, v, ts = (np.ascontiguousarray(x, dtype=np.int32) for x in (inst.u, inst.v, inst.ts))
        self.raw = (inst.u, inst.v, inst.ts) if cfg == 2 else None
        directed, n = inst.directed, inst.n
        del inst
        w = O.canonicalize_inplace(n, u, v, ts, directed)
        self.t = int(ts[:w].max())
        self.max_ts = self.t if max_ts is None else max_ts
        self.n, self.m = n, w
        self.G = O.BigGraph(n, u[:w], v[:w], ts[:w], directed, self.max_ts)
        del u, v, ts
        log(f"C{cfg} x{scale}: n={n} m={w} arcs={self.G.arcs} runs={self.G.runs} "
            f"prepared in {time.time() - t0:.1f} s")

    def shades(self, seed):
        if seed not in self.shades_by_seed:
            self.shades_by_seed[seed] = build_shades(
                MotifQuery.from_multiset(self.motif),
                VertexColoring(self.colors, int(self.colors.max())), SieveConfig(seed=seed))
        return self.shades_by_seed[seed]

    def eval(self, seed, p0, p1, lanes):
        sh = self.shades(seed)
        return self.G.eval(self.k, sh.vertex_off, sh.vertex_shades, seed, self.anchor[0], p0, p1,
                           lanes=lanes)

    def header(self, cfg, scale):
        return dict(self.inst_meta, config=cfg, scale=scale, m_canonical=int(self.m),
                    arcs=int(self.G.arcs), runs=int(self.G.runs), k=int(self.k),
                    anchor=list(self.anchor), t_canonical=int(self.t))


def gen_c2():
    cfg = 2
    P = Prepared(cfg)
    rec = P.header(cfg, 1.0)
    n, (u, v, ts) = P.n, P.raw
    evals = []
    threads = os.cpu_count() or 8
    for seed, max_ts in [(1, P.t), (2, P.t), (3, P.t), (4, P.t), (1, P.t // 2)]:
        t0 = time.time()
        r = O.ref_eval(n, u, v, ts, True, P.colors, P.motif, max_ts=max_ts, seed=seed, lanes=8,
                       threads=threads, t=P.t)
        sec = time.time() - t0
        ref = {"checksum": hx(r["checksum"]), "nflagged": r["nflagged"],
               "xor_total": hx(np.bitwise_xor.reduce(r["acc"]))}
        # the oracle on the same inputs (its own graph for the horizon)
        G = P.G if max_ts == P.t else None
        if G is None:
            cu, cv, ct = O.canonical_edges(n, u, v, ts, True)
            G = O.BigGraph(n, cu, cv, ct, True, max_ts)
        sh = P.shades(seed)
        acc = G.eval(P.k, sh.vertex_off, sh.vertex_shades, seed, -1, lanes=16)
        mine = summary(acc)
        if mine != ref:
            raise SystemExit(f"oracle != reference on C2 seed {seed} max_ts {max_ts}: "
                             f"{mine} vs {ref}")
        log(f"C2 seed {seed} max_ts {max_ts}: reference {sec:.1f} s, {ref}")
        evals.append(dict(seed=seed, max_ts=max_ts, source="reference (oracle/_ref) == oracle",
                          reference_seconds=round(sec, 2), reference_threads=threads, **ref))
    rec["evals"] = evals
    return rec


def gen_full_range(cfg, scale, lanes, per_point=False, seed=1):
    P = Prepared(cfg, scale)
    rec = P.header(cfg, scale)
    t0 = time.time()
    P_all = 1 << P.k
    if per_point:
        total = np.zeros(P.n, np.uint64)
        pts = []
        for p in range(P_all):
            t1 = time.time()
            acc = P.eval(seed, p, p + 1, 1)
            total ^= acc
            s = summary(acc)
            pts.append(dict(p_begin=p, p_end=p + 1, **s))
            log(f"C{cfg} point {p}: {s} ({time.time() - t1:.1f} s)")
        rec["points"] = pts
        acc = total
    else:
        acc = P.eval(seed, 0, P_all, lanes)
    s = summary(acc, P.anchor[1])
    log(f"C{cfg} x{scale} full range seed {seed}: {s} in {time.time() - t0:.1f} s")
    rec["evals"] = [dict(seed=seed, max_ts=P.max_ts, source="oracle/tsv_oracle_big.c",
                         oracle_seconds=round(time.time() - t0, 1),
                         oracle_threads=O.max_threads(), **s)]
    return rec


def gen_c4(blocks=((0, 4), (2048, 2052), (4092, 4096))):
    cfg = 4
    P = Prepared(cfg)
    rec = P.header(cfg, 1.0)
    pts = []
    for a, b in blocks:
        t0 = time.time()
        acc = P.eval(1, a, b, b - a)
        s = summary(acc)
        log(f"C4 points [{a},{b}): {s} ({time.time() - t0:.1f} s)")
        pts.append(dict(seed=1, p_begin=a, p_end=b, **s))
    rec["points"] = pts
    return rec


def main():
    which = sys.argv[1:] or ["2", "3", "4", "5s", "5"]
    data = {}
    if os.path.exists(OUT):
        with open(OUT) as f:
            data = json.load(f)
    data["generator"] = "tests/golden/make_golden_full.py"
    for w in which:
        if w == "2":
            rec = gen_c2()
        elif w == "3":
            rec = gen_full_range(3, 1.0, lanes=16)
        elif w == "4":
            rec = gen_c4()
        elif w == "5s":
            rec = gen_full_range(5, 0.1, lanes=8)
        elif w == "5":
            rec = gen_full_range(5, 1.0, lanes=1, per_point=True)
        else:
            raise SystemExit(f"unknown config {w}")
        key = f"C{w[0]}" + ("x0.1" if w.endswith("s") else "")
        data[key] = rec
        with open(OUT, "w") as f:        # after every config: long runs keep progress
            json.dump(data, f, indent=1, sort_keys=True)
        log(f"wrote {key}")


if __name__ == "__main__":
    main()

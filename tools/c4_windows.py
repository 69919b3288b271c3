"""C4 at full size (n=1e6, m=1e8, k_eff=12): the coefficient engine in time
windows against the point engine (the multi-GPU path, pinned by the sampled
point goldens of tests/golden/full_size.json), same accumulators expected.
`python tools/c4_windows.py [SCALE] [--points]`"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    scale = float(sys.argv[1]) if len(sys.argv) > 1 and not sys.argv[1].startswith("-") else 1.0
    import numpy as np
    import paper_2001_07158_b200 as T
    from paper_2001_07158_b200 import _native, synth
    inst = synth.make_config(4, scale=scale)
    k, colors, motif, anchor = synth.effective_query(inst)
    t0 = time.perf_counter()
    g = T.TemporalGraph.build(inst.n, (inst.u, inst.v, inst.ts), inst.directed, 0, 0)
    print(f"build {time.perf_counter() - t0:.2f} s", flush=True)
    del inst
    cfg = T.SieveConfig(seed=1, memory_cap_words=1 << 62)
    sh = T.build_shades(T.MotifQuery.from_multiset(motif),
                        T.VertexColoring(colors, int(colors.max())), cfg)
    an = T.AnchorSpec(*anchor)
    res = {}
    _native.Profile.reset()
    _native.Profile.enable(True)
    for i in range(3):
        t0 = time.perf_counter()
        o = T.eval_temporal_sieve(g, k, g.t(), sh, cfg, an)
        dt = time.perf_counter() - t0
        print(f"coef eval {i}: {dt:.3f} s checksum {o.checksum:016x} yes {o.global_nonzero} "
              f"peak_words {o.peak_field_words}", flush=True)
        res.setdefault("coef_s", []).append(round(dt, 4))
    kern = {}
    for nm in ("coef_arcs_first", "coef_arcs", "coef_arcs_last", "coef_fixup", "coef_ztrans",
               "coef_win_carry", "coef_readout"):
        c, ms = _native.Profile.get(nm)
        if c:
            kern[nm] = {"launches": c // 3, "ms_per_eval": round(ms / 3, 2)}
    c, ms = _native.Profile.get(None)
    kern["all"] = {"launches": c // 3, "ms_per_eval": round(ms / 3, 2)}
    _native.Profile.enable(False)
    res["kernels"] = kern
    res["checksum"] = f"{o.checksum:016x}"
    res["acc_sum"] = int(np.bitwise_xor.reduce(o.accumulators)) if len(o.accumulators) else 0
    if "--points" in sys.argv:
        os.environ["TSV_ENGINE"] = "points"
        t0 = time.perf_counter()
        p = T.eval_temporal_sieve(g, k, g.t(), sh, cfg, an)
        res["points_s"] = round(time.perf_counter() - t0, 3)
        res["points_checksum"] = f"{p.checksum:016x}"
        res["match"] = bool(np.array_equal(p.accumulators, o.accumulators))
        del os.environ["TSV_ENGINE"]
    print("RESULT " + json.dumps(res), flush=True)


if __name__ == "__main__":
    main()

"""Wall time of single eval_temporal_sieve calls (one repetition, one horizon)
on a BASELINE config, through the Python mirror of the C-ABI: what one
binary-search probe of `tsieve extract` costs.
`python tools/probe_timing.py --config 2`."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2001_07158_b200 as T  # noqa: E402
from paper_2001_07158_b200 import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--cap", type=int, default=62, help="log2 memory_cap_words")
    args = ap.parse_args()
    inst = synth.make_config(args.config, scale=args.scale)
    k, colors, motif, anchor = synth.effective_query(inst)
    t0 = time.perf_counter()
    g = T.TemporalGraph.build(inst.n, (inst.u, inst.v, inst.ts), inst.directed, 0, 0)
    t_build = time.perf_counter() - t0
    col = T.VertexColoring(colors, int(colors.max()))
    cfg = T.SieveConfig(seed=1, memory_cap_words=1 << args.cap)
    sh = T.build_shades(T.MotifQuery.from_multiset(motif), col, cfg)
    an = T.AnchorSpec(*anchor)
    full = g.t()
    rows = []
    for max_ts in [full, full, full // 2, full // 4, full // 2 + full // 8, full, full // 3]:
        t0 = time.perf_counter()
        o = T.eval_temporal_sieve(g, k, max_ts, sh, cfg, an)
        rows.append({"max_ts": max_ts, "s": round(time.perf_counter() - t0, 5),
                     "yes": bool(o.global_nonzero)})
    # per-kernel CUDA-event times of 3 full evaluations
    from paper_2001_07158_b200 import _native
    _native.Profile.reset()
    _native.Profile.enable(True)
    for _ in range(3):
        T.eval_temporal_sieve(g, k, full, sh, cfg, an)
    names = ["coef_vertex_first", "coef_vertex", "coef_vertex_last",
             "coef_arcs_first", "coef_arcs", "coef_arcs_last", "coef_ztrans", "coef_fixup",
             "coef_readout", "level_first", "level", "level_last", "level_grouped_first",
             "level_grouped", "zbatch", "zj", "fixup"]
    kern = {}
    for nm in names:
        cnt, ms = _native.Profile.get(nm)
        if cnt:
            kern[nm] = {"launches": cnt // 3, "ms_per_eval": round(ms / 3, 4)}
    cnt, ms = _native.Profile.get(None)
    kern["all"] = {"launches": cnt // 3, "ms_per_eval": round(ms / 3, 4)}
    _native.Profile.enable(False)
    print(json.dumps({"config": args.config, "scale": args.scale, "build_s": t_build,
                      "probes": rows, "kernels": kern}))


if __name__ == "__main__":
    main()

"""Compare engine builds on one BASELINE config: for every library given
(the in-tree lib/libtsv.so or exp_libs/libtsv_<name>.so from
tools/build_variant.sh), a fresh process builds the config, runs full
evaluations with per-kernel CUDA-event profiling and checks the checksum
against tests/golden/full_size.json when the config has one.

  python tools/variants.py --config 5 --scale 0.1 lib/libtsv.so exp_libs/libtsv_a.so
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, os, sys, time
sys.path.insert(0, ROOT)
import paper_2001_07158_b200 as T
from paper_2001_07158_b200 import synth, _native
inst = synth.make_config(CFG, scale=SCALE)
k, colors, motif, anchor = synth.effective_query(inst)
g = T.TemporalGraph.build(inst.n, (inst.u, inst.v, inst.ts), inst.directed, 0, 0)
del inst
cfg = T.SieveConfig(seed=1, memory_cap_words=1 << 62)
sh = T.build_shades(T.MotifQuery.from_multiset(motif), T.VertexColoring(colors, int(colors.max())), cfg)
an = T.AnchorSpec(*anchor)
o = T.eval_temporal_sieve(g, k, g.t(), sh, cfg, an)
_native.Profile.reset(); _native.Profile.enable(True)
R = 3
walls = []
for _ in range(R):
    t0 = time.perf_counter()
    o = T.eval_temporal_sieve(g, k, g.t(), sh, cfg, an)
    walls.append(time.perf_counter() - t0)
names = ["coef_vertex_first", "coef_vertex", "coef_vertex_last", "coef_arcs_first", "coef_arcs",
         "coef_arcs_last", "coef_ztrans", "coef_fixup", "coef_readout", "level_first", "level",
         "level_last", "level_grouped", "coef_win_carry"]
kern = {}
for nm in names:
    c, ms = _native.Profile.get(nm)
    if c:
        kern[nm] = round(ms / R, 3)
c, ms = _native.Profile.get(None)
kern["all"] = round(ms / R, 3)
print("RESULT " + json.dumps({"checksum": "%016x" % o.checksum, "nflagged": len(o.flagged),
                              "wall_s": [round(w, 4) for w in walls], "kernels_ms": kern}))
"""


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--scale", type=float, default=0.1)
    ap.add_argument("libs", nargs="+")
    a = ap.parse_args()
    with open(os.path.join(ROOT, "tests", "golden", "full_size.json")) as f:
        gold = json.load(f)
    key = f"C{a.config}" + ("" if a.scale == 1.0 else f"x{a.scale:g}")
    want = None
    if key in gold and gold[key].get("evals"):
        want = [e for e in gold[key]["evals"] if e["seed"] == 1 and e["max_ts"] == gold[key]["t"]]
        want = want[0]["checksum"] if want else None
    code = CHILD.replace("ROOT", repr(ROOT)).replace("CFG", str(a.config)).replace(
        "SCALE", repr(a.scale))
    for lib in a.libs:
        env = dict(os.environ, TSV_LIB=os.path.join(ROOT, lib) if not os.path.isabs(lib) else lib)
        p = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
        line = [x for x in p.stdout.splitlines() if x.startswith("RESULT ")]
        if p.returncode or not line:
            print(f"{lib}: FAILED rc={p.returncode}\n{p.stderr[-2000:]}", flush=True)
            continue
        r = json.loads(line[0][7:])
        r["golden"] = want
        r["parity"] = None if want is None else r["checksum"] == want
        print(f"{lib}: {json.dumps(r)}", flush=True)


if __name__ == "__main__":
    main()

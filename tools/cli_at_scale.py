"""Drive the tsieve CLI (C++ drop-in) on a BASELINE config written as text
files, e.g. C2 decide+extract: `python tools/cli_at_scale.py --config 2`.
Prints one JSON line per CLI run with wall time and the record's fields."""
import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2001_07158_b200 import synth  # noqa: E402

CLI = os.path.join(ROOT, "paper_2001_07158_b200", "lib", "tsieve")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--preprocess", nargs="+", default=["none", "both"])
    ap.add_argument("--commands", nargs="+", default=["decide", "extract"])
    ap.add_argument("--extraction", nargs="+", default=["localized"],
                    help="extraction strategies for the extract runs")
    args = ap.parse_args()
    inst = synth.make_config(args.config, scale=args.scale)
    d = tempfile.mkdtemp()
    ef, cf = os.path.join(d, "g.edges"), os.path.join(d, "g.colors")
    t0 = time.perf_counter()
    import pandas as pd
    pd.DataFrame({"u": inst.u, "v": inst.v, "ts": inst.ts}).to_csv(
        ef, sep=" ", header=False, index=False, chunksize=1 << 22)
    print(json.dumps({"config": args.config, "scale": args.scale, "m": int(inst.m),
                      "n": int(inst.n), "text_bytes": os.path.getsize(ef),
                      "write_s": time.perf_counter() - t0}), flush=True)
    with open(cf, "w") as f:
        f.write("".join(f"{i} {c}\n" for i, c in enumerate(inst.colors.tolist())))
    base = ["--graph", ef, "--colors", cf, "--problem", inst.problem, "--format", "json"]
    if inst.directed:
        base.append("--directed")
    if inst.motif:
        base += ["--motif", ",".join(map(str, inst.motif))]
    else:
        base += ["--k", str(inst.k)]
    if inst.problem == "sdcolorful":
        base += ["--source", str(inst.source), "--dest", str(inst.dest)]
    runs = [(pre, cmd, ex) for pre in args.preprocess for cmd in args.commands
            for ex in (args.extraction if cmd == "extract" else ["localized"])]
    for pre, cmd, ex in runs:
        t0 = time.perf_counter()
        p = subprocess.run([CLI, cmd] + base + ["--preprocess", pre, "--extraction", ex],
                           capture_output=True, text=True)
        wall = time.perf_counter() - t0
        try:
            rec = json.loads(p.stdout)
        except Exception:
            print(json.dumps({"cmd": cmd, "preprocess": pre, "rc": p.returncode,
                              "stderr": p.stderr[-500:]}))
            continue
        print(json.dumps({"config": args.config, "cmd": cmd, "preprocess": pre,
                          "extraction": ex,
                          "rc": p.returncode, "wall_s": wall,
                          "decision": rec["decision"], "optimum_ts": rec["optimum_ts"],
                          "oracle_calls": rec["oracle_calls"], "timings": rec["timings"],
                          "witness": rec["witness"]["vertices"] if rec["witness"] else None,
                          "planted": inst.planted, "checksum": rec["accumulator_checksum"],
                          "preprocessed": rec["preprocessed"]}), flush=True)


if __name__ == "__main__":
    main()

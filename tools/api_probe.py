"""One decide through the C++ drop-in API (libtsieve: TemporalGraph::build +
solve(decide)) on a BASELINE config, with the phase traces of the C++ layer
(TSIEVE_TRACE) and the C-ABI (TSV_TRACE_API) on stderr:
`python tools/api_probe.py CONFIG [SCALE] [REPEATS]`."""
import os
import sys
import time

os.environ.setdefault("TSIEVE_TRACE", "1")
os.environ.setdefault("TSV_TRACE_API", "1")
os.environ.setdefault("TSV_TRACE_COEF", "1")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import bench
    from paper_2001_07158_b200 import synth
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
    rep = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    inst = synth.make_config(cfg, scale=scale)
    reps = {2: 4}.get(cfg, 1)
    for i in range(rep):
        t0 = time.perf_counter()
        out = bench.e2e_api_leg(inst, reps, 1, inst.updates() * reps, None)
        print(f"decide {i}: {time.perf_counter() - t0:.3f} s (leg {out['ms_per_step']:.1f} ms) "
              f"{out['checksums']}", flush=True)


if __name__ == "__main__":
    main()

"""Measure the integer-pipe peaks the roofline needs on the GPU box (the
driver's MEASURED_PEAKS.json has none): mul.wide.u32 and
3-input LOP3 throughput (tsv_gf_bench pipe probes), and GF(2^64) product
throughput per multiply variant.  Writes gpurun_out/int_pipe_peaks.json
(committed as profiles/int_pipe_peaks.json)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2001_07158_b200 import _native  # noqa: E402

NAMES = {7: "mul.wide.u32 ops/s (FMA-heavy pipe)", 8: "LOP3 ops/s (ALU pipe)",
         1: "GF product, bit-serial", 2: "GF product, holes + Karatsuba",
         3: "GF product, holes + schoolbook", 9: "GF product, holes period 5",
         4: "GF product, smem table, 1 per lane per table",
         5: "GF product, smem table, 2 per lane per table",
         6: "GF product, smem table, 4 per lane per table",
         10: "GF product, lane table, 1 per build",
         11: "GF product, lane table, 5 per build",
         12: "GF product, lane table, 10 per build"}


def main():
    out = {}
    import numpy as np
    rng = np.random.default_rng(3)
    a = rng.integers(0, 2**64 - 1, 100_000, dtype=np.uint64, endpoint=True)
    b = rng.integers(0, 2**64 - 1, 100_000, dtype=np.uint64, endpoint=True)
    a[:64] = 1 << np.arange(64, dtype=np.uint64)
    b[:64] = np.uint64(2**64 - 1)
    ok = bool(np.array_equal(_native.gf_mul_device(a, b, 10), _native.gf_mul_device(a, b, 1)))
    print("lane table self-test vs bit-serial:", ok)
    out["lane_table_selftest"] = ok
    for v, name in NAMES.items():
        best = max(_native.gf_bench(v, 4096) for _ in range(3))
        out[name] = best
        print(f"{name:48s} {best:.3e}")
    sm = 148
    clk = 1.965e9
    out["per_sm_per_clock"] = {k: v / (sm * clk) for k, v in out.items() if "ops/s" in k}
    out["note"] = "best of 3 launches, full grid, SM clock assumed at its 1965 MHz maximum"
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)  # copied to profiles/ by hand
    with open(os.path.join(ROOT, "gpurun_out", "int_pipe_peaks.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()

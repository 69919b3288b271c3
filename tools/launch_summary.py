"""Summarize an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel.

    python tools/launch_summary.py gpurun_out/launches.csv
"""
import collections
import csv
import re
import sys

SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def short(name: str) -> str:
    m = re.search(r"(k_[a-z_0-9]+)(<[^()]*>)?", name)
    if not m:
        return name.split("(")[0].replace("void ", "")[:60]
    return m.group(1) + (m.group(2) or "")


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        us = float(r[iv].replace(",", "")) * SCALE.get(r[iu], 1.0)
        k = short(r[ik])
        agg[k][0] += 1
        agg[k][1] += us
    tot = sum(v[1] for v in agg.values())
    print(f"| kernel | launches | total ms | share | avg us |")
    print(f"|---|---:|---:|---:|---:|")
    for k, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| `{k}` | {n} | {us / 1e3:.3f} | {100 * us / tot:.1f}% | {us / n:.1f} |")


if __name__ == "__main__":
    main(sys.argv[1])

"""Opcode mix of one kernel section of an `ncu --page source --csv
--print-source sass` dump: warp-instructions executed per opcode, normalized
per unit of work.  Usage: python tools/sass_mix.py dump.csv SECTION UNITS"""
import csv
import re
import sys
from collections import Counter


def sections(path):
    cur, name = None, None
    with open(path) as f:
        for row in csv.reader(f):
            if row and row[0] == "Kernel Name":
                if cur is not None:
                    yield name, cur
                name, cur = row[1], []
            elif row and row[0] == "Address":
                hdr = row
            elif cur is not None and row:
                cur.append(dict(zip(hdr, row)))
    if cur is not None:
        yield name, cur


def main():
    path, which, units = sys.argv[1], int(sys.argv[2]), float(sys.argv[3])
    name, rows = list(sections(path))[which]
    mix, total = Counter(), 0
    for r in rows:
        n = int(r["Instructions Executed"] or 0)
        src = re.sub(r"^@!?U?P[T0-9]+\s+", "", r["Source"].strip())
        op = src.split()[0] if src else "?"
        op = op.split(".")[0]
        mix[op] += n
        total += n
    print(name)
    print(f"total warp-instr {total:.4g}  per unit (thread-instr) {32 * total / units:.1f}")
    for op, n in mix.most_common(25):
        print(f"  {op:10s} {32 * n / units:8.2f}")


if __name__ == "__main__":
    main()


def dump(path, which, units, pattern):
    """Lines of a section whose opcode matches `pattern`, with per-unit counts."""
    name, rows = list(sections(path))[which]
    for r in rows:
        n = int(r["Instructions Executed"] or 0)
        if n and re.search(pattern, r["Source"]):
            print(f"{32 * n / units:7.3f}  {r['Address'][-5:]}  {r['Source'].strip()}")

"""Per-source-line totals (instructions executed, stall samples) of one kernel
launch in an ncu report.  Usage: python tools/ncu_lines.py REP KERNEL_REGEX [SKIP] [TOP]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
skip = sys.argv[3] if len(sys.argv) > 3 else "0"
top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name",
                      f"regex:{kern}", "--launch-skip", skip, "--launch-count", "1",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
lines = []
cur = None
for r in rows:
    if len(r) > 4 and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    d = dict(zip(hdr[:4], r[:4]))
    ie = int(r[7]) if r[7].isdigit() else 0
    st = int(r[4]) if r[4].isdigit() else 0
    if r[0]:
        cur = [int(r[0]), r[1][:90], 0, 0]
        lines.append(cur)
    elif cur is not None:
        cur[2] += ie
        cur[3] += st
tot_i = sum(l[2] for l in lines) or 1
tot_s = sum(l[3] for l in lines) or 1
print(f"total warp-inst {tot_i}  stall samples {tot_s}")
for l in sorted(lines, key=lambda x: -x[2])[:top]:
    print(f"{l[0]:5d} inst {100*l[2]/tot_i:5.1f}%  stall {100*l[3]/tot_s:5.1f}%  {l[1]}")

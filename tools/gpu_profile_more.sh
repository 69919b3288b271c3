#!/bin/bash
# ncu captures of the kernels outside the wide level kernel: the grouped
# level kernel (W < 32, C5 x 0.1 at 16 points per batch) and the junction
# sieve of the default preprocessing (CLI on C2).  Plain runs first.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
tag=${1:-r1}
G="python bench.py --config 5 --scale 0.1 --points-per-batch 16 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0"
$G > gpurun_out/plain_grouped_$tag.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k k_level -s 0 -c 4 \
    -o gpurun_out/prof_grouped_$tag $G > gpurun_out/ncu_grouped_$tag.log 2>&1
echo "grouped rc=$?"
python - <<'PY'
import os, sys
sys.path.insert(0, ".")
from paper_2001_07158_b200 import synth
import pandas as pd
inst = synth.make_config(2)
pd.DataFrame({"u": inst.u, "v": inst.v, "ts": inst.ts}).to_csv(
    "gpurun_out/c2.edges", sep=" ", header=False, index=False)
with open("gpurun_out/c2.colors", "w") as f:
    f.write("".join(f"{i} {c}\n" for i, c in enumerate(inst.colors.tolist())))
PY
J="paper_2001_07158_b200/lib/tsieve decide --graph gpurun_out/c2.edges --colors gpurun_out/c2.colors --problem pathmotif --motif 1,1,2,3,4,5 --directed --preprocess both --format json"
$J > gpurun_out/plain_junction_$tag.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_static -c 6 \
    -o gpurun_out/prof_junction_$tag $J > gpurun_out/ncu_junction_$tag.log 2>&1
echo "junction rc=$?"
rm -f gpurun_out/c2.edges gpurun_out/c2.colors

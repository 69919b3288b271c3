#!/bin/bash
# ncu --set full of one middle-level item-stream launch on C4 x0.1 (level 7).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
tag=${1:-items}
CMD="python tools/probe_timing.py --config 4 --scale 0.1"
$CMD > gpurun_out/plain_$tag.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k_coef_items -s 5 -c 1 \
    -o gpurun_out/prof_$tag $CMD > gpurun_out/ncu_full_$tag.log 2>&1
echo "rc=$?"; tail -2 gpurun_out/ncu_full_$tag.log

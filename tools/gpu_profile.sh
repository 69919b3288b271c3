#!/bin/bash
# GPU-box profile of the C2 bench: plain run, per-launch device times, then
# one `ncu --set full` capture of one evaluation's level launches (level 2,
# the middle levels, and level k fused with the readout).
# Usage: gpurun -- bash tools/gpu_profile.sh [tag]
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
tag=${1:-r1}
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0"
$CMD > gpurun_out/plain_$tag.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$tag.csv $CMD > gpurun_out/ncu_launch_$tag.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k_level_wide -s 5 -c 5 \
    -o gpurun_out/prof_$tag $CMD > gpurun_out/ncu_full_$tag.log 2>&1
echo "rc=$?"
tail -3 gpurun_out/ncu_full_$tag.log

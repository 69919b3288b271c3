#!/bin/bash
# Bench line + launch list + one `ncu --set full` capture of one evaluation's
# coefficient-engine launches (C2).  Usage: gpurun -- bash tools/gpu_profile_coef.sh [tag]
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
tag=${1:-r1c}
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_$tag.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_$tag.log | cut -c1-600
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 0"
$CMD > gpurun_out/plain_$tag.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$tag.csv $CMD > gpurun_out/ncu_launch_$tag.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k_coef -s 40 -c 10 \
    -o gpurun_out/prof_$tag $CMD > gpurun_out/ncu_full_$tag.log 2>&1
echo "rc=$?"
tail -3 gpurun_out/ncu_full_$tag.log

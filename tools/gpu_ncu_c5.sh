#!/bin/bash
# ncu --set full of the C5 (x0.1) coefficient-engine kernels: one middle
# k_coef_arcs launch and one k_coef_ztrans_direct launch.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
CMD="python tools/probe_timing.py --config 5 --scale 0.1"
$CMD > gpurun_out/plain_c5.log 2>&1 && echo "plain rc=0" &&
ncu --set full --clock-control none --import-source on -k "regex:k_coef_arcs|k_coef_ztrans_direct" \
    -s 2 -c 3 -o gpurun_out/prof_c5_r1i $CMD > gpurun_out/ncu_c5.log 2>&1
echo "rc=$?"; tail -2 gpurun_out/ncu_c5.log

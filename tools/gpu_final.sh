#!/bin/bash
# Round check + capture: GPU suite, smoke, per-evaluation kernel timings
# (C2, C3, C4 x0.1, C5 x0.1), e2e breakdown, then the default bench line,
# launch list and one ncu --set full capture of one C2 evaluation
# (gpu_profile_coef.sh).  Usage: gpurun -- bash tools/gpu_final.sh [tag]
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
bash tools/gpu_round.sh
bash tools/gpu_profile_coef.sh ${1:-r1g}

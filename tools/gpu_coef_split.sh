#!/bin/bash
# Per-kernel split of one evaluation, coefficient vs point engine, several configs.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
out=gpurun_out/coef_split.log; : > $out
for cfg in "2 1.0" "3 1.0" "5 0.1" "4 0.1"; do
  set -- $cfg
  timeout 600 python tools/probe_timing.py --config $1 --scale $2 >> $out 2>&1
  TSV_ENGINE=points timeout 600 python tools/probe_timing.py --config $1 --scale $2 >> $out 2>&1
done
cat $out

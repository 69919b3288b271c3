#!/bin/bash
# GPU parity suite + per-kernel split of one evaluation on several configs.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
out=gpurun_out/zsplit.log; : > $out
for cfg in ${CFGS:-"2 1.0" "3 1.0" "4 0.1" "5 0.1"}; do
  set -- $cfg
  timeout 600 python tools/probe_timing.py --config $1 --scale $2 >> $out 2>&1
done
python - <<'PY'
import json
for line in open("gpurun_out/zsplit.log"):
    if not line.startswith("{"): print(line.strip()[:200]); continue
    d=json.loads(line); k=d["kernels"]
    print(d["config"], d["scale"], {n:v["ms_per_eval"] for n,v in k.items()})
PY

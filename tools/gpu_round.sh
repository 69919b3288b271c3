#!/bin/bash
# Round check: GPU suite, smoke, per-evaluation kernel timings (C2, C3,
# C4 x0.1, C5 x0.1), the e2e breakdown of C2 and the default bench line.
# Usage: gpurun -- bash tools/gpu_round.sh
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
out=gpurun_out/round_pt.log; : > $out
for cfg in "2" "3" "4 --scale 0.1" "5 --scale 0.1"; do
  timeout 600 python tools/probe_timing.py --config $cfg >> $out 2>&1
done
python - <<'PY'
import json
for line in open("gpurun_out/round_pt.log"):
    if not line.startswith("{"): print(line.strip()[:200]); continue
    d=json.loads(line); k=d["kernels"]
    print(d["config"], d["scale"], "build", round(d["build_s"], 3), "probes", [p["s"] for p in d["probes"]][:4], {n:v["ms_per_eval"] for n,v in k.items()})
PY
timeout 300 python tools/e2e_breakdown.py > gpurun_out/e2e_breakdown.log 2>&1; tail -12 gpurun_out/e2e_breakdown.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log | cut -c1-300

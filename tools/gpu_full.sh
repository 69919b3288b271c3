#!/bin/bash
# Full-size per-evaluation timings: C4 (n=1e6, m=1e8, k_eff=12) and C5
# (n=1e8, m=1e9, k=5) with the coefficient engine.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
out=gpurun_out/full_pt.log; : > $out
timeout 1500 python tools/probe_timing.py --config 5 >> $out 2>&1; echo "c5 rc=$?"
timeout 1500 python tools/probe_timing.py --config 4 >> $out 2>&1; echo "c4 rc=$?"
python - <<'PY'
import json
for line in open("gpurun_out/full_pt.log"):
    if not line.startswith("{"): print(line.strip()[:300]); continue
    d=json.loads(line); k=d["kernels"]
    print(d["config"], d["scale"], "build", round(d["build_s"], 3), "probes", [p["s"] for p in d["probes"]][:4], {n:v["ms_per_eval"] for n,v in k.items()})
PY

#!/bin/bash
# Per-evaluation timings: C2 with both arc kernels, C3 full, C4 x0.1, C5 x0.1 and full.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
out=gpurun_out/sizes.log; : > $out
TSV_ITEMS=0 timeout 300 python tools/probe_timing.py --config 2 >> $out 2>&1
TSV_ITEMS=1 timeout 300 python tools/probe_timing.py --config 2 >> $out 2>&1
timeout 600 python tools/probe_timing.py --config 3 >> $out 2>&1
TSV_ITEMS=0 timeout 600 python tools/probe_timing.py --config 3 >> $out 2>&1
timeout 600 python tools/probe_timing.py --config 4 --scale 0.1 >> $out 2>&1
TSV_ENGINE=points timeout 600 python tools/probe_timing.py --config 3 >> $out 2>&1
timeout 1200 python tools/probe_timing.py --config 5 >> $out 2>&1
python - <<'PY'
import json
for line in open("gpurun_out/sizes.log"):
    if not line.startswith("{"): print(line.strip()[:300]); continue
    d=json.loads(line); k=d["kernels"]
    print(d["config"], d["scale"], "build", round(d["build_s"],2), "probes", [p["s"] for p in d["probes"]], {n:v["ms_per_eval"] for n,v in k.items()})
PY

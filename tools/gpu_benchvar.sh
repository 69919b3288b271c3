#!/bin/bash
# Run-to-run variance of the default bench step (4 runs, no CPU arm, no e2e),
# and per-evaluation timings of the persistent item kernel on / off.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_gpu.log
for i in 1 2 3 4; do
  timeout 300 python bench.py --no-cpu-baseline --e2e-steps 0 > gpurun_out/bv_$i.log 2>&1
  tail -1 gpurun_out/bv_$i.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('run', $i, round(d['ms_per_step'],3), 'ms/step', round(d['kernel_ms_per_step']['all'],3), d['clocks'])"
done
out=gpurun_out/bv_pt.log; : > $out
for cfg in 2 3; do
  TSV_PERSIST=0 timeout 300 python tools/probe_timing.py --config $cfg >> $out 2>&1
  timeout 300 python tools/probe_timing.py --config $cfg >> $out 2>&1
done
python - <<'PY'
import json
for line in open("gpurun_out/bv_pt.log"):
    if not line.startswith("{"): print(line.strip()[:200]); continue
    d=json.loads(line); k=d["kernels"]
    print(d["config"], d["scale"], {n:v["ms_per_eval"] for n,v in k.items()})
PY

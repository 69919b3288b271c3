#!/bin/bash
# Quick GPU-box check: parity tests, then C2 bench for each y-multiply path.
# Usage (from the build container): gpurun -- bash tools/gpu_quick.sh [modes...]
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
tail -2 gpurun_out/pytest_gpu.log
modes="${@:-table}"
for m in $modes; do
  TSV_YMUL=$m timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0 \
    > gpurun_out/bench_$m.log 2>&1
  python - "$m" <<'PY'
import json, sys
m = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/bench_{m}.log").read().strip().splitlines()[-1])
    r = d["roofline"]
    print(f"{m}: {d['value']:.3e} upd/s  level {r['avg_launch_ms']:.3f} ms  frac {r['frac']:.3f}  {d['checksums']}")
except Exception as e:
    print(m, "FAILED", e, open(f"gpurun_out/bench_{m}.log").read()[-800:])
PY
done

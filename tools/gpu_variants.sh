#!/bin/bash
# Bench the default engine and every exp_libs/libtsv_*.so variant on one box.
# Usage: gpurun -- bash tools/gpu_variants.sh [bench args...]
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
args="${@:---steps 3 --warmup 2}"
for lib in default exp_libs/libtsv_*.so; do
  tag=$(basename "$lib" .so)
  if [ "$lib" = default ]; then unset TSV_LIB; else export TSV_LIB=$PWD/$lib; fi
  timeout 600 python bench.py $args --no-cpu-baseline --e2e-steps 0 > gpurun_out/var_$tag.log 2>&1
  python - "$tag" <<'PY'
import json, sys
t = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/var_{t}.log").read().strip().splitlines()[-1])
    r = d["roofline"] or {}
    print(f"{t:14s} {d['value']:.4e} upd/s  step {d['ms_per_step']:.3f} ms  mid {r.get('avg_launch_ms', 0):.4f} ms  "
          f"kern {d['kernel_ms_per_step']}  {d['checksums'][:2]}")
except Exception as e:
    print(t, "FAILED", e, open(f"gpurun_out/var_{t}.log").read()[-600:])
PY
done

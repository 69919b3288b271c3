#!/bin/bash
# Probe timings (C2, C3, C5 x0.1) of the default engine and every
# exp_libs/libtsv_*.so variant.  Usage: gpurun -- bash tools/gpu_var_pt.sh
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "coefficient_engine_kernels or golden" > gpurun_out/var_test.log 2>&1; echo "variant test rc=$?"; tail -2 gpurun_out/var_test.log
out=gpurun_out/var_pt.log; : > $out
for lib in default exp_libs/libtsv_*.so; do
  if [ "$lib" = default ]; then unset TSV_LIB; else export TSV_LIB=$PWD/$lib; fi
  for cfg in "2" "3" "5 --scale 0.1"; do
    echo "# $lib $cfg" >> $out
    timeout 300 python tools/probe_timing.py --config $cfg >> $out 2>&1
  done
done
python - <<'PY'
import json
for line in open("gpurun_out/var_pt.log"):
    if line.startswith("#"): print(line.strip()); continue
    if not line.startswith("{"): print(line.strip()[:200]); continue
    d=json.loads(line); k=d["kernels"]
    print("  ", d["config"], d["scale"], {n:v["ms_per_eval"] for n,v in k.items()})
PY

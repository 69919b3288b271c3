#!/bin/bash
# Register-walk item kernel: variant parity test, GPU suite, C2/C3/C5 probe
# timings with and without it, then bench + launch list + ncu capture
# (gpu_profile_coef.sh).  Usage: gpurun -- bash tools/gpu_reg.sh [tag]
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k coefficient_engine_kernels > gpurun_out/reg_test.log 2>&1; echo "variant test rc=$?"; tail -3 gpurun_out/reg_test.log
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
out=gpurun_out/reg_pt.log; : > $out
for cfg in "2" "3" "5 --scale 0.1"; do
  TSV_ITEMS_REG=0 timeout 300 python tools/probe_timing.py --config $cfg >> $out 2>&1
  timeout 300 python tools/probe_timing.py --config $cfg >> $out 2>&1
done
python - <<'PY'
import json
for line in open("gpurun_out/reg_pt.log"):
    if not line.startswith("{"): print(line.strip()[:300]); continue
    d=json.loads(line); k=d["kernels"]
    print(d["config"], d["scale"], "probes", [p["s"] for p in d["probes"]][:4], {n:v["ms_per_eval"] for n,v in k.items()})
PY
bash tools/gpu_profile_coef.sh ${1:-r1f}

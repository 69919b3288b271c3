#!/bin/bash
# Direct z map of multi-shade rows: variant parity test, GPU suite, C2/C5
# probe timings (direct vs table), bench with 2 and 4 streams.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k coefficient_engine_kernels > gpurun_out/zd_test.log 2>&1; echo "variant test rc=$?"; tail -3 gpurun_out/zd_test.log
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
out=gpurun_out/zd_pt.log; : > $out
for cfg in "2" "5 --scale 0.1"; do
  TSV_ZTRANS=tab timeout 300 python tools/probe_timing.py --config $cfg >> $out 2>&1
  timeout 300 python tools/probe_timing.py --config $cfg >> $out 2>&1
done
python - <<'PY'
import json
for line in open("gpurun_out/zd_pt.log"):
    if not line.startswith("{"): print(line.strip()[:300]); continue
    d=json.loads(line); k=d["kernels"]
    print(d["config"], d["scale"], "probes", [p["s"] for p in d["probes"]][:4], {n:v["ms_per_eval"] for n,v in k.items()})
PY
for s in 2 4; do
timeout 600 python bench.py --steps 50 --warmup 3 --streams $s --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_s$s.log 2>&1; echo "bench streams=$s rc=$?"; tail -1 gpurun_out/bench_s$s.log | cut -c1-330
done

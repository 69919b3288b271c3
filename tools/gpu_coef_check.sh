#!/bin/bash
# Coefficient engine: GPU parity suite (default engine) + probe timings of both engines.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/coef_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/coef_pytest.log
timeout 300 python tools/probe_timing.py > gpurun_out/coef_pt.log 2>&1
TSV_ENGINE=points timeout 300 python tools/probe_timing.py >> gpurun_out/coef_pt.log 2>&1
cat gpurun_out/coef_pt.log

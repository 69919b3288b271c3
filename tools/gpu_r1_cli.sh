#!/bin/bash
# GPU-box check of the C++ drop-in at scale: GPU tests, then the CLI on C2
# and C5 x 0.1 text files (tools/cli_at_scale.py).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python tools/cli_at_scale.py --config 2 --preprocess none both --commands decide extract \
  --extraction localized self-reducible > gpurun_out/cli_c2.log 2>&1; echo "cli c2 rc=$?"
cut -c1-400 gpurun_out/cli_c2.log
timeout 1500 python tools/cli_at_scale.py --config 5 --scale ${C5_SCALE:-0.1} --preprocess none \
  --commands decide > gpurun_out/cli_c5.log 2>&1; echo "cli c5 rc=$?"
cut -c1-600 gpurun_out/cli_c5.log

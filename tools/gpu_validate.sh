#!/bin/bash
# Round-end style validation on one B200: GPU tests, smoke(), the default
# bench line, the reference arm, and the CLI at C2 scale.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/val_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/val_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/val_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/val_smoke.log
timeout 900 python bench.py > gpurun_out/val_bench.log 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/val_ref.log 2>&1; echo "ref rc=$?"
timeout 900 python tools/cli_at_scale.py --config 2 --preprocess none both --commands decide extract > gpurun_out/val_cli.log 2>&1; echo "cli rc=$?"

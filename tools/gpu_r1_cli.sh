cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python tools/cli_at_scale.py --config 2 --preprocess none both --commands decide extract --extraction localized self-reducible > gpurun_out/cli_c2.log 2>&1; echo "cli c2 rc=$?"
cat gpurun_out/cli_c2.log | cut -c1-600
timeout 1500 python tools/cli_at_scale.py --config 5 --scale 0.1 --preprocess none --commands decide > gpurun_out/cli_c5.log 2>&1; echo "cli c5 rc=$?"
cat gpurun_out/cli_c5.log | cut -c1-600
free -g | head -2; nproc

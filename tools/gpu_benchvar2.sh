#!/bin/bash
# Bench step variance: 4 runs with the NVML clock sampler, 4 without, 2 with one stream.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
run() {
  timeout 300 python bench.py --no-cpu-baseline --e2e-steps 0 "$@" > gpurun_out/bv.log 2>&1
  tail -1 gpurun_out/bv.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), 'ms/step', round(d['kernel_ms_per_step']['all'],3), d['clocks'].get('samples'))"
}
for i in 1 2 3 4; do echo -n "sampler: "; run; done
for i in 1 2 3 4; do echo -n "no sampler: "; BENCH_NO_CLOCKS=1 run; done
for i in 1 2; do echo -n "1 stream: "; run --streams 1; done
for i in 1 2; do echo -n "200 steps: "; run --steps 200; done

#!/bin/bash
# bench.py on every BASELINE config (short runs) to check the line for each.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
for c in "1" "3" "4 --scale 0.1" "5 --scale 0.1"; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/cfg.log 2>&1
  echo "config $c rc=$?"
  tail -1 gpurun_out/cfg.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(' ', d['config']['workload'], round(d['ms_per_step'],3), 'ms', '%.3e' % d['value'], 'e2e %.3e' % d['e2e']['value'], d['roofline'] and round(d['roofline']['frac'],3), d['decision'])" 2>&1 | tail -2
done

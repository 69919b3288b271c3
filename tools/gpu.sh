#!/bin/bash
# One driver for every GPU-box job (run it under gpurun):
#
#   gpurun --timeout S -- bash tools/gpu.sh JOB [JOB ...]
#
# Jobs run in order; each writes its log under gpurun_out/ and prints a
# one-line summary.  A JOB is NAME or NAME:ARG1,ARG2,...
#
#   box                      host CPU model / cores / RAM, GPU name -> box.txt
#   tests[:PYTEST-ARGS]      pytest -m gpu (extra args, e.g. -k,full)   -> pytest_gpu.log
#   smoke                    __graft_entry__.smoke()                     -> smoke.log
#   timings:CFG[,SCALE]      tools/probe_timing.py (per-kernel times of one evaluation)
#   bench[:ARGS]             bench.py ARGS (comma-separated)             -> bench_<i>.log
#   ref[:ARGS]               bench.py --impl reference ARGS              -> ref_<i>.log
#   launches:TAG[,ARGS]      ncu launch list of `bench.py --steps 1 --warmup 3 ARGS`
#   ncu:TAG,REGEX,SKIP,COUNT[,ARGS]
#                            ncu --set full of the matching launches of the same command
#   ncueval:TAG,REGEX,SKIP,COUNT,CFG[,SCALE]
#                            ncu --set full of `tools/one_eval.py CFG SCALE 2`
#   launcheval:TAG,CFG[,SCALE]
#                            ncu launch list (gpu__time_duration) of the same
#   launchpy:TAG,SCRIPT[,ARGS]
#                            ncu launch list (gpu__time_duration) of python SCRIPT ARGS
#   sanitize:TOOL[,K]        compute-sanitizer --tool TOOL over pytest -m gpu -k K
#   py:SCRIPT[,ARGS]         python SCRIPT ARGS                          -> py_<i>.log
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
i=0
for job in "$@"; do
  i=$((i + 1))
  name=${job%%:*}
  arg=""; [[ "$job" == *:* ]] && arg=${job#*:}
  IFS=',' read -r -a A <<< "$arg"
  # ENV=VALUE jobs set an environment variable for the jobs after them
  if [[ "$name" == *=* ]]; then export "$job"; echo "env $job"; continue; fi
  case $name in
    box)
      (nproc; lscpu | grep -E "Model name|Socket|Thread|Core|NUMA node\(s\)"; free -g;
       nvidia-smi --query-gpu=name,memory.total,clocks.sm,clocks.max.sm --format=csv) > gpurun_out/box.txt 2>&1
      cat gpurun_out/box.txt ;;
    tests)
      timeout 2400 python -m pytest tests -q -m gpu -x "${A[@]}" > gpurun_out/pytest_gpu.log 2>&1
      echo "tests rc=$?"; tail -3 gpurun_out/pytest_gpu.log ;;
    smoke)
      timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
      echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log ;;
    timings)
      out=gpurun_out/timings_${A[0]}_${A[1]:-1}_$i.log
      timeout 1800 python tools/probe_timing.py --config "${A[0]}" --scale "${A[1]:-1.0}" > $out 2>&1
      echo "timings ${A[*]} rc=$?"; tail -c 1200 $out; echo ;;
    bench)
      out=gpurun_out/bench_$i.log
      timeout 1800 python bench.py "${A[@]}" > $out 2>&1
      echo "bench ${A[*]} rc=$?"; tail -c 3000 $out; echo ;;
    ref)
      out=gpurun_out/ref_$i.log
      timeout 1800 python bench.py --impl reference "${A[@]}" > $out 2>&1
      echo "ref ${A[*]} rc=$?"; tail -c 1500 $out; echo ;;
    launches)
      tag=${A[0]}; rest=("${A[@]:1}")
      CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 ${rest[*]}"
      $CMD > gpurun_out/plain_$tag.log 2>&1 && echo "plain rc=0" &&
      timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
          --log-file gpurun_out/launches_$tag.csv $CMD > gpurun_out/ncu_launch_$tag.log 2>&1
      echo "launches $tag rc=$?" ;;
    ncu)
      tag=${A[0]}; rx=${A[1]}; skip=${A[2]}; cnt=${A[3]}; rest=("${A[@]:4}")
      CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 ${rest[*]}"
      $CMD > gpurun_out/plain_ncu_$tag.log 2>&1 && echo "plain rc=0" &&
      timeout 3000 ncu --set full --clock-control none --import-source on -k "regex:$rx" \
          -s "$skip" -c "$cnt" -o gpurun_out/prof_$tag $CMD > gpurun_out/ncu_full_$tag.log 2>&1
      echo "ncu $tag rc=$?"; tail -2 gpurun_out/ncu_full_$tag.log ;;
    ncueval)
      tag=${A[0]}; rx=${A[1]}; skip=${A[2]}; cnt=${A[3]}
      CMD="python tools/one_eval.py ${A[4]} ${A[5]:-1.0} 2"
      $CMD > gpurun_out/plain_ncu_$tag.log 2>&1 && echo "plain rc=0" && tail -2 gpurun_out/plain_ncu_$tag.log &&
      timeout 3000 ncu --set full --clock-control none --import-source on -k "regex:$rx" \
          -s "$skip" -c "$cnt" -o gpurun_out/prof_$tag $CMD > gpurun_out/ncu_full_$tag.log 2>&1
      echo "ncueval $tag rc=$?"; tail -2 gpurun_out/ncu_full_$tag.log ;;
    launcheval)
      tag=${A[0]}
      CMD="python tools/one_eval.py ${A[1]} ${A[2]:-1.0} 2"
      timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
          --log-file gpurun_out/launches_$tag.csv $CMD > gpurun_out/ncu_launch_$tag.log 2>&1
      echo "launcheval $tag rc=$?"; tail -3 gpurun_out/ncu_launch_$tag.log ;;
    launchpy)
      tag=${A[0]}; rest=("${A[@]:1}")
      timeout 2400 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
          --log-file gpurun_out/launches_$tag.csv python "${rest[@]}" > gpurun_out/ncu_launch_$tag.log 2>&1
      echo "launchpy $tag rc=$?"; tail -3 gpurun_out/ncu_launch_$tag.log ;;
    sanitize)
      tool=${A[0]}; k=${A[1]:-small}
      timeout 2400 compute-sanitizer --tool "$tool" --print-limit 20 \
          python -m pytest tests -q -m gpu -x -k "$k" -p no:cacheprovider > gpurun_out/sanitize_$tool.log 2>&1
      echo "sanitize $tool rc=$?"; tail -5 gpurun_out/sanitize_$tool.log ;;
    py)
      out=gpurun_out/py_$i.log
      timeout 3000 python "${A[@]}" > $out 2>&1
      echo "py ${A[*]} rc=$?"; tail -c 2500 $out; echo ;;
    *) echo "unknown job $job" ;;
  esac
done

#!/bin/bash
# lane-group tier: parity + timing vs the thread tier on configs 1-5
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/group_tests.log
for c in "1 1.0" "2 1.0" "3 1.0" "4 1.0" "5 0.2"; do
  set -- $c
  for f in 0 32 64; do
    echo "flags $f: $(timeout 300 python scripts/prof_run.py --config $1 --scale $2 --runs 3 --flags $f 2>&1 | tail -1)"
  done
done > gpurun_out/group_prof.log 2>&1
cat gpurun_out/group_tests.log gpurun_out/group_prof.log

#!/bin/bash
# start-tier sweep for the latency-bound configs (lane groups forced: 32|8|t<<8)
mkdir -p gpurun_out
for c in "1 1.0" "2 1.0" "3 1.0"; do
  set -- $c
  for f in 0 40 296 552 808 1064; do
    echo "cfg $1 flags $f: $(timeout 300 python scripts/prof_run.py --config $1 --scale $2 --runs 3 --flags $f 2>&1 | tail -1 | sed 's/.*tiers ms/tiers ms/')"
  done
done > gpurun_out/tiers_sweep.log 2>&1
cat gpurun_out/tiers_sweep.log

#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
for c in "3 1.0 0" "3 10 0" "3 10 64" "5 0.2 0" "1 1.0 0" "2 1.0 0"; do
  set -- $c
  echo "cfg $1 x$2 flags $3: $(timeout 300 python scripts/prof_run.py --config $1 --scale $2 --runs 3 --flags $3 2>&1 | tail -1 | sed 's/.*tiers ms/tiers ms/')"
done

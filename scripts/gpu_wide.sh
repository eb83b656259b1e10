#!/bin/bash
for w in 0 1; do
  for c in "1 1.0" "2 1.0" "3 1.0" "5 0.2"; do
    set -- $c
    echo "wide $w cfg $1: $(XB_GROUP_WIDE=$w timeout 300 python scripts/prof_run.py --config $1 --scale $2 --runs 3 2>&1 | tail -1 | sed 's/.*tiers ms/tiers ms/')"
  done
done

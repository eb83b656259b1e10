#!/bin/bash
# A/B: device time of the bench workload for (library, flags) pairs on one box.
# usage: RUNS="lib:flags lib:flags ..." bash scripts/ab_flags.sh
for spec in ${RUNS}; do
  lib=${spec%%:*}; fl=${spec##*:}
  for i in 1 2; do
    echo "$lib flags=$fl: $(XB_LIB_PATH=$lib timeout 400 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --e2e-steps 1 --flags $fl 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); t=d["tiers"]; print(round(d["value"],1), round(d["ms_per_step"],2), t["start_tier"], [round(x,2) for x in t["ms"]], t["escalated"])')"
  done
done

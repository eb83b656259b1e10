#!/bin/bash
# A/B: device time of the bench workload with two library builds on one box
for lib in ${LIBS}; do
  for i in 1 2; do
    echo "$lib: $(XB_LIB_PATH=$lib timeout 400 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1), round(d["ms_per_step"],2), [round(x,2) for x in d["tiers"]["ms"][:3]])')"
  done
done

#!/bin/bash
# Latency-bound configs: device ms per step vs resident lane-group blocks per
# SM of the start tier ("default" = the engine's own choice).
for cfg in ${CFGS:-1 2 3}; do
  for b in ${BLOCKS:-default 4 3 2 1}; do
    if [ "$b" = default ]; then envs=""; else envs="XB_LATENCY_BLOCKS=$b"; fi
    echo "cfg$cfg blocks=$b: $(env $envs timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); t=d["tiers"]; print(round(d["value"],1), round(d["ms_per_step"],3), t["start_tier"], [round(x,2) for x in t["ms"]])')"
  done
done

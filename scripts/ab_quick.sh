#!/bin/bash
# Quick A/B evidence for a kernel change: GPU parity, latency-bound configs,
# device GCUPS of config 5 and config 4 (no CPU baseline, one e2e step).
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -1
timeout 300 python scripts/lat_probe.py --configs ${LAT_CFGS:-1,2,3} --settings default
for c in ${BENCH_CFGS:-5 4}; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | \
    python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("cfg", d["config"]["workload"], round(d["value"],1), "GCUPS", round(d["ms_per_step"],3), "ms frac", round(d["roofline"]["frac"],4), "sm_mhz", d["clocks"]["sm_mhz"])'
done

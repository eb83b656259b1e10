#!/bin/bash
# parity + timing (C5 by default; CONFIGS="1 2 3" etc.) + (NCU=1) one full ncu capture
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/q_tests.log
ok=1
for c in ${CONFIGS:-5}; do
  sc=1.0; [ $c = 5 ] && sc=${SCALE:-0.2}; [ $c = 4 ] && sc=0.2
  for f in ${FLAGS:-0 64}; do
    out=$(timeout 300 python scripts/prof_run.py --config $c --scale $sc --runs 3 --flags $f 2>&1) || ok=0
    echo "cfg $c flags $f: $(echo "$out" | tail -1 | sed 's/.*tiers ms/tiers ms/')"
  done
done > gpurun_out/q_prof.log 2>&1
cat gpurun_out/q_tests.log gpurun_out/q_prof.log
if [ -n "$NCU" ] && [ $ok = 1 ]; then
  ncu --set full --import-source on --clock-control none -k regex:thread_tier_kernel --launch-skip 1 -c 1 \
    -o gpurun_out/q_k24 -f python scripts/prof_run.py --config 5 --scale 0.2 --runs 1 --flags 64 > gpurun_out/q_ncu.log 2>&1
  tail -2 gpurun_out/q_ncu.log
fi

#!/bin/bash
# parity + C5 timing + (NCU=1) one full ncu capture of the start-tier kernel
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/q_tests.log
ok=1
for f in 0 64; do
  out=$(timeout 300 python scripts/prof_run.py --config 5 --scale ${SCALE:-0.2} --runs 3 --flags $f 2>&1) || ok=0
  echo "flags $f: $(echo "$out" | tail -1)"
done > gpurun_out/q_prof.log 2>&1
cat gpurun_out/q_tests.log gpurun_out/q_prof.log
if [ -n "$NCU" ] && [ $ok = 1 ]; then
  ncu --set full --import-source on --clock-control none -k regex:thread_tier_kernel --launch-skip 2 -c 1 \
    -o gpurun_out/q_k24 -f python scripts/prof_run.py --config 5 --scale 0.2 --runs 1 --flags 64 > gpurun_out/q_ncu.log 2>&1
  tail -2 gpurun_out/q_ncu.log
fi

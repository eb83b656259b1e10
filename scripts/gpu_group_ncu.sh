#!/bin/bash
mkdir -p gpurun_out
python scripts/prof_run.py --config 1 --scale 1.0 --runs 1 --flags 40 > gpurun_out/g_c1.log 2>&1 || exit 1
python scripts/prof_run.py --config 1 --scale 1.0 --runs 1 --flags 72 >> gpurun_out/g_c1.log 2>&1 || exit 1
ncu --set full --import-source on --clock-control none -k regex:group_tier -c 1 -o gpurun_out/g_c1_group -f \
  python scripts/prof_run.py --config 1 --scale 1.0 --runs 1 --flags 40 > gpurun_out/ncu1.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:thread_tier -c 1 -o gpurun_out/g_c1_thread -f \
  python scripts/prof_run.py --config 1 --scale 1.0 --runs 1 --flags 72 > gpurun_out/ncu2.log 2>&1
cat gpurun_out/g_c1.log; tail -3 gpurun_out/ncu1.log gpurun_out/ncu2.log

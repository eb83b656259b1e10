mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -5
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench2.json 2> gpurun_out/bench2.log; echo "bench rc=$?"
cat gpurun_out/bench2.json
python scripts/prof_run.py --scale 0.05 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:thread_tier -c 1 -o gpurun_out/prof_t0 python scripts/prof_run.py --scale 0.05 > gpurun_out/ncu_full.log 2>&1; echo "ncu rc=$?"
cat gpurun_out/prof_plain.log
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_plain.json 2>/dev/null && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_launches.log 2>&1; echo "ncu2 rc=$?"

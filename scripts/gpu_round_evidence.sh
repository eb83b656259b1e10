# Full evidence run: GPU tests, bench line, launch list, ncu of the top kernel.
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print(\"smoke ok\")" 2>&1 | tail -2
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -5
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.log; echo "bench rc=$?"
cat gpurun_out/bench.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.log; echo "ref rc=$?"
cat gpurun_out/bench_ref.json
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_plain.json 2>/dev/null && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_launches.log 2>&1; echo "ncu-launches rc=$?"
python scripts/prof_run.py --config 5 --scale 1.0 --runs 1 > gpurun_out/prof_full_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:thread_tier_kernelILi24ELi0E -c 1 -o gpurun_out/prof_main python scripts/prof_run.py --config 5 --scale 1.0 --runs 1 > gpurun_out/ncu_main.log 2>&1; echo "ncu-main rc=$?"

# Evidence: tests, bench, reference arm, launch list (ncu), full ncu of the K24 start tier,
# per-config report.  Every ncu run under its own timeout (ncu serialises kernels).
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.log; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.log; echo "ref rc=$?"
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_plain.json 2>/dev/null && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_launches.log 2>&1; echo "ncu-launches rc=$?"
timeout 600 python scripts/prof_run.py --config 5 --scale 1.0 --runs 1 > gpurun_out/prof_full_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:thread_tier_kernelILi24ELi0E -c 1 -o gpurun_out/prof_main python scripts/prof_run.py --config 5 --scale 1.0 --runs 1 > gpurun_out/ncu_main.log 2>&1; echo "ncu-main rc=$?"
timeout 1500 python scripts/config_report.py --out gpurun_out/configs > gpurun_out/configs.log 2>&1; echo "configs rc=$?"

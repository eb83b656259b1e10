mkdir -p gpurun_out
timeout 900 python scripts/shard_balance.py --n 8
timeout 900 python scripts/shard_balance.py --n 2
timeout 600 python scripts/prof_run.py --config 4 --scale 1.0 --x 100 --runs 2
timeout 600 python bench.py --config 4 --x 100 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/bench_c4x100.json 2> gpurun_out/bench_c4x100.err; echo "bench rc=$?"; tail -c 600 gpurun_out/bench_c4x100.json
M="gpu__time_duration.sum,smsp__inst_executed.sum,smsp__thread_inst_executed.sum,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum"
timeout 900 ncu --metrics $M --clock-control none -k regex:wide_tier_kernel --csv python scripts/prof_run.py --config 4 --scale 0.2 --x 100 --runs 1 --flags 1288 > gpurun_out/ncu_wide_c4x100.csv 2>&1; echo "ncu rc=$?"
timeout 900 ncu --metrics $M --clock-control none -k regex:thread_tier_kernel --csv python scripts/prof_run.py --config 4 --scale 0.2 --runs 1 --flags 128 > gpurun_out/ncu_k64_c4.csv 2>&1; echo "ncu rc=$?"

# Round-2 evidence: tests (product and bounds-checked builds), smoke, bench + reference arm,
# launch list (ncu), full ncu of the K24 start tier and of the wide K128 tier, the per-config
# report.  Every ncu run under its own timeout; .ncu-rep files are summarised and removed
# (gpurun_out/ must stay under 64 MiB to come back).
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
XB_LIB_PATH=$PWD/paper_2304_08662_b200/_lib/libxdrop_b200_checked.so timeout 2400 python -m pytest tests -q -m gpu -k "not full_size_every_row" 2>&1 | tail -2
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.log; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.log; echo "ref rc=$?"
timeout 900 python bench.py --config 4 --x 100 --steps 3 --warmup 3 --e2e-steps 2 --no-cpu-baseline > gpurun_out/bench_c4x100.json 2> gpurun_out/bench_c4x100.log; echo "bench c4x100 rc=$?"
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_plain.json 2>/dev/null && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_launches.log 2>&1; echo "ncu-launches rc=$?"
timeout 1200 ncu --set full --clock-control none --kernel-name-base mangled -k regex:wide_tier_kernelILi128ELi8ELi0E -c 1 -o gpurun_out/prof_wide python scripts/prof_run.py --config 4 --scale 1.0 --x 100 --runs 1 > gpurun_out/ncu_wide.log 2>&1; echo "ncu-wide rc=$?"
python scripts/ncu_summary.py report gpurun_out/prof_wide.ncu-rep gpurun_out/r2_wide_k128_config4_x100.txt; rm -f gpurun_out/prof_wide.ncu-rep
timeout 1500 python scripts/config_report.py --out gpurun_out/r2_configs > gpurun_out/configs.log 2>&1; echo "configs rc=$?"
# lane tiers (xb_lane.cu): config 1 runs on them; summary of one full capture, and the
# longest task alone under both several-lanes-per-unit families (cycles per antidiagonal)
timeout 600 ncu --set full --clock-control none -k regex:lane_tier -c 1 -o gpurun_out/prof_lane python scripts/prof_run.py --config 1 --scale 1.0 --runs 1 > gpurun_out/ncu_lane.log 2>&1; echo "ncu-lane rc=$?"
python scripts/ncu_summary.py report gpurun_out/prof_lane.ncu-rep gpurun_out/r2_lane_k16_config1.txt; rm -f gpurun_out/prof_lane.ncu-rep
for fam in 4 8; do echo "== XB_GROUP_FAMILY=$fam"; XB_GROUP_FAMILY=$fam timeout 600 python scripts/lat_probe.py --configs 1,2,3 --settings default,g0,g2; done > gpurun_out/r2_lat_probe.txt 2>&1

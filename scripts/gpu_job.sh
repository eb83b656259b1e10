mkdir -p gpurun_out
timeout 300 python scripts/lat_probe.py --configs 2 --alone-only --settings g2 > gpurun_out/lat.log 2>&1; cat gpurun_out/lat.log
T=$(python -c "import json;print(json.loads(open('gpurun_out/lat.log').readline())['longest_task'])")
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base mangled -k regex:group_tier_kernelILi32ELi4ELi0E -c 1 -o gpurun_out/gsrc python scripts/lat_probe.py --configs 2 --alone-only --task $T --settings g2 > gpurun_out/ncu_gsrc.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/gsrc.ncu-rep --page source --csv --print-source sass > gpurun_out/gsrc.csv 2>/dev/null
python scripts/ncu_summary.py report gpurun_out/gsrc.ncu-rep gpurun_out/r2_group_k32_c2_alone.txt; rm -f gpurun_out/gsrc.ncu-rep

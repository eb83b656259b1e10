mkdir -p gpurun_out
./build/lat_bench
python scripts/prof_run.py --config 5 --scale 0.2 > gpurun_out/p7a.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:ILi24ELi0E -c 1 -o gpurun_out/prof_k24b python scripts/prof_run.py --config 5 --scale 0.2 > gpurun_out/ncu7a.log 2>&1; echo "ncu rc=$?"
python scripts/prof_run.py --config 2 --scale 1.0 > gpurun_out/p7b.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:ILi24ELi0E -c 1 -o gpurun_out/prof_c2 python scripts/prof_run.py --config 2 --scale 1.0 > gpurun_out/ncu7b.log 2>&1; echo "ncu rc=$?"
cat gpurun_out/p7a.log gpurun_out/p7b.log

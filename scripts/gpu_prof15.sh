mkdir -p gpurun_out
python scripts/prof_run.py --config 5 --scale 0.2 > gpurun_out/p15.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:ILi24ELi0E -c 1 -o gpurun_out/prof_k24e python scripts/prof_run.py --config 5 --scale 0.2 > gpurun_out/ncu15.log 2>&1; echo "ncu rc=$?"
cat gpurun_out/p15.log

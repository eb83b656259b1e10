mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -4
for c in 2 4 5; do python scripts/prof_run.py --config $c --scale 1.0 --runs 2; done
python scripts/prof_run.py --config 5 --scale 0.2 > gpurun_out/p12.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:ILi24ELi0E -c 1 -o gpurun_out/prof_k24d python scripts/prof_run.py --config 5 --scale 0.2 > gpurun_out/ncu12.log 2>&1; echo "ncu rc=$?"

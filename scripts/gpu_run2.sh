mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -15
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench1.json 2> gpurun_out/bench1.log; echo "bench rc=$?"
cat gpurun_out/bench1.json; tail -5 gpurun_out/bench1.log

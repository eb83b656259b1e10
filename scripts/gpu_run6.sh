mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -15
for c in 1 2 3 4 5; do python scripts/prof_run.py --config $c --scale 1.0 --runs 2; done
python scripts/prof_run.py --config 5 --scale 1.0 --runs 2 --flags 16
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench4.json 2> gpurun_out/bench4.log; echo "bench rc=$?"
cat gpurun_out/bench4.json

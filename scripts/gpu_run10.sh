mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -4
for c in 1 2 3 4 5; do python scripts/prof_run.py --config $c --scale 1.0 --runs 2; done
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench5.json 2> gpurun_out/bench5.log; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench5.json')); print(d['value'], d['e2e'], d['roofline']['frac'], d['tiers']['ms'])"

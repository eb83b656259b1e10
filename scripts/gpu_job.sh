mkdir -p gpurun_out
for c in 1 2 3; do timeout 300 python scripts/prof_run.py --config $c --scale 1.0 --runs 3 | grep -o "start tier [0-9]*\|tiers ms \[[^]]*\]\|GCUPS [0-9.]*" | tr '\n' ' '; echo; done
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -2

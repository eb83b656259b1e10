mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "wide or vectors_all_tiers" 2>&1 | tail -2
timeout 600 python scripts/prof_run.py --config 4 --scale 1.0 --x 100 --runs 2
timeout 600 python scripts/prof_run.py --config 4 --scale 0.1 --x 100 --runs 2

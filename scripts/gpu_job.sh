mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "wide or vectors_all_tiers or band_failures or route_guard or edge or config5 or sample_vs_oracle" 2>&1 | tail -4
timeout 600 python scripts/prof_run.py --config 4 --scale 1.0 --x 100 --runs 2
timeout 600 python scripts/prof_run.py --config 4 --scale 0.1 --x 100 --runs 2
timeout 600 python scripts/prof_run.py --config 2 --scale 1.0 --x 40 --band 1024 --runs 2
timeout 600 python scripts/prof_run.py --config 4 --scale 1.0 --runs 2
timeout 600 python scripts/prof_run.py --config 5 --scale 1.0 --runs 2

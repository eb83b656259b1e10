for c in 5; do XB_LIB_PATH=build_dbg/libxdrop_b200_dbg.so python scripts/prof_run.py --config $c --scale 0.2 --runs 1; done
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
for c in 1 2 3 4 5; do python scripts/prof_run.py --config $c --scale 1.0 --runs 2; done

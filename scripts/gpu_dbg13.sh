for c in 2 4 5; do XB_LIB_PATH=build_dbg/libxdrop_b200_dbg.so python scripts/prof_run.py --config $c --scale 0.2 --runs 1; done

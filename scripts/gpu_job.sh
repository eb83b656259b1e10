mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "configs_vs_reference_golden or vectors_all_tiers" 2>&1 | tail -2
for c in 2 3 1; do for e in "XB_NO_PRIO=1" "XB_PRIO=1"; do echo "C$c [$e]"; env $e timeout 300 python scripts/prof_run.py --config $c --scale 1.0 --runs 3 | grep -o "tiers ms \[[^,]*, [^,]*, [^,]*\|GCUPS [0-9.]*"; done; done

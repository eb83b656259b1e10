# A/B: device GCUPS of configs under two library builds, alternating (A = XB_LIB_PATH=$A_LIB).
# usage: A_LIB=paper_2304_08662_b200/_lib/libxdrop_b200_A.so bash scripts/ab_run.sh "--config 5 --scale 1.0" ...
mkdir -p gpurun_out
for args in "$@"; do
  for rep in 1 2; do
    for lib in A B; do
      if [ $lib = A ]; then L=$A_LIB; else L=""; fi
      echo -n "$lib [$args] "; XB_LIB_PATH=$L timeout 300 python scripts/prof_run.py --runs 3 $args | grep -o "tiers ms \[[^,]*, [^,]*, [^,]*, [^,]*, [^,]*\|GCUPS [0-9.]*" | tr '\n' ' '; echo
    done
  done
done

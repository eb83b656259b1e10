#!/bin/bash
# Table modes (protein, BLOSUM62): device ms per step for library builds (LIBS) on C3 and C3 x10.
for L in ${LIBS:-paper_2304_08662_b200/_lib/libxdrop_b200.so}; do
  for spec in "3 1.0" "3 10"; do set -- $spec
    echo "$L cfg$1 x$2: $(XB_LIB_PATH=$L timeout 300 python bench.py --config $1 --scale $2 --steps 4 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); t=d["tiers"]; print(round(d["value"],1), round(d["ms_per_step"],3), [round(x,2) for x in t["ms"]])')"
  done
done

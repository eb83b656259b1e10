"""§8(f) band survey: GPU sweep_band vs the reference's sweep_band
(oracle/_ref, single-threaded as the reference runs it) on paper-scale grids;
checks the TSVs are identical and writes profiles/r1_sweep_band.json."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import paper_2304_08662_b200 as xb  # noqa: E402
from oracle_py import Ref  # noqa: E402

GRIDS = {
    "paper_L20000_6x7": (20000, [5, 10, 15, 20, 30, 50], [0.70, 0.75, 0.80, 0.85, 0.90, 0.95, 1.0]),
    "dense_L20000_10x30": (20000, list(range(5, 55, 5)), [round(0.70 + 0.01 * i, 2) for i in range(30)]),
}
R = Ref()
out = {}
for name, (L, xs, ps) in GRIDS.items():
    xb.sweep_band(L, xs, ps)  # warm-up: context, one cached workspace per concurrent X
    t0 = time.perf_counter()
    g = xb.sweep_band(L, xs, ps)
    tg = time.perf_counter() - t0
    t0 = time.perf_counter()
    r = R.sweep_band(L, xs, ps)
    tr = time.perf_counter() - t0
    out[name] = {"length": L, "n_x": len(xs), "n_p": len(ps), "cells_grid": len(xs) * len(ps),
                 "gpu_s": tg, "reference_cpu_s": tr, "speedup": tr / tg, "identical_tsv": g == r}
    print(name, json.dumps(out[name]), flush=True)
dst = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "r1_sweep_band.json")
json.dump(out, open(dst, "w"), indent=1)

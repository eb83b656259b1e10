"""One device-resident batch of a config (for ncu): python scripts/prof_run.py --config 5 --scale 0.05"""
import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2304_08662_b200 as xb  # noqa: E402
from paper_2304_08662_b200 import capi, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--scale", type=float, default=0.05)
ap.add_argument("--runs", type=int, default=2)
ap.add_argument("--flags", type=int, default=0)
ap.add_argument("--shard", default=None, help="i/N: only shard i of N (xb_shard_tasks, locality)")
ap.add_argument("--x", type=int, default=None)
ap.add_argument("--band", type=int, default=None)
a = ap.parse_args()
ds = synth.make(a.config, a.scale)
if a.x is not None:
    ds.x = a.x
if a.band is not None:
    ds.band = a.band
if ds.cfg == 3:
    s = xb.ScoringScheme.from_matrix(xb.parse_submatrix(synth.blosum62_text()), -1, ds.x)
else:
    s = xb.ScoringScheme.match_mismatch(1, -1, -1, ds.x)
pool = xb.DevicePool(s, ds.symbols, ds.offsets)
L = capi.lib()
tk = ds.tasks
if a.shard:
    i, n = (int(v) for v in a.shard.split("/"))
    tk = tk[xb.xband.shard_tasks(pool, tk, ds.k, n, locality=True) == i]
t = xb.xband.tasks_array(tk)
ex = capi.make_exec(1, [0], None, a.flags)
err, bad = C.c_int(0), C.c_int64(-1)
b = L.xb_batch_create(pool._h, t.ctypes.data, len(t), ds.k, ds.band, C.byref(ex), C.byref(bad), C.byref(err))
capi.check(err.value, "create")
for _ in range(a.runs):
    capi.check(L.xb_batch_run(b), "run")
    capi.check(L.xb_batch_sync(b), "sync")
st = capi.XbStats()
L.xb_batch_stats(b, C.byref(st))
d = st.as_dict()
cells = sum(d["cells_tier"])
print(f"config {a.config} x{a.scale}: {len(t)} tasks, {cells} cells, start tier {d['start_tier']}, "
      f"tiers ms {[round(x, 3) for x in d['ms_tier']]}, units {d['units_tier']}, escalated {d['escalated']}, "
      f"prep {d['ms_prep']:.2f} ms, pilot {d['ms_pilot']:.2f} ms, "
      f"GCUPS {cells / (d['ms_total'] / 1e3) / 1e9:.1f}" + (f" dbg {d['dbg']}" if any(d['dbg']) else ""))
L.xb_batch_free(b)

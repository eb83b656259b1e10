"""Per-shard device time of config 5 split N ways (xb_shard_tasks, LPT and
locality), each shard run alone on this GPU: the max/mean ratio is the strong-
scaling efficiency loss from imbalance; uploaded bytes show the locality gain.
python scripts/shard_balance.py --n 8"""
import argparse
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2304_08662_b200 as xb  # noqa: E402
from paper_2304_08662_b200 import capi, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--scale", type=float, default=1.0)
ap.add_argument("--n", type=int, default=8)
ap.add_argument("--runs", type=int, default=2)
a = ap.parse_args()
ds = synth.make(a.config, a.scale)
s = xb.ScoringScheme.match_mismatch(1, -1, -1, ds.x)
L = capi.lib()
out = {}
for mode in ("lpt", "locality"):
    pool = xb.DevicePool(s, ds.symbols, ds.offsets)
    sh = xb.xband.shard_tasks(pool, ds.tasks, ds.k, a.n, locality=mode == "locality")
    rows = []
    for g in range(a.n):
        p = xb.DevicePool(s, ds.symbols, ds.offsets)  # a fresh device copy per shard: what one rank uploads
        t = xb.xband.tasks_array(ds.tasks[sh == g])
        ex = capi.make_exec(1, [0], None, 0)
        err, bad = C.c_int(0), C.c_int64(-1)
        b = L.xb_batch_create(p._h, t.ctypes.data, len(t), ds.k, ds.band, C.byref(ex), C.byref(bad), C.byref(err))
        capi.check(err.value, "create")
        st = capi.XbStats()
        L.xb_batch_stats(b, C.byref(st))
        h2d = st.h2d_bytes
        for _ in range(a.runs):
            capi.check(L.xb_batch_run(b), "run")
            capi.check(L.xb_batch_sync(b), "sync")
        L.xb_batch_stats(b, C.byref(st))
        d = st.as_dict()
        rows.append({"shard": g, "tasks": len(t), "cells": int(sum(d["cells_tier"])), "ms": d["ms_total"],
                     "h2d_bytes": int(h2d)})
        L.xb_batch_free(b)
    ms = np.array([r["ms"] for r in rows])
    out[mode] = {"shards": rows, "max_ms": float(ms.max()), "mean_ms": float(ms.mean()),
                 "balance": float(ms.mean() / ms.max()),
                 "h2d_mean_bytes": float(np.mean([r["h2d_bytes"] for r in rows]))}
    print(f"{mode}: max {ms.max():.2f} ms mean {ms.mean():.2f} ms balance {ms.mean() / ms.max():.4f} "
          f"h2d/shard {out[mode]['h2d_mean_bytes'] / 1e6:.1f} MB", flush=True)
json.dump(out, open(os.path.join("gpurun_out", f"shard_balance_n{a.n}.json"), "w"), indent=1)

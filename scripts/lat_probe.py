"""Latency probe: device ms of a latency-bound config's whole batch and of
the task holding its longest unit alone, under several start-tier settings
(lane groups vs one thread per unit, forced tiers).  Prints one JSON line per
(config, setting).

    python scripts/lat_probe.py --configs 1,2,3
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2304_08662_b200 as xb  # noqa: E402
from paper_2304_08662_b200 import capi, synth  # noqa: E402

NO_GROUP, FORCE, GROUP = 64, 8, 32


def run(L, pool, t, k, band, flags, reps=4):
    ex = capi.make_exec(1, [0], None, flags)
    err, bad = capi.C.c_int(0), capi.C.c_int64(-1)
    b = L.xb_batch_create(pool._h, t.ctypes.data, len(t), k, band, capi.C.byref(ex),
                          capi.C.byref(bad), capi.C.byref(err))
    capi.check(err.value, "create")
    best, st = 1e30, None
    for rep in range(reps):
        capi.check(L.xb_batch_run(b), "run")
        capi.check(L.xb_batch_sync(b), "sync")
        x = capi.XbStats()
        L.xb_batch_stats(b, capi.C.byref(x))
        if (rep or reps == 1) and x.ms_total < best:
            best, st = x.ms_total, x.as_dict()
    out = np.zeros(2 * len(t), dtype=capi.RESULT_DTYPE)
    ss = np.zeros(len(t), dtype=np.int32)
    capi.check(L.xb_batch_fetch(b, out.ctypes.data, ss.ctypes.data), "fetch")
    L.xb_batch_free(b)
    return best, st, out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3")
    ap.add_argument("--settings", default="default,nogroup,t1,t2,t3,g2,g3")
    ap.add_argument("--task", type=int, default=-1,
                    help="with --alone-only: this task index, no full-batch run")
    ap.add_argument("--alone-only", action="store_true",
                    help="run only the longest task alone, once per setting (for ncu)")
    a = ap.parse_args()
    L = capi.lib()
    settings = {"default": 0, "nogroup": NO_GROUP,
                "t0": FORCE | NO_GROUP | (0 << 8), "t1": FORCE | NO_GROUP | (1 << 8),
                "t2": FORCE | NO_GROUP | (2 << 8), "t3": FORCE | NO_GROUP | (3 << 8),
                "t4": FORCE | NO_GROUP | (4 << 8),
                "g0": FORCE | GROUP | (0 << 8), "g1": FORCE | GROUP | (1 << 8), "g2": FORCE | GROUP | (2 << 8), "g3": FORCE | GROUP | (3 << 8)}
    for cfg in [int(c) for c in a.configs.split(",")]:
        ds = synth.make(cfg, 1.0)
        if cfg == 3:
            s = xb.ScoringScheme.from_matrix(xb.parse_submatrix(synth.blosum62_text()), -1, ds.x)
        else:
            s = xb.ScoringScheme.match_mismatch(1, -1, -1, ds.x)
        pool = xb.DevicePool(s, ds.symbols, ds.offsets)
        t = xb.xband.tasks_array(ds.tasks)
        ref = None
        if a.alone_only:
            if a.task >= 0:
                lt = a.task
            else:
                ms, st, out = run(L, pool, t, ds.k, ds.band, 0, reps=1)
                ext = (out["h_ext"] + out["v_ext"]).reshape(-1, 2).max(axis=1)
                lt = int(np.argmax(ext))
            print(json.dumps({"cfg": cfg, "longest_task": lt}), flush=True)
            one = t[lt:lt + 1].copy()
            for name in a.settings.split(","):
                ms1, _, _ = run(L, pool, one, ds.k, ds.band, settings[name], reps=1)
                print(json.dumps({"cfg": cfg, "setting": name, "alone_ms": round(ms1, 3)}), flush=True)
            continue
        for name in a.settings.split(","):
            fl = settings[name]
            ms, st, out = run(L, pool, t, ds.k, ds.band, fl)
            if ref is None:
                ref = out
                ext = (out["h_ext"] + out["v_ext"]).reshape(-1, 2).max(axis=1)
                lt = int(np.argmax(ext))
                longest = int(ext[lt])
            same = bool(np.array_equal(out, ref))
            one = t[lt:lt + 1].copy()
            ms1, st1, _ = run(L, pool, one, ds.k, ds.band, fl)
            print(json.dumps({"cfg": cfg, "setting": name, "ms": round(ms, 3), "alone_ms": round(ms1, 3),
                              "cyc_per_antidiag_alone": round(ms1 * 1.965e6 / longest, 1),
                              "start_tier": st["start_tier"], "groups": st["start_lane_groups"],
                              "tier_ms": [round(v, 3) for v in st["ms_tier"]], "identical": same}),
                  flush=True)


if __name__ == "__main__":
    main()

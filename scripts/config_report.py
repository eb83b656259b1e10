"""Per-config report: for each of the five configs at BASELINE
size, on one GPU:

  * GCUPS_computed = sum(cells) / device time (best of 3 resident runs),
    the INT32 roofline fraction, and GCUPS_paper = sum(|H|.|V|) / time;
  * e2e GCUPS through xb_extend_batch from host buffers (pool re-uploaded);
  * the reference CPU kernel (oracle/_ref, the reference's own sources) on
    all host cores and on one thread, same tasks (all of C1-C3, a seeded
    sample of C4/C5), with the CPU model and core count;
  * bit-exact parity of every compared row against that reference run;
  * the per-unit critical path: the longest unit's antidiagonals (to its
    best cell, a lower bound) and the device time of the task holding it,
    run alone -- the wall time no schedule of the batch can beat.

    python scripts/config_report.py --out profiles/r1_configs
"""
import argparse
import json
import os
import platform
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np  # noqa: E402

import paper_2304_08662_b200 as xb  # noqa: E402
from paper_2304_08662_b200 import capi, synth  # noqa: E402

OPS_PER_CELL = 8
GROUP_STEP_CYCLES = 490  # lone K32 DNA lane group, measured


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def rows_equal(a, b):
    f = ["score", "h_ext", "v_ext", "cells", "delta_w", "status", "spread"]
    return np.all(np.stack([a[x] == b[x] for x in f]), axis=0)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="profiles/r1_configs")
    ap.add_argument("--configs", default="1,2,3,4,5")
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    a = ap.parse_args()
    from oracle_py import Ref
    R = Ref()
    L = capi.lib()
    alu, mixed, clk, sms = (capi.C.c_double(), capi.C.c_double(), capi.C.c_double(), capi.C.c_int())
    capi.check(L.xb_measure_int32_peak(0, capi.C.byref(alu), capi.C.byref(mixed), capi.C.byref(clk),
                                       capi.C.byref(sms)), "peak")
    peak_clk = 1965.0
    try:
        peak_clk = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["sm_max_mhz"]
    except (OSError, KeyError, ValueError):
        pass
    peak_ops = alu.value * sms.value * peak_clk * 1e6
    peak_all = mixed.value * sms.value * peak_clk * 1e6  # ALU + FMA pipes: the roofline
    cores = host_cores()
    report = {"gpu": "B200", "sm_count": sms.value, "peak_alu_lane_ops_per_clk_sm": alu.value,
              "cpu_model": cpu_model(), "cpu_cores": cores, "configs": []}
    for cfg in [int(c) for c in a.configs.split(",")]:
        ds = synth.make(cfg, 1.0)
        if cfg == 3:
            s = xb.ScoringScheme.from_matrix(xb.parse_submatrix(synth.blosum62_text()), -1, ds.x)
            rs = R.scheme_matrix(synth.blosum62_text(), -1, ds.x)
        else:
            s = xb.ScoringScheme.match_mismatch(1, -1, -1, ds.x)
            rs = R.scheme_mm(1, -1, -1, ds.x)
        pool = xb.DevicePool(s, ds.symbols, ds.offsets)
        # device time, resident inputs, best of 3 (after a warm-up)
        t = xb.xband.tasks_array(ds.tasks)
        ex = capi.make_exec(1, [0], None, 0)
        err, bad = capi.C.c_int(0), capi.C.c_int64(-1)
        b = L.xb_batch_create(pool._h, t.ctypes.data, len(t), ds.k, ds.band, capi.C.byref(ex),
                              capi.C.byref(bad), capi.C.byref(err))
        capi.check(err.value, "create")
        best, st = 1e30, None
        for rep in range(4):
            capi.check(L.xb_batch_run(b), "run")
            capi.check(L.xb_batch_sync(b), "sync")
            x = capi.XbStats()
            L.xb_batch_stats(b, capi.C.byref(x))
            if rep and x.ms_total < best:
                best, st = x.ms_total, x.as_dict()
        out = np.zeros(2 * len(t), dtype=capi.RESULT_DTYPE)
        ss = np.zeros(len(t), dtype=np.int32)
        capi.check(L.xb_batch_fetch(b, out.ctypes.data, ss.ctypes.data), "fetch")
        L.xb_batch_free(b)
        cells = int(out["cells"].sum())
        lens = np.diff(ds.offsets)
        paper_products = float(np.sum(lens[ds.tasks[:, 0]].astype(np.float64) *
                                      lens[ds.tasks[:, 1]].astype(np.float64)))
        # end to end: pool and tasks from host buffers, results back, every call
        e2e = []
        for rep in range(3):
            pool.evict()
            t0 = time.perf_counter()
            xb.extend_tasks(pool, t, ds.k, ds.band)  # tasks already in the ABI layout
            if rep:
                e2e.append(time.perf_counter() - t0)
        # reference CPU: same tasks (all, or a seeded sample of ~cpu_seconds)
        rp = R.pool(ds.symbols, ds.offsets)
        est_rate = 1.8e9
        n_cmp = ds.n_tasks if cells / est_rate < a.cpu_seconds else \
            int(ds.n_tasks * a.cpu_seconds * est_rate / cells)
        sel = np.sort(np.random.default_rng(cfg).permutation(ds.n_tasks)[:n_cmp])
        t0 = time.perf_counter()
        ref, ref_ss = R.extend_batch(rp, rs, ds.tasks[sel], ds.k, ds.band, threads=cores)
        t_all = time.perf_counter() - t0
        sel1 = sel[: max(1, len(sel) // (4 * cores))]
        t0 = time.perf_counter()
        ref1, _ = R.extend_batch(rp, rs, ds.tasks[sel1], ds.k, ds.band, threads=1)
        t_one = time.perf_counter() - t0
        ours = out.reshape(-1, 2)[sel].reshape(-1)
        eq = rows_equal(ours, ref)
        cells_ref = int(ref["cells"].sum())
        cells_one = int(ref1["cells"].sum())
        longest = int((out["h_ext"] + out["v_ext"]).max())
        # the critical path measured: the task holding the longest unit, alone
        lt = int(np.argmax((out["h_ext"] + out["v_ext"]).reshape(-1, 2).max(axis=1)))
        one = t[lt:lt + 1].copy()
        b1 = L.xb_batch_create(pool._h, one.ctypes.data, 1, ds.k, ds.band, capi.C.byref(ex),
                               capi.C.byref(bad), capi.C.byref(err))
        capi.check(err.value, "create")
        alone = 1e30
        for rep in range(4):
            capi.check(L.xb_batch_run(b1), "run")
            capi.check(L.xb_batch_sync(b1), "sync")
            x = capi.XbStats()
            L.xb_batch_stats(b1, capi.C.byref(x))
            if rep:
                alone = min(alone, x.ms_total)
        L.xb_batch_free(b1)
        row = {
            "config": cfg, "tasks": ds.n_tasks, "units": 2 * ds.n_tasks, "cells": cells,
            "device_ms": best, "gcups_computed": cells / (best / 1e3) / 1e9,
            "roofline_frac_alu": cells * OPS_PER_CELL / (best / 1e3) / peak_ops,
            "roofline_frac": cells * OPS_PER_CELL / (best / 1e3) / peak_all,
            "gcups_paper": paper_products / (best / 1e3) / 1e9,
            "e2e_ms": 1e3 * min(e2e), "e2e_gcups": cells / min(e2e) / 1e9,
            "start_tier": (f"k{[16, 24, 32, 48, 64][st['start_tier']]} "
                           + ("lane tiers (8 lanes)" if st["start_lane_groups"] == 2 else "lane groups" if st["start_lane_groups"] else "thread/unit"))
            if 0 <= st["start_tier"] < 5 else None,
            "tier_ms": [round(v, 3) for v in st["ms_tier"]], "escalated": st["escalated"],
            "ref_tasks_compared": int(len(sel)), "ref_rows_equal": int(eq.sum()),
            "ref_rows": int(len(eq)), "seed_scores_equal": bool((ss[sel] == ref_ss).all()),
            "cpu_gcups_all_cores": cells_ref / t_all / 1e9, "cpu_gcups_1_thread": cells_one / t_one / 1e9,
            "speedup_vs_cpu_all_cores_e2e": (cells / min(e2e)) / (cells_ref / t_all),
            "longest_unit_antidiagonals_lb": longest,
            "critical_path_ms_at_group_latency": longest * GROUP_STEP_CYCLES / (peak_clk * 1e3),
            "longest_task_alone_ms": alone,
            "group_step_cycles_measured": alone * 1e3 * peak_clk / max(longest, 1),
        }
        report["configs"].append(row)
        print(json.dumps(row), flush=True)
    os.makedirs(os.path.dirname(os.path.join(ROOT, a.out)) or ".", exist_ok=True)
    json.dump(report, open(os.path.join(ROOT, a.out + ".json"), "w"), indent=1)
    lines = [f"# Per-config report (1 B200; CPU reference: {report['cpu_model']}, {cores} threads)", "",
             "| cfg | cells | start | device ms | GCUPS | roofline (all INT32 pipes / ALU only) | GCUPS paper | e2e GCUPS | "
             "CPU GCUPS (all / 1 thr) | e2e speed-up | parity rows | critical path: longest unit, its task alone |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|"]
    for r in report["configs"]:
        lines.append(
            f"| C{r['config']} | {r['cells']:.3g} | {r['start_tier']} | {r['device_ms']:.2f} | "
            f"{r['gcups_computed']:.1f} | {r['roofline_frac']:.3f} / {r['roofline_frac_alu']:.3f} | {r['gcups_paper']:.0f} | "
            f"{r['e2e_gcups']:.1f} | {r['cpu_gcups_all_cores']:.2f} / {r['cpu_gcups_1_thread']:.3f} | "
            f"{r['speedup_vs_cpu_all_cores_e2e']:.0f}x | {r['ref_rows_equal']}/{r['ref_rows']} "
            f"({r['ref_tasks_compared']} tasks) | {r['longest_unit_antidiagonals_lb']} antidiag; "
            f"alone {r['longest_task_alone_ms']:.2f} ms |")
    open(os.path.join(ROOT, a.out + ".md"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()

"""Runs the kernel vectors one scheme group per process (a fault kills only
that process): python scripts/debug_vectors.py [flags]"""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
flags = int(sys.argv[1]) if len(sys.argv) > 1 else 0
if len(sys.argv) > 2:
    import test_gpu_parity as T
    import paper_2304_08662_b200 as xb
    entries = T.VEC["kats"] + T.VEC["random"]
    key = json.loads(sys.argv[2])
    for (spec, band), idx in T._by_scheme(entries).items():
        if [list(spec), band] != key:
            continue
        sel = [entries[i] for i in idx]
        sym, off, units = T._units_for(xb, sel)
        pool = xb.DevicePool(T._scheme(xb, list(spec)), sym, off)
        out = xb.extend_units(pool, units, band, exec_flags=flags)
        bad = sum(T.rec_tuple(r) != T.expect_tuple(entries[i]["kernel"]) for i, r in zip(idx, out))
        print("group", key, len(idx), "units, mismatches", bad, "stats", xb.xband.last_stats()["units_tier"])
    sys.exit(0)
import test_gpu_parity as T
entries = T.VEC["kats"] + T.VEC["random"]
for (spec, band), idx in T._by_scheme(entries).items():
    r = subprocess.run([sys.executable, __file__, str(flags), json.dumps([list(spec), band])],
                       capture_output=True, text=True, timeout=120)
    print(r.returncode, r.stdout.strip()[-300:], r.stderr.strip()[-300:])

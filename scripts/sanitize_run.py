"""One batch of a config under compute-sanitizer, checked against the C oracle
(every row of a seeded sample): python scripts/sanitize_run.py --config 5 --scale 0.01 --flags 8

flags 8 (XB_FLAG_FORCE_TIER, tier 0): start at K16 so most units escalate and
the concurrent escalation consumer (and the serial tail) carry the batch;
flags 32: lane groups throughout (the latency-mode kernels)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import paper_2304_08662_b200 as xb  # noqa: E402
from helpers import oracle_scheme, result_rows_equal  # noqa: E402
from oracle_py import Oracle  # noqa: E402  (the checker only)
from paper_2304_08662_b200 import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--scale", type=float, default=0.01)
ap.add_argument("--flags", type=int, default=0)
ap.add_argument("--sample", type=int, default=2000)
a = ap.parse_args()
ds = synth.make(a.config, a.scale)
if ds.cfg == 3:
    s = xb.ScoringScheme.from_matrix(xb.parse_submatrix(synth.blosum62_text()), -1, ds.x)
else:
    s = xb.ScoringScheme.match_mismatch(1, -1, -1, ds.x)
pool = xb.DevicePool(s, ds.symbols, ds.offsets)
out, ss = xb.extend_tasks(pool, ds.tasks, ds.k, ds.band, exec_flags=a.flags)
st = xb.xband.last_stats()
O = Oracle()
rng = np.random.default_rng(a.config)
pick = np.sort(rng.choice(ds.n_tasks, size=min(ds.n_tasks, a.sample), replace=False))
exp, ess = O.extend_batch(ds.symbols, ds.offsets, ds.tasks[pick], ds.k,
                          oracle_scheme(O, ["BLOSUM62", -1, ds.x] if ds.cfg == 3 else [1, -1, -1, ds.x]),
                          ds.band, threads=os.cpu_count() or 1)
ok = result_rows_equal(out.reshape(-1, 2)[pick].reshape(-1), exp).all() and (ss[pick] == ess).all()
print(f"config {a.config} x{a.scale} flags {a.flags}: {ds.n_tasks} tasks, units per tier {st['units_tier']}, "
      f"escalated {st['escalated']}, {len(pick)} sampled tasks vs oracle: {'identical' if ok else 'MISMATCH'}")
sys.exit(0 if ok else 1)

"""§8(f) item 2: ingest throughput.  Config 5's pool as FASTA text (200,000
reads, 2.2 GB) and its 2,000,000 seeds as a seed list: native parsers (all
host threads) vs the reference's parse_fasta / parse_seeds (oracle/_ref),
identical output checked; then text -> packed pool -> GPU results."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np  # noqa: E402

import paper_2304_08662_b200 as xb  # noqa: E402
from paper_2304_08662_b200 import synth  # noqa: E402
from oracle_py import Ref  # noqa: E402

scale = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
dst = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "profiles", "r1_ingest.json")
ds = synth.make(5, scale)
sym = ds.symbols.tobytes()
off = ds.offsets.tolist()
# one header + one sequence line per read (valid FASTA; fast to build)
fasta = b"".join(b">read%d\n%s\n" % (i, sym[off[i]:off[i + 1]]) for i in range(len(off) - 1))
seeds = "\n".join(" ".join(map(str, r)) for r in ds.tasks.tolist()).encode() + b"\n"
R = Ref()
out = {"fasta_bytes": len(fasta), "records": len(ds.offsets) - 1, "seed_bytes": len(seeds),
       "seeds": int(ds.n_tasks)}
t0 = time.perf_counter()
rec = xb.FastaRecords(fasta, "ACGTN")
out["ours_fasta_s"] = time.perf_counter() - t0
t0 = time.perf_counter()
tasks = xb.parse_seeds(seeds)
out["ours_seeds_s"] = time.perf_counter() - t0
t0 = time.perf_counter()
ref = R.parse_fasta(fasta, "ACGTN")
out["ref_fasta_s"] = time.perf_counter() - t0
t0 = time.perf_counter()
rt = R.parse_tasks(seeds, False)
out["ref_seeds_s"] = time.perf_counter() - t0
out["identical_fasta"] = ref[0] == rec.symbols.tobytes() and list(ref[1]) == rec.offsets.tolist()
out["identical_seeds"] = bool(np.array_equal(rt[:, 1:], np.stack([tasks[f] for f in
                                                                  ("h_id", "v_id", "h_seed", "v_seed")], 1)))
out["ours_fasta_GBps"] = len(fasta) / out["ours_fasta_s"] / 1e9
out["ref_fasta_GBps"] = len(fasta) / out["ref_fasta_s"] / 1e9
# text to results: parse, pack + upload, extend on the GPU
try:
    s = xb.ScoringScheme.match_mismatch(1, -1, -1, ds.x)
    t0 = time.perf_counter()
    rec2 = xb.FastaRecords(fasta, "ACGTN")
    pool = xb.DevicePool.from_fasta(rec2, s)
    t2 = xb.parse_seeds(seeds)
    res, _ = xb.extend_tasks(pool, t2, ds.k, ds.band)
    out["text_to_results_s"] = time.perf_counter() - t0
    out["text_to_results_cells"] = int(res["cells"].sum())
except Exception as e:  # no GPU
    out["text_to_results_s"] = None
    out["note"] = str(e)
print(json.dumps(out, indent=1))
json.dump(out, open(dst, "w"), indent=1)

"""Regenerates the golden fixtures in tests/golden/ from the UNMODIFIED reference.

Runs only in the dev container (needs /root/reference and oracle/_ref, built
by `make -C oracle ref`).  Every expected value here is produced by the
reference library itself (proj/src/align.cpp, scoring.cpp, pipeline.cpp via
oracle/ref_harness.cpp); nothing is hand-written except the inputs, which
restate the reference tests' inputs (proj/tests/test_align.cpp:41-331,
proj/tests/acceptance.cpp:171-276) and SURVEY.md Appendix B.

    python tests/golden/make_golden.py
"""
from __future__ import annotations

import hashlib
import json
import os
import random
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, ROOT)

from oracle_py import RESULT_DTYPE, Ref  # noqa: E402

REF_MATRIX = "/root/reference/proj/data/BLOSUM62"


def res_tuple(r):
    if r.status:
        return {"status": 1, "spread": r.spread, "cells": r.cells}
    return {"status": 0, "score": r.score, "h_ext": r.h_ext, "v_ext": r.v_ext, "cells": r.cells,
            "delta_w": r.delta_w}


def mutate(rng: random.Random, s: bytes, p: float, alphabet=b"ACGT") -> bytes:
    out = bytearray()
    for c in s:
        u = rng.random()
        if u < p / 3:
            out.append(rng.choice([a for a in alphabet if a != c] or [c]))
        elif u < 2 * p / 3:
            out += bytes([rng.choice(alphabet), c])
        elif u < p:
            pass
        else:
            out.append(c)
    return bytes(out)


def main():
    R = Ref()
    # ---- BLOSUM62 as the reference parses it ----
    text = open(REF_MATRIX).read()
    alpha, cells = R.parse_matrix(text)
    json.dump({"alphabet": alpha, "cells": cells.ravel().tolist(),
               "source": "proj/data/BLOSUM62 via xband::parse_submatrix"},
              open(os.path.join(HERE, "blosum62.json"), "w"))

    # ---- known-answer tests (test_align.cpp:41-123, Appendix B) ----
    kats = []

    def kat(h, v, x, band, **kw):
        s = R.scheme_mm(1, -1, -1, x)
        r = R.extend(h, v, s, band, **kw)
        entry = {"h": h.decode(), "v": v.decode(), "x": x, "band": band, "kw": kw,
                 "kernel": res_tuple(r)}
        if not kw:
            entry["oracle"] = res_tuple(R.full(h, v, s))
        kats.append(entry)

    kat(b"ACGT", b"ACGT", 3, 16)
    kat(b"", b"ACGT", 3, 8)
    kat(b"", b"", 3, 4)
    kat(b"AAAA", b"AATA", 10, 16)
    kat(b"AAAAAA", b"AATAAA", 10, 16)
    kat(b"ACGT", b"TTTT", 1, 16)
    kat(b"AC", b"GT", 0, 16)
    kat(b"ACGTACGTAC", b"ACGTACGTAC", 4, 12)
    kat(b"ACGTACGTACGT", b"ACGTACGTACGT", 4, 16)
    kat(b"AAAAAA", b"AATAAA", 10, 2)
    kat(b"NNNN", b"NNNN", 3, 8)
    kat(b"ACGTNACGT", b"ACGTNACGT", 5, 16)
    # seed stitching (test_align.cpp:243-302)
    seeds = []
    s5 = R.scheme_mm(1, -1, -1, 5)
    for (h, v, hs, vs, k, band, hid, vid) in [
        (b"AAAAAAAAAA", b"AAAAAAAAAA", 3, 3, 4, 16, 0, 1),
        (b"ACGTAC", b"ACGTAC", 0, 0, 6, 16, 0, 1),
        (b"ACGT", b"ACGT", 0, 0, 2, 8, 0, 7),
        (b"ACGT", b"ACGT", 3, 0, 2, 8, 0, 1),
        (b"ACGT", b"ACGT", 0, 4, 1, 8, 0, 1),
    ]:
        rc, L, Rr, ss, tot, side, sp = R.extend_seed(h, v, hs, vs, k, s5, band, hid, vid)
        seeds.append({"h": h.decode(), "v": v.decode(), "h_seed": hs, "v_seed": vs, "k": k,
                      "band": band, "h_id": hid, "v_id": vid, "x": 5, "rc": rc,
                      "left": res_tuple(L) if rc == 0 else None,
                      "right": res_tuple(Rr) if rc == 0 else None,
                      "seed_score": ss if rc == 0 else None, "total": tot if rc == 0 else None})
    # band failure names its side (test_align.cpp:284-302 shape)
    rng = random.Random(11)
    hs_ = bytes(rng.choice(b"ACGT") for _ in range(120))
    vs_ = mutate(rng, hs_, 0.5)
    h2, v2 = hs_[:17] + hs_, hs_[:17] + vs_
    s40 = R.scheme_mm(1, -1, -1, 40)
    rc, L, Rr, ss, tot, side, sp = R.extend_seed(h2, v2, 0, 0, 17, s40, 3)
    seeds.append({"h": h2.decode(), "v": v2.decode(), "h_seed": 0, "v_seed": 0, "k": 17,
                  "band": 3, "h_id": 0, "v_id": 1, "x": 40, "rc": rc, "side": side,
                  "spread": sp})

    # ---- random pairs incl. Left views, N, band failures ----
    rng = random.Random(20260822)
    rand = []
    for it in range(600):
        L_ = rng.randint(0, 160)
        alphabet = b"ACGTN" if it % 9 == 0 else b"ACGT"
        h = bytes(rng.choice(alphabet) for _ in range(L_))
        v = mutate(rng, h, rng.choice([0.0, 0.05, 0.15, 0.3, 0.7, 1.0]), alphabet)
        if it % 4 == 0:
            v = v[: rng.randint(0, len(v))]
        x = rng.choice([0, 1, 3, 5, 10, 15, 20, 50, 100])
        band = rng.choice([1, 3, 8, 16, 24, 32, 33, 64, 65, 100, 300])
        ho, vo = rng.randint(0, len(h)), rng.randint(0, len(v))
        hd, vd = rng.randint(0, 1), rng.randint(0, 1)
        kw = dict(h_origin=ho, v_origin=vo, h_dir=hd, v_dir=vd)
        s = R.scheme_mm(1, -1, -1, x)
        r = R.extend(h, v, s, band, **kw)
        rand.append({"h": h.decode(), "v": v.decode(), "x": x, "band": band, "kw": kw,
                     "scheme": [1, -1, -1, x], "kernel": res_tuple(r)})
    # other DNA schemes (table path) and BLOSUM62 proteins
    for it in range(200):
        L_ = rng.randint(0, 120)
        h = bytes(rng.choice(b"ACGT") for _ in range(L_))
        v = mutate(rng, h, rng.choice([0.05, 0.15, 0.3]))
        sc = rng.choice([[1, -2, -2], [2, -3, -5], [1, -1, -2], [5, -4, -3]])
        x = rng.choice([3, 10, 25])
        band = rng.choice([16, 32, 64, 128])
        s = R.scheme_mm(sc[0], sc[1], sc[2], x)
        r = R.extend(h, v, s, band)
        rand.append({"h": h.decode(), "v": v.decode(), "x": x, "band": band, "kw": {},
                     "scheme": sc + [x], "kernel": res_tuple(r)})
    aa = alpha.encode()
    for it in range(200):
        L_ = rng.randint(0, 200)
        h = bytes(rng.choice(aa[:20]) for _ in range(L_))
        v = mutate(rng, h, rng.choice([0.1, 0.3, 0.5]), aa[:20])
        x = rng.choice([5, 20, 49])
        gap = rng.choice([-1, -2, -4])
        band = rng.choice([16, 32, 64, 200])
        s = R.scheme_matrix(text, gap, x)
        r = R.extend(h, v, s, band, h_dir=it % 2, v_dir=it % 2,
                     h_origin=len(h) if it % 2 == 0 else 0, v_origin=len(v) if it % 2 == 0 else 0)
        rand.append({"h": h.decode(), "v": v.decode(), "x": x, "band": band,
                     "kw": {"h_dir": it % 2, "v_dir": it % 2,
                            "h_origin": len(h) if it % 2 == 0 else 0,
                            "v_origin": len(v) if it % 2 == 0 else 0},
                     "scheme": ["BLOSUM62", gap, x], "kernel": res_tuple(r)})
    json.dump({"kats": kats, "seeds": seeds, "random": rand}, open(os.path.join(HERE, "kernel_vectors.json"), "w"))

    # ---- the reference pipeline on its own synthetic data (Appendix B) ----
    ec, txt = R.pipeline_synth(8, 2000, 0.9, x=15)
    rows = [l for l in txt.splitlines() if not l.startswith("#") or l.startswith("# total\t")
            or l.startswith("# failed\t")]
    pipe = {"pairs": 8, "length": 2000, "p_match": 0.9, "x": 15, "band": 1024, "k": 17,
            "seed": 42, "exit_code": ec, "sha256_full": hashlib.sha256(txt.encode()).hexdigest(),
            "rows": rows}
    ec2, txt2 = R.pipeline_synth(40, 3000, 0.75, x=25, band=40, seed=7, uniform_seed=True)
    rows2 = [l for l in txt2.splitlines() if not l.startswith("#") or l.startswith("# total\t")
             or l.startswith("# failed\t")]
    pipe2 = {"pairs": 40, "length": 3000, "p_match": 0.75, "x": 25, "band": 40, "k": 17,
             "seed": 7, "uniform_seed": True, "exit_code": ec2, "rows": rows2}
    json.dump({"readme_smoke": pipe, "band_failures": pipe2},
              open(os.path.join(HERE, "pipeline_rows.json"), "w"))

    # ---- reference results on (small slices of) the five configs ----
    from paper_2304_08662_b200 import synth
    cfgs = {1: 1.0, 2: 0.01, 3: 0.02, 4: 0.004, 5: 0.0005}
    meta = {}
    for cfg, scale in cfgs.items():
        ds = synth.make(cfg, scale)
        pool = R.pool(ds.symbols, ds.offsets)
        if cfg == 3:
            s = R.scheme_matrix(text, -1, ds.x)
        else:
            s = R.scheme_mm(1, -1, -1, ds.x)
        out, ss = R.extend_batch(pool, s, ds.tasks, ds.k, ds.band, threads=8)
        np.savez_compressed(os.path.join(HERE, f"cfg{cfg}_ref.npz"), results=out, seed_score=ss)
        h = hashlib.sha256(ds.symbols.tobytes() + ds.offsets.tobytes() + ds.tasks.tobytes())
        meta[cfg] = {"scale": scale, "n_tasks": int(ds.n_tasks), "k": ds.k, "x": ds.x,
                     "band": ds.band, "input_sha256": h.hexdigest(),
                     "cells": int(out["cells"].sum()),
                     "band_failures": int((out["status"] != 0).sum())}
        print("cfg", cfg, meta[cfg])
    json.dump(meta, open(os.path.join(HERE, "configs_meta.json"), "w"), indent=1)


if __name__ == "__main__":
    main()

"""Randomised parity sweep: many small batches over random pools and random
parameters -- DNA with and without N, BLOSUM62 protein, other match /
mismatch / gap schemes, X from 0 to 200, bands from 1 to 1100 (band failures
included), every planning override (forced start tiers across the thread,
lane-group and wide tiers, lane groups everywhere, one thread per unit,
escalations straight to the warp tier, the serial tail, multi-device shards)
-- each batch checked row for row against the C oracle (itself pinned to the
reference, tests/test_oracle.py)."""
import os
import random

import numpy as np
import pytest

from helpers import blosum62, result_rows_equal

pytestmark = pytest.mark.gpu

# 16384 / 32768: the lane tiers (8 lanes per unit) / the 4-lane groups for every
# several-lanes-per-unit launch
FLAGS = [0, 1, 2, 128, 128 | 64, 32 | 16384, 32 | 32768, 64, 16, 4096, 8192] + [8 | (t << 8) for t in range(10)] + \
        [32 | 8 | (t << 8) | 32768 for t in range(5)] + [32 | 8 | (t << 8) | 16384 for t in range(5)] + \
        [64 | 8 | (t << 8) for t in range(5)]


def _mutate(rng, s, alpha, rate):
    out = []
    for ch in s:
        r = rng.random()
        if r < rate / 3:
            continue                       # deletion
        if r < 2 * rate / 3:
            out.append(rng.choice(alpha))  # insertion
            out.append(ch)
            continue
        if r < rate:
            out.append(rng.choice(alpha))  # substitution (maybe the same)
            continue
        out.append(ch)
    return "".join(out)


@pytest.mark.parametrize("round_", range(80))
def test_random_batches_vs_oracle(round_):
    import paper_2304_08662_b200 as xb
    from oracle_py import Oracle
    O = Oracle()
    rng = random.Random(9000 + round_)
    kind = rng.choice(["dna", "dna_n", "protein", "scheme"])
    if kind == "protein":
        alpha_s, cells = blosum62()
        alpha = alpha_s[:20]
        gap = rng.choice([-1, -2, -4])
        x = rng.choice([0, 3, 10, 25, 60, 120])
        scheme = xb.ScoringScheme.from_matrix(xb.SubMatrix(alpha_s, cells), gap, x)
        os_ = O.scheme_matrix(alpha_s, cells, gap, x)
    else:
        alpha = "ACGTN" if kind == "dna_n" else "ACGT"
        m, mm, gap = (1, -1, -1) if kind != "scheme" else (rng.choice([1, 2, 3]), rng.choice([-1, -2, -3]),
                                                          rng.choice([-1, -2, -5]))
        x = rng.choice([0, 1, 5, 15, 40, 100, 200])
        scheme = xb.ScoringScheme.match_mismatch(m, mm, gap, x)
        os_ = O.scheme_mm(m, mm, gap, x)
    n_seq = rng.randint(2, 60)
    seqs = []
    for _ in range(n_seq // 2 + 1):
        base = "".join(rng.choice(alpha[:4] if kind != "protein" else alpha) for _ in range(rng.randint(0, 3000)))
        seqs.append(base)
        seqs.append(_mutate(rng, base, alpha, rng.choice([0.0, 0.05, 0.15, 0.3])))
    k = rng.choice([0, 1, 6, 17])
    tasks = []
    for _ in range(rng.randint(1, 900)):
        h, v = rng.randrange(len(seqs)), rng.randrange(len(seqs))
        if len(seqs[h]) < k or len(seqs[v]) < k:
            continue
        tasks.append((h, v, rng.randint(0, len(seqs[h]) - k), rng.randint(0, len(seqs[v]) - k)))
    if not tasks:
        tasks = [(0, 0, 0, 0)]
        k = 0
    t = np.array(tasks, dtype=np.int64)
    sym = "".join(seqs).encode()
    off = np.zeros(len(seqs) + 1, dtype=np.int64)
    np.cumsum([len(s) for s in seqs], out=off[1:])
    band = rng.choice([1, 2, 8, 16, 33, 64, 100, 256, 700, 1100])
    pool = xb.DevicePool(scheme, sym, off)
    exp, ess = O.extend_batch(np.frombuffer(sym, np.uint8), off, t, k, os_, band, threads=os.cpu_count() or 1)
    for flags in rng.sample(FLAGS, 8):
        nd = 2 if flags & 8192 else 1
        out, ss = xb.extend_tasks(pool, t, k, band, exec_flags=flags, n_devices=nd,
                                  device_ids=[0] * nd)
        eq = result_rows_equal(out, exp)
        assert eq.all(), (kind, x, band, flags, int((~eq).sum()), np.nonzero(~eq)[0][:4])
        assert (ss == ess).all(), (kind, flags)

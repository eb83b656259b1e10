"""GPU parity: the sm_100a engine, called through the C-ABI, against the
reference's golden vectors and the C oracle.  Bar: bit-exact on every field
(score, h_ext, v_ext, cells, delta_w; spread + cells on band failures)."""
import hashlib
import os
import random

import numpy as np
import pytest

from helpers import blosum62, expect_tuple, load_json, oracle_scheme, rec_tuple, result_rows_equal

pytestmark = pytest.mark.gpu

VEC = load_json("kernel_vectors.json")


@pytest.fixture(scope="module")
def xb():
    import paper_2304_08662_b200 as xb
    assert xb.capi.lib().xb_device_count() > 0, "no CUDA device: the engine has no CPU fallback"
    return xb


def _scheme(xb, spec):
    if spec[0] == "BLOSUM62":
        a, c = blosum62()
        return xb.ScoringScheme.from_matrix(xb.SubMatrix(a, c), spec[1], spec[2])
    return xb.ScoringScheme.match_mismatch(*spec)


def _units_for(xb, entries):
    """All entries of one scheme as explicit units over one pool."""
    from paper_2304_08662_b200.capi import UNIT_DTYPE
    syms, off = [], [0]
    units = np.zeros(len(entries), dtype=UNIT_DTYPE)
    for q, e in enumerate(entries):
        h, v = e["h"].encode(), e["v"].encode()
        syms += [h, v]
        off += [off[-1] + len(h), off[-1] + len(h) + len(v)]
        kw = e["kw"]
        hd, vd = kw.get("h_dir", 1), kw.get("v_dir", 1)
        ho, vo = kw.get("h_origin", 0), kw.get("v_origin", 0)
        units[q] = (2 * q, 2 * q + 1, hd, vd, ho, vo,
                    (len(h) - ho) if hd else ho, (len(v) - vo) if vd else vo)
    return b"".join(syms), np.array(off, dtype=np.int64), units


def _by_scheme(entries):
    groups = {}
    for i, e in enumerate(entries):
        spec = tuple(e.get("scheme", [1, -1, -1, e["x"]]))
        groups.setdefault((spec, e["band"]), []).append(i)
    return groups


# 64 = NO_GROUP (one thread per unit), 32 = GROUP (lane groups throughout),
# 8 | t << 8 = start at tier t without the pilot
# 128 = THROUGHPUT (pilot + cost model even for a small batch)
# 8 | t << 8 with t = WIDE_FIRST..: start on the wide tiers (8-32 lanes per unit, K96..K1024)
from paper_2304_08662_b200.capi import NUM_TIERS, TIER_WIDTHS, WARP_TIER, WIDE_FIRST  # noqa: E402
# 16384 = LANES (lane tiers, 8 lanes per unit), 32768 = NO_LANES (4-lane groups): small
# batches pick the lane tiers by themselves, so both families are forced here
LANES, NO_LANES = 16384, 32768
TIER_FLAGS = ([0, 2, 128, 128 | 64] + [64 | 8 | (t << 8) for t in range(5)]
              + [32 | 8 | (t << 8) | NO_LANES for t in range(5)] + [32 | 8 | (t << 8) | LANES for t in range(5)]
              + [8 | (t << 8) for t in range(WIDE_FIRST, WARP_TIER)])
TIER_IDS = (["auto", "warp_tier_only", "pilot_cascade", "thread_pilot_cascade"]
            + [f"thread_k{w}" for w in (16, 24, 32, 48, 64)]
            + [f"group_k{w}" for w in (16, 24, 32, 48, 64)]
            + [f"lane_k{w}" for w in (16, 24, 32, 48, 64)]
            + [f"wide_k{w}" for w in TIER_WIDTHS[WIDE_FIRST:]])


@pytest.mark.parametrize("flags", TIER_FLAGS, ids=TIER_IDS)
def test_vectors_all_tiers(xb, flags):
    entries = VEC["kats"] + VEC["random"]
    bad = []
    for (spec, band), idx in _by_scheme(entries).items():
        sel = [entries[i] for i in idx]
        sym, off, units = _units_for(xb, sel)
        pool = xb.DevicePool(_scheme(xb, list(spec)), sym, off)
        out = xb.extend_units(pool, units, band, exec_flags=flags)
        for i, r in zip(idx, out):
            if rec_tuple(r) != expect_tuple(entries[i]["kernel"]):
                bad.append((i, rec_tuple(r), expect_tuple(entries[i]["kernel"])))
    assert not bad, f"{len(bad)} mismatches: {bad[:4]}"


def test_reference_api_kats(xb):
    # proj/tests/test_align.cpp:41-123 in the reference's own vocabulary
    S, full = xb.Sequence, xb.full
    s3 = xb.ScoringScheme.match_mismatch(1, -1, -1, 3)
    a = S(0, "s", "ACGT")
    r = xb.xdrop_extend(full(a), full(a), s3, 16)
    assert (r.score, r.h_ext, r.v_ext) == (4, 4, 4)
    r = xb.xdrop_extend(full(S(0, "h", "")), full(S(1, "v", "ACGT")), s3, 8)
    assert (r.score, r.h_ext, r.v_ext) == (0, 0, 0)
    e = S(0, "e", "")
    r = xb.xdrop_extend(full(e), full(e), s3, 4)
    assert r.cells == 1 and r.delta_w == 1
    s10 = xb.ScoringScheme.match_mismatch(1, -1, -1, 10)
    r = xb.xdrop_extend(full(S(0, "h", "AAAAAA")), full(S(1, "v", "AATAAA")), s10, 16)
    assert (r.score, r.h_ext, r.v_ext) == (4, 5, 6)
    with pytest.raises(xb.BandExceededError) as ei:
        xb.xdrop_extend(full(S(0, "h", "AAAAAA")), full(S(1, "v", "AATAAA")), s10, 2)
    assert ei.value.observed_spread == 3 and ei.value.cells == 3
    with pytest.raises(xb.InputError):
        xb.xdrop_extend(full(a), full(a), s3, 16, scratch=xb.BandBuffers(8))
    with pytest.raises(xb.InputError):
        xb.BandBuffers(0)


def test_seed_extension(xb):
    # align.cpp:268-309; test_align.cpp:243-302
    for e in VEC["seeds"]:
        store = xb.SequenceStore([xb.Sequence(0, "h", e["h"]), xb.Sequence(1, "v", e["v"])])
        t = xb.ExtensionTask(0, e["h_id"], e["v_id"], e["h_seed"], e["v_seed"])
        s = xb.ScoringScheme.match_mismatch(1, -1, -1, e["x"])
        if e["rc"] == 2:
            with pytest.raises(xb.DanglingReference):
                xb.extend_seed(t, store, e["k"], s, e["band"])
        elif e["rc"] == 3:
            with pytest.raises(xb.SeedOutOfBounds):
                xb.extend_seed(t, store, e["k"], s, e["band"])
        elif e["rc"] == 1:
            with pytest.raises(xb.BandExceededError) as ei:
                xb.extend_seed(t, store, e["k"], s, e["band"])
            assert ei.value.side == e["side"] and ei.value.observed_spread == e["spread"]
        else:
            a = xb.extend_seed(t, store, e["k"], s, e["band"])
            assert a.seed_score == e["seed_score"] and a.total == e["total"]
            assert _er(a.left) == expect_tuple(e["left"])
            assert _er(a.right) == expect_tuple(e["right"])


def _er(r):
    return (r.score, r.h_ext, r.v_ext, r.cells, r.delta_w)


def _config_pool(xb, ds):
    if ds.cfg == 3:
        a, c = blosum62()
        s = xb.ScoringScheme.from_matrix(xb.SubMatrix(a, c), -1, ds.x)
    else:
        s = xb.ScoringScheme.match_mismatch(1, -1, -1, ds.x)
    return xb.DevicePool(s, ds.symbols, ds.offsets)


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
@pytest.mark.parametrize("flags", [0, 1, 2, 128, 128 | 64, 32 | NO_LANES, 64 | 8, 64 | 8 | (2 << 8), 32 | 8 | NO_LANES,
                                   32 | 8 | (2 << 8) | NO_LANES, 32 | LANES, 32 | 8 | LANES, 32 | 8 | (2 << 8) | LANES],
                         ids=["auto", "unsorted", "warp_tier_only", "pilot_cascade", "thread_cascade", "group_cascade",
                              "thread_from_k16", "thread_from_k32", "group_from_k16", "group_from_k32",
                              "lane_cascade", "lane_from_k16", "lane_from_k32"])
def test_configs_vs_reference_golden(xb, cfg, flags):
    from paper_2304_08662_b200 import synth
    meta = load_json("configs_meta.json")[str(cfg)]
    ds = synth.make(cfg, meta["scale"])
    h = hashlib.sha256(ds.symbols.tobytes() + ds.offsets.tobytes() + ds.tasks.tobytes()).hexdigest()
    assert h == meta["input_sha256"]
    ref = np.load(os.path.join(os.path.dirname(__file__), "golden", f"cfg{cfg}_ref.npz"))
    pool = _config_pool(xb, ds)
    out, ss = xb.extend_tasks(pool, ds.tasks, ds.k, ds.band, exec_flags=flags)
    eq = result_rows_equal(out, ref["results"])
    assert eq.all(), f"{(~eq).sum()} of {len(eq)} sides differ; first {np.nonzero(~eq)[0][:5]}"
    assert (ss == ref["seed_score"]).all()


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_configs_sample_vs_oracle_full_size(xb, oracle, cfg):
    """BASELINE-size inputs: a seeded sample of tasks checked against the
    oracle, and the whole batch checked for run-to-run identity."""
    from paper_2304_08662_b200 import synth
    scale = {1: 1.0, 2: 0.2, 3: 1.0, 4: 0.1, 5: 0.02}[cfg]
    ds = synth.make(cfg, scale)
    pool = _config_pool(xb, ds)
    rng = np.random.default_rng(cfg)
    pick = np.sort(rng.choice(ds.n_tasks, size=min(ds.n_tasks, 300), replace=False))
    out, ss = xb.extend_tasks(pool, ds.tasks[pick], ds.k, ds.band)
    s = oracle_scheme(oracle, ["BLOSUM62", -1, ds.x] if cfg == 3 else [1, -1, -1, ds.x])
    exp, ess = oracle.extend_batch(ds.symbols, ds.offsets, ds.tasks[pick], ds.k, s, ds.band,
                                   threads=os.cpu_count() or 1)
    assert result_rows_equal(out, exp).all()
    assert (ss == ess).all()
    a, _ = xb.extend_tasks(pool, ds.tasks, ds.k, ds.band)
    # unsorted, lane groups throughout, one thread per unit, and K16 starts whose
    # escalations resume from saved records (past the record capacity on config 5);
    # K16 starts whose escalations a concurrent consumer takes while the start
    # tier runs (8: most units escalate) and the serial tail (4096)
    for flags in (1, 32 | NO_LANES, 32 | LANES, 64, 64 | 8, 32 | 8 | NO_LANES, 32 | 8 | LANES, 8, 4096, 8 | 4096):
        b, _ = xb.extend_tasks(pool, ds.tasks, ds.k, ds.band, exec_flags=flags)
        assert result_rows_equal(a, b).all(), flags
    # every sampled row inside the full run equals the sampled run
    full = a.reshape(-1, 2)[pick].reshape(-1)
    assert result_rows_equal(full, out).all()


def test_x_monotone_full_size(xb):
    """Size-independent property at BASELINE lengths (acceptance.cpp:355-375,
    test_align.cpp:186-200): raising X never lowers the score nor narrows the
    spread while the band suffices."""
    from paper_2304_08662_b200 import synth
    ds = synth.make(2, 0.05)
    res = []
    for x in (5, 15, 40):
        pool = xb.DevicePool(xb.ScoringScheme.match_mismatch(1, -1, -1, x), ds.symbols, ds.offsets)
        res.append(xb.extend_tasks(pool, ds.tasks, ds.k, 1024)[0])
    for lo, hi in zip(res, res[1:]):
        ok = (lo["status"] == 0) & (hi["status"] == 0)
        assert ok.mean() > 0.99
        assert (hi["score"][ok] >= lo["score"][ok]).all()
        assert (hi["delta_w"][ok] >= lo["delta_w"][ok]).all()


def test_self_extension_full_length(xb):
    """Perfect matches extend to the full view whatever the length
    (test_align.cpp:202-213): score = length, spread independent of length."""
    from paper_2304_08662_b200 import synth
    ds = synth.make(5, 0.0005)
    n = len(ds.offsets) - 1
    pool = xb.DevicePool(xb.ScoringScheme.match_mismatch(1, -1, -1, 6), ds.symbols, ds.offsets)
    t = np.zeros((n, 4), dtype=np.int64)
    t[:, 0] = t[:, 1] = np.arange(n)
    out, ss = xb.extend_tasks(pool, t, 0, 64)
    ln = np.diff(ds.offsets)
    right = out[1::2]
    assert (right["status"] == 0).all()
    assert (right["score"] == ln).all() and (right["h_ext"] == ln).all() and (right["v_ext"] == ln).all()
    assert len(set(right["delta_w"].tolist())) == 1


@pytest.mark.parametrize("flags", [0, 32 | NO_LANES, 128 | 64, 64 | 8, 32 | 8 | NO_LANES, 32 | LANES, 32 | 8 | LANES],
                         ids=["auto", "group", "thread_pilot", "thread_from_k16", "group_from_k16", "lane",
                              "lane_from_k16"])
def test_band_failures_and_escalation(xb, oracle, flags):
    """Wide windows: X large so spreads exceed 32 and 64 slots (tier escalation)
    and a band small enough that some sides fail with exact spread/cells."""
    rng = random.Random(7)
    entries = []
    for it in range(120):
        n = rng.randint(50, 900)
        h = bytes(rng.choice(b"ACGT") for _ in range(n))
        v = bytearray(h)
        for q in range(len(v)):
            if rng.random() < 0.25:
                v[q] = rng.choice(b"ACGT")
        entries.append((h, bytes(v)))
    even_resumes = 0
    for x, band in ((60, 1000), (120, 1000), (60, 70), (30, 40)):
        so = oracle.scheme_mm(1, -1, -1, x)
        sym = b"".join(h + v for h, v in entries)
        off = [0]
        for h, v in entries:
            off += [off[-1] + len(h), off[-1] + len(h) + len(v)]
        from paper_2304_08662_b200.capi import UNIT_DTYPE
        units = np.zeros(len(entries), dtype=UNIT_DTYPE)
        for q, (h, v) in enumerate(entries):
            units[q] = (2 * q, 2 * q + 1, 1, 1, 0, 0, len(h), len(v))
        pool = xb.DevicePool(xb.ScoringScheme.match_mismatch(1, -1, -1, x), sym, np.array(off))
        out = xb.extend_units(pool, units, band, exec_flags=flags)
        even_resumes += xb.xband.last_stats()["dbg"][5]
        for q, (h, v) in enumerate(entries):
            assert rec_tuple(out[q]) == rec_tuple(oracle.extend(h, v, so, band)), (x, band, q)
    if flags & ~(LANES | NO_LANES) == 32 | 8:
        # lane-group / lane tiers from K16 up: records written at even antidiagonals
        # take the first-step-in-fetch() path, and it was exercised here
        assert even_resumes > 0


def test_pipeline_drop_in(xb):
    """The reference pipeline's result rows (pipeline.cpp:99-137 +
    io.cpp:258-298) rebuilt from the batch API on the reference's own synthetic
    dataset equal the reference's rows byte for byte."""
    import ctypes  # noqa: F401
    rows = load_json("pipeline_rows.json")
    from oracle_py import REF_SO, Ref
    for name, p in rows.items():
        if not os.path.exists(REF_SO):
            pytest.skip("reference dataset generator not available on this host")
        R = Ref()
        sym, off, tasks = R.generate_synthetic(p["pairs"], p["length"], p["p_match"], p["k"],
                                               p["seed"], p.get("uniform_seed", False))
        store = xb.SequenceStore(
            [xb.Sequence(i, "s", sym[off[i]:off[i + 1]].tobytes().decode()) for i in range(len(off) - 1)])
        tl = [xb.ExtensionTask(t, *map(int, tasks[t])) for t in range(len(tasks))]
        s = xb.ScoringScheme.match_mismatch(1, -1, -1, p["x"])
        al, failed, _ = xb.extend_batch(store, tl, p["k"], s, p["band"])
        got = ["task_id\tside\tscore\th_ext\tv_ext\tcells\tdelta_w"]
        tot = 0
        for a in al:
            for side, r in (("L", a.left), ("R", a.right)):
                got.append(f"{a.task_id}\t{side}\t{r.score}\t{r.h_ext}\t{r.v_ext}\t{r.cells}\t{r.delta_w}")
            tot += a.total
        got.append(f"# total\t{tot}")
        for f in failed:
            got.append(f"# failed\ttask {f.task_id} side {f.side} spread {f.observed_spread}")
        assert got == p["rows"], name


def test_multi_device_sharding_same_results(xb):
    """xb_exec with several device ids shards tasks LPT across them (here two
    shards on one GPU: no collective, host gather by task index)."""
    from paper_2304_08662_b200 import synth
    ds = synth.make(5, 0.001)
    pool = _config_pool(xb, ds)
    a, sa = xb.extend_tasks(pool, ds.tasks, ds.k, ds.band)
    b, sb = xb.extend_tasks(pool, ds.tasks, ds.k, ds.band, n_devices=2, device_ids=[0, 0])
    assert result_rows_equal(a, b).all() and (sa == sb).all()
    st = xb.xband.last_stats()
    assert st["n_devices"] == 2


def test_batch_stream_same_results(xb):
    """extend_batches (one batch in flight ahead, pools re-uploaded every
    batch) returns, for each batch, exactly the synchronous call's rows;
    throughput-planned and latency-planned batches mixed in one stream."""
    from paper_2304_08662_b200 import synth
    ds = synth.make(5, 0.01)
    pools = [_config_pool(xb, ds), _config_pool(xb, ds)]
    cuts = [ds.tasks, ds.tasks[:500], ds.tasks[7:20000], ds.tasks]
    want = [xb.extend_tasks(pools[0], t, ds.k, ds.band) for t in cuts]
    stats = []
    got = list(xb.xband.extend_batches(((pools[i % 2], t) for i, t in enumerate(cuts)), ds.k, ds.band,
                                       reupload=True, stats=stats))
    assert len(got) == len(cuts) == len(stats)
    for (a, sa), (b, sb) in zip(want, got):
        assert result_rows_equal(a, b).all() and (sa == sb).all()
    assert all(s["h2d_bytes"] > 0 for s in stats)  # every batch re-uploaded its pool
    with pytest.raises(ValueError):  # one pool cannot be re-uploaded under an in-flight batch
        list(xb.xband.extend_batches(((pools[0], t) for t in cuts[:2]), ds.k, ds.band, reupload=True))
    # without re-upload one pool serves the whole stream
    got = list(xb.xband.extend_batches(((pools[0], t) for t in cuts), ds.k, ds.band))
    for (a, sa), (b, sb) in zip(want, got):
        assert result_rows_equal(a, b).all() and (sa == sb).all()


def test_sweep_band_matches_reference(xb):
    """§8(f) band survey on the GPU (pipeline.cpp:181-208): the reference's TSV
    byte for byte, including acceptance criterion 2 (L=20000, p=0.9, X=15:
    spread 20) and criterion 3's grid, and the paper-scale grid."""
    g = load_json("sweep_band.json")
    for c in g["sweeps"]:
        assert xb.sweep_band(c["length"], c["xs"], c["ps"], c["seed"]) == c["tsv"], c["source"]


def test_route_guard_mixed_batch(xb, oracle):
    """Units whose drift-space values could pass 2^23 (host/prep bound:
    max_score*min(n,m) + beta*(n+m+2) + X) go to the warp tier, the rest to
    the thread tiers, in one batch, both exact.  The bound is set by the view
    lengths (scheme +1/-2/-2: bound = min(n,m) + 2(n+m+2) + X + 2): 3M-base
    views route to the warp tier, 1.5M-base and short ones do not.  A
    ~1000-base shared prefix, then unrelated sequence (negative drift under
    this scheme) keeps every X-drop short."""
    rng = np.random.default_rng(23)
    acgt = np.frombuffer(b"ACGT", dtype=np.uint8)
    entries = []
    for n in (3_000_000, 1_500_000, 700, 3_000_001, 150):
        pre = int(min(n, 1000))
        h = rng.choice(acgt, n)
        v = rng.choice(acgt, n)
        v[:pre] = h[:pre]
        mut = rng.random(pre) < 0.05
        v[:pre][mut] = rng.choice(acgt, int(mut.sum()))
        entries.append((h.tobytes(), v.tobytes()))
    sym = b"".join(h + v for h, v in entries)
    off = [0]
    for h, v in entries:
        off += [off[-1] + len(h), off[-1] + len(h) + len(v)]
    from paper_2304_08662_b200.capi import UNIT_DTYPE
    units = np.zeros(len(entries), dtype=UNIT_DTYPE)
    for q, (h, v) in enumerate(entries):
        units[q] = (2 * q, 2 * q + 1, 1, 1, 0, 0, len(h), len(v))
    band = 256
    pool = xb.DevicePool(xb.ScoringScheme.match_mismatch(1, -2, -2, 10), sym, np.array(off))
    out = xb.extend_units(pool, units, band)
    st = xb.xband.last_stats()
    assert st["units_tier"][WARP_TIER] == 2 and sum(st["units_tier"][:WARP_TIER]) == 3, st["units_tier"]
    assert sum(st["escalated"]) == 0, st["escalated"]
    so = oracle.scheme_mm(1, -2, -2, 10)
    for q, (h, v) in enumerate(entries):
        assert rec_tuple(out[q]) == rec_tuple(oracle.extend(h, v, so, band)), q


def test_million_base_self_extension_both_directions(xb):
    """Maximum-size views: a 1,048,579-base read against itself from a seed in
    the middle, left (reversing view) and right, plus a 3-base mismatch tail."""
    rng = np.random.default_rng(5)
    n = (1 << 20) + 3
    s = rng.choice(np.frombuffer(b"ACGT", dtype=np.uint8), n).tobytes()
    t = s[:-3] + bytes((b"ACGT"[(b"ACGT".index(c) + 1) % 4] for c in s[-3:]))
    pool = xb.DevicePool(xb.ScoringScheme.match_mismatch(1, -1, -1, 10), s + t,
                         np.array([0, n, 2 * n], dtype=np.int64))
    seed = n // 2 - 7
    out, ss = xb.extend_tasks(pool, np.array([[0, 1, seed, seed]]), 17, 64)
    L, R = out[0], out[1]
    assert ss[0] == 17
    assert (L["score"], L["h_ext"], L["v_ext"]) == (seed, seed, seed)
    right = n - seed - 17
    assert (R["score"], R["h_ext"], R["v_ext"]) == (right - 3, right - 3, right - 3)
    assert L["status"] == 0 and R["status"] == 0


@pytest.mark.parametrize("case", ["dna_table_2bit", "protein_bytes"])
def test_table_modes_at_throughput_scale(xb, oracle, case):
    """The table modes (2-bit pool with a non-unit DNA scheme; byte pool with
    BLOSUM62) through the thread tiers at batch scale (throughput planning:
    pilot, K24 threads, resumed escalations, streamed byte windows, sentinel
    bytes at view ends), a seeded sample checked against the oracle."""
    from paper_2304_08662_b200 import synth
    if case == "dna_table_2bit":
        ds = synth.make(2, 0.2)
        s = xb.ScoringScheme.match_mismatch(2, -3, -5, 40)
        so = oracle.scheme_mm(2, -3, -5, 40)
    else:
        ds = synth.make(3, 1.0)
        s = xb.ScoringScheme.from_matrix(xb.parse_submatrix(synth.blosum62_text()), -1, ds.x)
        so = oracle_scheme(oracle, ["BLOSUM62", -1, ds.x])
    pool = xb.DevicePool(s, ds.symbols, ds.offsets)
    assert pool.bits_per_symbol == (2 if case == "dna_table_2bit" else 5)
    out, ss = xb.extend_tasks(pool, ds.tasks, ds.k, ds.band, exec_flags=128 | 64)  # THROUGHPUT, threads
    st = xb.xband.last_stats()
    assert not st["start_lane_groups"]
    rng = np.random.default_rng(7)
    pick = np.sort(rng.choice(ds.n_tasks, size=min(ds.n_tasks, 250), replace=False))
    exp, ess = oracle.extend_batch(ds.symbols, ds.offsets, ds.tasks[pick], ds.k, so, ds.band,
                                   threads=os.cpu_count() or 1)
    assert result_rows_equal(out.reshape(-1, 2)[pick].reshape(-1), exp).all()
    assert (ss[pick] == ess).all()
    g, _ = xb.extend_tasks(pool, ds.tasks, ds.k, ds.band, exec_flags=128)  # lane-group escalations
    assert result_rows_equal(g, out).all()


def test_config5_full_size(xb, oracle):
    """Config 5 at BASELINE size (2,000,000 extensions, 2.43e11 cells), the
    bench workload: a seeded sample of 3000 tasks against the oracle; the
    concurrent escalation consumer and the serial tail give identical rows;
    size-independent properties of the whole batch (every side OK, cells
    and delta_w within the band, stats consistent with the rows)."""
    from paper_2304_08662_b200 import synth
    ds = synth.make(5, 1.0)
    assert ds.n_tasks == 2_000_000
    pool = _config_pool(xb, ds)
    out, ss = xb.extend_tasks(pool, ds.tasks, ds.k, ds.band)
    st = xb.xband.last_stats()
    assert not st["start_lane_groups"] and sum(st["units_tier"]) == 2 * ds.n_tasks
    assert sum(st["cells_tier"]) == int(out["cells"].sum())
    assert (out["status"] == 0).all() and (out["delta_w"] <= ds.band).all()
    rng = np.random.default_rng(5)
    pick = np.sort(rng.choice(ds.n_tasks, size=3000, replace=False))
    exp, ess = oracle.extend_batch(ds.symbols, ds.offsets, ds.tasks[pick], ds.k,
                                   oracle_scheme(oracle, [1, -1, -1, ds.x]), ds.band,
                                   threads=os.cpu_count() or 1)
    assert result_rows_equal(out.reshape(-1, 2)[pick].reshape(-1), exp).all()
    assert (ss[pick] == ess).all()
    serial, ss2 = xb.extend_tasks(pool, ds.tasks, ds.k, ds.band, exec_flags=4096)  # XB_FLAG_SERIAL_TAIL
    assert result_rows_equal(serial, out).all() and (ss2 == ss).all()


def test_edge_batches(xb, oracle):
    """Empty batches, one-task batches, zero-length views (seeds at either end
    of a sequence, sequences exactly k long), N in DNA (byte pool), and a
    throughput-size batch of one repeated task: each against the oracle."""
    s = xb.ScoringScheme.match_mismatch(1, -1, -1, 10)
    so = oracle.scheme_mm(1, -1, -1, 10)
    rng = np.random.default_rng(11)
    base = "".join(rng.choice(list("ACGT"), 300))
    seqs = [base, base[:150] + "T" + base[151:], base[:17], "AC" + base[:40], base[100:117]]
    syms = np.frombuffer("".join(seqs).encode(), dtype=np.uint8)
    off = np.cumsum([0] + [len(x) for x in seqs]).astype(np.int64)
    pool = xb.DevicePool(s, syms, off)
    k = 17
    tasks = np.array([[0, 1, 0, 0],          # left views empty
                      [0, 1, 283, 283],      # right views empty
                      [2, 2, 0, 0],          # sequence exactly k long: both views empty
                      [0, 3, 0, 2],          # left view of h empty, of v two bases
                      [4, 0, 0, 100],        # h exactly k, seed inside v
                      [1, 0, 150, 150]], dtype=np.int64)
    out, ss = xb.extend_tasks(pool, tasks, k, 64)
    exp, ess = oracle.extend_batch(syms, off, tasks, k, so, 64, threads=1)
    assert result_rows_equal(out, exp).all() and (ss == ess).all()
    one, s1 = xb.extend_tasks(pool, tasks[3:4], k, 64)
    assert result_rows_equal(one, exp[6:8]).all() and s1[0] == ess[3]
    empty, se = xb.extend_tasks(pool, tasks[:0], k, 64)
    assert len(empty) == 0 and len(se) == 0
    got = list(xb.xband.extend_batches([(pool, tasks[:0]), (pool, tasks)], k, 64))
    assert len(got[0][0]) == 0 and result_rows_equal(got[1][0], exp).all()
    # N never matches, so the pool falls back to byte codes
    seqs_n = [base[:120] + "N" * 5 + base[125:], base]
    sn = np.frombuffer("".join(seqs_n).encode(), dtype=np.uint8)
    on = np.cumsum([0] + [len(x) for x in seqs_n]).astype(np.int64)
    pn = xb.DevicePool(s, sn, on)
    assert pn.bits_per_symbol == 5
    tn = np.array([[0, 1, 200, 200], [1, 0, 10, 10], [0, 0, 60, 60]], dtype=np.int64)
    o2, s2 = xb.extend_tasks(pn, tn, k, 64)
    e2, es2 = oracle.extend_batch(sn, on, tn, k, so, 64, threads=1)
    assert result_rows_equal(o2, e2).all() and (s2 == es2).all()
    # one task repeated at throughput scale: every row equals the single run
    rep = np.repeat(tasks[5:6], 60000, axis=0)
    o3, _ = xb.extend_tasks(pool, rep, k, 64)
    assert not xb.xband.last_stats()["start_lane_groups"]
    assert result_rows_equal(o3, np.tile(exp[10:12], 60000)).all()


def test_pool_grows_after_upload(xb, oracle):
    """A pool used by a batch, then grown (more sequences; then an 'N' that
    widens it from 2-bit to byte codes), then used again: every batch equals
    the oracle over the pool's contents at that point (the device copy is
    reallocated when the packed image outgrows it)."""
    rng = random.Random(77)

    def rnd(n, alpha="ACGT"):
        return "".join(rng.choice(alpha) for _ in range(n))

    scheme = xb.ScoringScheme.match_mismatch(1, -1, -1, 12)
    pool = xb.DevicePool(scheme, b"", np.zeros(1, dtype=np.int64))
    seqs = []

    def grow(count, alpha="ACGT"):
        for _ in range(count):
            base = rnd(rng.randint(300, 3000), alpha)
            seqs.append(base)
            assert pool.add(base) == len(seqs) - 1

    def check():
        sym = "".join(seqs).encode()
        off = np.zeros(len(seqs) + 1, dtype=np.int64)
        np.cumsum([len(s) for s in seqs], out=off[1:])
        tasks = []
        for _ in range(400):
            h, v = rng.randrange(len(seqs)), rng.randrange(len(seqs))
            hs = rng.randrange(len(seqs[h]) - 17)
            vs = rng.randrange(len(seqs[v]) - 17)
            tasks.append((h, v, hs, vs))
        t = np.array(tasks, dtype=np.int64)
        out, ss = xb.extend_tasks(pool, t, 17, 256)
        exp, ess = oracle.extend_batch(np.frombuffer(sym, np.uint8), off, t, 17,
                                       oracle.scheme_mm(1, -1, -1, 12), 256)
        assert result_rows_equal(out, exp).all()
        assert (ss == ess).all()

    grow(20)
    assert pool.bits_per_symbol == 2
    check()
    grow(300)                 # far more words than the first upload held
    check()
    grow(5, "ACGTN")          # first N: the image widens to byte codes (4x the words)
    assert pool.bits_per_symbol == 5
    check()
    grow(50)
    check()


# Workloads whose live windows outgrow K64 (large X, low identity, the
# reference's default band 1024): the wide tiers (one warp per unit, K128..
# K1024, xb_wide.cu) carry them, entered from K64 escalations (resume
# records from the thread, lane-group and pilot paths) or as the start tier.
WIDE_CASES = {
    "c4_x100": (4, 0.002, 100, 1024, "mm"),
    "c2_x40": (2, 0.01, 40, 1024, "mm"),
    "c5_x60_band512": (5, 0.0005, 60, 512, "mm"),
    "c3_blosum_x80": (3, 0.01, 80, 1024, "blosum"),
    "c4_x300_band200": (4, 0.001, 300, 200, "mm"),  # band failures inside the wide tiers
}


@pytest.mark.parametrize("case", sorted(WIDE_CASES))
@pytest.mark.parametrize("flags", [0, 128, 32, 64 | 8, 8 | (WIDE_FIRST << 8), 8 | ((WIDE_FIRST + 1) << 8),
                                   8 | ((WARP_TIER - 1) << 8), 16],
                         ids=["auto", "pilot", "groups", "thread_k16", "wide_k96", "wide_k128", "wide_k1024",
                              "esc_to_warp"])
def test_wide_tiers_vs_oracle(xb, oracle, case, flags):
    from paper_2304_08662_b200 import synth
    cfg, scale, x, band, kind = WIDE_CASES[case]
    ds = synth.make(cfg, scale)
    if kind == "blosum":
        a, c = blosum62()
        s = xb.ScoringScheme.from_matrix(xb.SubMatrix(a, c), -1, x)
        os_ = oracle_scheme(oracle, ["BLOSUM62", -1, x])
    else:
        s = xb.ScoringScheme.match_mismatch(1, -1, -1, x)
        os_ = oracle_scheme(oracle, [1, -1, -1, x])
    pool = xb.DevicePool(s, ds.symbols, ds.offsets)
    out, ss = xb.extend_tasks(pool, ds.tasks, ds.k, band, exec_flags=flags)
    st = xb.xband.last_stats()
    exp, ess = oracle.extend_batch(ds.symbols, ds.offsets, ds.tasks, ds.k, os_, band,
                                   threads=os.cpu_count() or 1)
    eq = result_rows_equal(out, exp)
    assert eq.all(), f"{(~eq).sum()} of {len(eq)} sides differ; first {np.nonzero(~eq)[0][:5]}"
    assert (ss == ess).all()
    wide_units = sum(st["units_tier"][WIDE_FIRST:WARP_TIER])
    if flags & 8 and flags >> 8 >= WIDE_FIRST:  # wide start: every thread-tier-routable unit is wide
        assert sum(st["units_tier"][:WIDE_FIRST]) == 0 and wide_units > 0, st["units_tier"]
    elif flags != 16 and (exp["delta_w"] > 66).any():  # windows beyond K64 (+ slack) reach the wide tiers
        assert wide_units > 0, st["units_tier"]
    if case == "c4_x300_band200":
        assert (out["status"] == 1).any() and (out["status"] == 0).any()


def test_wide_tier_is_the_start_for_wide_batches(xb):
    """Throughput planning: when most of the pilot sample outgrows K64, the
    whole batch starts on the wide tiers (no thread-tier pass first)."""
    from paper_2304_08662_b200 import synth
    ds = synth.make(4, 0.02)
    s = xb.ScoringScheme.match_mismatch(1, -1, -1, 200)
    pool = xb.DevicePool(s, ds.symbols, ds.offsets)
    xb.extend_tasks(pool, ds.tasks, ds.k, 1024, exec_flags=128)
    st = xb.xband.last_stats()
    assert st["start_tier"] >= 5, st
    assert sum(st["units_tier"][:WIDE_FIRST]) == 0 and sum(st["units_tier"][WIDE_FIRST:WARP_TIER]) > 0, st["units_tier"]


def test_locality_shards_same_results(xb):
    """Multi-device batches with locality-aware shards (XB_FLAG_LOCALITY):
    each device uploads only the sequences its shard references; rows equal
    the single-device run (two shards on one GPU here)."""
    from paper_2304_08662_b200 import synth
    ds = synth.make(5, 0.01)
    s = xb.ScoringScheme.match_mismatch(1, -1, -1, ds.x)
    pool = xb.DevicePool(s, ds.symbols, ds.offsets)
    a, sa = xb.extend_tasks(pool, ds.tasks, ds.k, ds.band)
    full_h2d = xb.xband.last_stats()["h2d_bytes"]
    for locality in (False, True):
        pool2 = xb.DevicePool(s, ds.symbols, ds.offsets)
        b, sb = xb.extend_tasks(pool2, ds.tasks, ds.k, ds.band, n_devices=2, device_ids=[0, 0],
                                exec_flags=8192 if locality else 0)
        assert result_rows_equal(a, b).all() and (sa == sb).all()
        h2d = xb.xband.last_stats()["h2d_bytes"]
        if locality:  # the two shards together upload about one pool, not two
            assert h2d < 1.4 * full_h2d, (h2d, full_h2d)


def test_partial_residency_uploads_each_sequence_once(xb, oracle):
    """A batch referencing a few sequences of a large pool uploads only their
    words; a later batch over other sequences uploads the missing ones; the
    rows equal the oracle's over the whole pool."""
    from paper_2304_08662_b200 import synth
    ds = synth.make(5, 0.02)
    s = xb.ScoringScheme.match_mismatch(1, -1, -1, ds.x)
    pool = xb.DevicePool(s, ds.symbols, ds.offsets)
    image = (len(ds.symbols) + 2 * 4096) / 4
    os_ = oracle_scheme(oracle, [1, -1, -1, ds.x])
    rng = np.random.default_rng(3)
    seen = np.zeros(len(ds.offsets) - 1, dtype=bool)
    for rnd in range(3):
        pick = np.sort(rng.choice(ds.n_tasks, size=150, replace=False))
        t = ds.tasks[pick]
        out, ss = xb.extend_tasks(pool, t, ds.k, ds.band)
        h2d = xb.xband.last_stats()["h2d_bytes"]
        ref = np.unique(np.concatenate([t[:, 0], t[:, 1]]))
        new = ref[~seen[ref]]
        seen[ref] = True
        words = np.diff(ds.offsets)[new].sum() / 4
        assert h2d < 150 * 32 + 16 * (len(ds.offsets) - 1) + 2 * words + 4096 + 0.02 * image, (rnd, h2d, words)
        exp, ess = oracle.extend_batch(ds.symbols, ds.offsets, t, ds.k, os_, ds.band)
        assert result_rows_equal(out, exp).all() and (ss == ess).all()

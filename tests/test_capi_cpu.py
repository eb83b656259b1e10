"""CPU: the C-ABI library loads, exports every declared symbol, validates
inputs like the reference, packs pools, and generates the configs
deterministically.  No kernel is launched here (no GPU in this container)."""
import ctypes as C
import hashlib
import re

import numpy as np
import pytest

from helpers import blosum62, load_json

import paper_2304_08662_b200 as xb
from paper_2304_08662_b200 import capi, synth


def test_exports_match_header():
    hdr = open(capi.os.path.join(capi.os.path.dirname(capi.HERE), "include", "xdrop_b200.h")).read()
    declared = set(re.findall(r"\b(xb_[a-z0-9_]+)\s*\(", hdr))
    assert declared == set(capi.EXPORTED)
    L = capi.lib()
    for name in declared:
        assert hasattr(L, name), name
    assert L.xb_version().decode().startswith("xdrop_b200")


def test_flag_constants_match_header():
    """The Python binding's XB_FLAG_* / tier constants are the header's."""
    hdr = open(capi.os.path.join(capi.os.path.dirname(capi.HERE), "include", "xdrop_b200.h")).read()
    flags = dict(re.findall(r"#define\s+(XB_FLAG_[A-Z_]+)\s+(\d+)", hdr))
    assert {"XB_FLAG_LANES", "XB_FLAG_NO_LANES", "XB_FLAG_GROUP", "XB_FLAG_LOCALITY"} <= set(flags)
    for name, val in flags.items():
        assert getattr(capi, name) == int(val), name
    assert len(set(flags.values())) == len(flags)  # distinct bits
    assert capi.NUM_TIERS == int(re.search(r"#define\s+XB_NUM_TIERS\s+(\d+)", hdr).group(1))
    # the kernel a tier ran on, as the reports name it
    st = {"start_tier": 0, "start_lane_groups": 2}
    assert capi.tier_kernel_name(0, st) == "lane_k16"
    assert capi.tier_kernel_name(0, {"start_tier": 0, "start_lane_groups": 1}) == "group_k16"
    assert capi.tier_kernel_name(1, {"start_tier": 1, "start_lane_groups": 0}) == "thread_k24"


def test_plan_group_family():
    """The planner's choice between the 4-lane groups (1) and the lane tiers (2)
    for latency-planned batches, at the points measured on a 148-SM B200
    (DESIGN.md 4.2b): est_max = the longest unit's antidiagonals, est_sum = the
    batch's."""
    L = capi.lib()
    f = lambda table, nu, lmax, total: L.xb_plan_group_family(148, table, nu, float(lmax), float(total))
    # config 1 (1,000-antidiagonal units) at x1, x2, x3, x4
    assert [f(0, n, 990, 990 * n) for n in (2000, 4000, 6000, 8000)] == [2, 2, 1, 1]
    # config 2 (uniform up to 20,000) at x0.1 .. x1
    assert [f(0, n, 20000, 10000 * n) for n in (2000, 4000, 8000, 12000, 16000, 20000)] == [2, 2, 2, 2, 1, 1]
    # config 3 (protein, table mode, up to ~9,930) at x0.1 .. x1
    assert [f(1, n, 9930, 2950 * n) for n in (2000, 4000, 8000, 12000, 16000, 20000)] == [2, 2, 2, 2, 2, 1]
    # a single task is pure latency; no estimate falls back to the unit count
    assert f(0, 2, 20000, 30000) == 2 and f(1, 2, 5000, 8000) == 2
    assert f(0, 2000, 0, 0) == 2 and f(0, 20000, 0, 0) == 1
    # more work at the same longest unit never moves a batch to the lane tiers
    for nu in (3000, 9000, 30000):
        picks = [f(0, nu, 10000, w) for w in (1e6, 1e7, 1e8, 1e9, 1e10)]
        assert picks == sorted(picks, reverse=True), picks


def test_parse_submatrix_matches_reference():
    a, c = blosum62()  # produced by the reference's parse_submatrix
    m = xb.parse_submatrix(synth.blosum62_text())
    assert m.alphabet == a and m.cells == c
    s = xb.ScoringScheme.from_matrix(m, -1, 20)
    assert s.sim("A", "A") == 4 and s.sim("W", "W") == 11 and s.sim("*", "*") == 1  # test_scoring.cpp:89-98
    assert all(s.sim(p, q) == s.sim(q, p) for p in a for q in a)
    with pytest.raises(xb.UnknownSymbol):
        s.sim("a", "A")
    with pytest.raises(xb.InputError):
        xb.parse_submatrix("   A  B\nA 1 2\nB 1\n")  # NonSquare
    with pytest.raises(xb.InputError):
        xb.parse_submatrix("   A  B\nB 1 2\nA 1 2\n")  # row order != header


def test_scheme_validation_and_n_rule():
    with pytest.raises(xb.InputError):
        xb.ScoringScheme.match_mismatch(0, -1, -1, 3)
    with pytest.raises(xb.InputError):
        xb.ScoringScheme.match_mismatch(1, 1, -1, 3)
    with pytest.raises(xb.InputError):
        xb.ScoringScheme.match_mismatch(1, -1, 0, 3)
    with pytest.raises(xb.InputError):
        xb.ScoringScheme.match_mismatch(1, -1, -1, -1)
    s = xb.ScoringScheme.match_mismatch(2, -3, -1, 3)
    assert s.sim("A", "A") == 2 and s.sim("A", "C") == -3
    assert s.sim("N", "N") == -3  # N never matches (scoring.cpp:25-31)


def test_pool_packing_choice_and_validation():
    s = xb.ScoringScheme.match_mismatch(1, -1, -1, 5)
    p = xb.DevicePool(s, b"ACGTACGT", np.array([0, 4, 8]))
    assert p.bits_per_symbol == 2
    p2 = xb.DevicePool(s, b"ACGNACGT", np.array([0, 4, 8]))
    assert p2.bits_per_symbol == 5
    with pytest.raises(xb.UnknownSymbol):
        xb.DevicePool(s, b"ACGUACGT", np.array([0, 4, 8]))
    with pytest.raises(xb.UnknownSymbol):
        xb.DevicePool(s, b"acgt", np.array([0, 4]))


def test_task_validation_precedes_device():
    s = xb.ScoringScheme.match_mismatch(1, -1, -1, 5)
    p = xb.DevicePool(s, b"ACGTACGT", np.array([0, 4, 8]))
    with pytest.raises(xb.DanglingReference):
        xb.extend_tasks(p, np.array([[0, 7, 0, 0]]), 2, 8)
    with pytest.raises(xb.SeedOutOfBounds):
        xb.extend_tasks(p, np.array([[0, 1, 3, 0]]), 2, 8)
    with pytest.raises(xb.SeedOutOfBounds):
        xb.extend_tasks(p, np.array([[0, 1, 0, 4]]), 1, 8)
    with pytest.raises(xb.InputError):
        xb.extend_tasks(p, np.array([[0, 1, 0, 0]]), 1, 0)  # band < 1


def test_no_cpu_fallback():
    if capi.lib().xb_device_count() > 0:
        pytest.skip("a GPU is visible")
    s = xb.ScoringScheme.match_mismatch(1, -1, -1, 5)
    p = xb.DevicePool(s, b"ACGTACGT", np.array([0, 4, 8]))
    with pytest.raises(xb.xband.DeviceError, match="no CUDA device"):
        xb.extend_tasks(p, np.array([[0, 1, 0, 0]]), 2, 8)
    # the batch stream (bench e2e) has no fallback either, and releases what it holds
    with pytest.raises(xb.xband.DeviceError, match="no CUDA device"):
        list(xb.xband.extend_batches([(p, np.array([[0, 1, 0, 0]]))], 2, 8))


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_synth_matches_golden_inputs(cfg):
    meta = load_json("configs_meta.json")[str(cfg)]
    ds = synth.make(cfg, meta["scale"])
    h = hashlib.sha256(ds.symbols.tobytes() + ds.offsets.tobytes() + ds.tasks.tobytes()).hexdigest()
    assert h == meta["input_sha256"]
    assert (ds.k, ds.x, ds.band) == (meta["k"], meta["x"], meta["band"])
    # seeds are exact k-mers on both sides
    for t in ds.tasks[:50]:
        a = ds.symbols[ds.offsets[t[0]] + t[2]: ds.offsets[t[0]] + t[2] + ds.k]
        b = ds.symbols[ds.offsets[t[1]] + t[3]: ds.offsets[t[1]] + t[3] + ds.k]
        assert (a == b).all()


def test_synth_thread_count_invariance():
    a = synth.make(5, 0.0003, threads=1)
    b = synth.make(5, 0.0003, threads=8)
    assert (a.symbols == b.symbols).all() and (a.tasks == b.tasks).all()


def test_split_lr_mirror():
    # partition.cpp:45-81 / test_partition.cpp:69-105 shape
    store = xb.SequenceStore([xb.Sequence(0, "h", "A" * 100), xb.Sequence(1, "v", "A" * 80)])
    l, r = xb.split_lr(xb.ExtensionTask(3, 0, 1, 30, 20), store, 17)
    assert (l.unit_id, l.h_len, l.v_len, l.est_cost) == (6, 30, 20, 600)
    assert (r.unit_id, r.h_origin, r.v_origin, r.h_len, r.v_len) == (7, 47, 37, 53, 43)
    with pytest.raises(xb.SeedOutOfBounds):
        xb.split_lr(xb.ExtensionTask(0, 0, 1, 90, 0), store, 17)
    assert xb.gcups(1000, 1000, 1e-3) == pytest.approx(1.0)


def test_synth_pairs_match_reference_generator():
    """xb_synth_pairs restates generate_synthetic (io.cpp:198-255): same bytes,
    offsets and seed tasks as the reference's own generator."""
    import hashlib
    g = load_json("sweep_band.json")
    for c in g["synth"]:
        sym, off, tasks = synth.pairs(c["pairs"], c["length"], c["p_match"], c["k"], c["seed"],
                                      c["uniform_seed"])
        assert hashlib.sha256(sym.tobytes()).hexdigest() == c["symbols_sha256"], c
        assert off.tolist() == c["offsets"] and tasks.tolist() == c["tasks"], c
    with pytest.raises(xb.InputError):
        synth.pairs(1, 10, 0.9, 17)  # k > length (io.cpp:200-202)
    with pytest.raises(xb.InputError):
        synth.pairs(1, 10, 0.9, 0)


def test_sweep_band_validation_precedes_device():
    with pytest.raises(xb.InputError):
        xb.sweep_band(100, [-1], [0.9])  # X < 0 (scoring.cpp:17-20)
    with pytest.raises(xb.InputError):
        xb.sweep_band(10, [5], [0.9])  # 17-mer seed longer than the pair
    assert xb.sweep_band(100, [], [0.9]) == "x\terror_rate\tdelta_w\n"


def test_pool_packs_incrementally():
    """The pool keeps only the packed image: 2-bit while every sequence is
    ACGT, byte codes from the first N on; ids are dense across adds."""
    import paper_2304_08662_b200 as xb
    s = xb.ScoringScheme.match_mismatch(1, -1, -1, 5)
    p = xb.DevicePool(s, b"ACGT", np.array([0, 2, 4], dtype=np.int64))
    assert p.bits_per_symbol == 2
    assert p.add("ACGTACGT" * 1000) == 2
    assert p.bits_per_symbol == 2
    assert p.add("ACNGT") == 3
    assert p.bits_per_symbol == 5
    assert p.add("T") == 4
    assert xb.capi.lib().xb_pool_size(p._h) == 5
    assert xb.capi.lib().xb_pool_seq_len(p._h, 3) == 5
    with pytest.raises(xb.UnknownSymbol):
        p.add("ACGX")
    m = xb.ScoringScheme.from_matrix(xb.SubMatrix("AB", [2, -1, -1, 3]), -1, 4)
    q = xb.DevicePool(m, b"ABBA", np.array([0, 4], dtype=np.int64))
    assert q.bits_per_symbol == 5


def test_package_blosum62_matches_reference_fixture():
    """The package's BLOSUM62 constant equals the reference's parse of
    proj/data/BLOSUM62 (tests/golden/blosum62.json, made by the reference)."""
    from paper_2304_08662_b200 import blosum62 as B
    a, c = blosum62()
    assert B.ALPHABET == a and list(B.CELLS) == list(c)
    m = xb.parse_submatrix(B.text())
    assert m.alphabet == a and list(m.cells) == list(c)


def test_shard_tasks_validation_and_modes():
    """xb_shard_tasks (host-only): both modes cover every task once, the
    assignment is deterministic, and task errors mirror xb_extend_batch."""
    ds = synth.make(5, 0.002)
    pool = xb.DevicePool(xb.ScoringScheme.match_mismatch(1, -1, -1, ds.x), ds.symbols, ds.offsets)
    for loc in (False, True):
        a = xb.xband.shard_tasks(pool, ds.tasks, ds.k, 3, locality=loc)
        b = xb.xband.shard_tasks(pool, ds.tasks, ds.k, 3, locality=loc)
        assert (a == b).all() and set(np.unique(a)) == {0, 1, 2}
        one = xb.xband.shard_tasks(pool, ds.tasks, ds.k, 1, locality=loc)
        assert (one == 0).all()
    bad = ds.tasks.copy()
    bad[5, 0] = len(ds.offsets) + 10  # an unknown sequence
    with pytest.raises(xb.DanglingReference):
        xb.xband.shard_tasks(pool, bad, ds.k, 2)
    bad = ds.tasks.copy()
    bad[7, 2] = 10 ** 9  # a seed past its sequence
    with pytest.raises(xb.SeedOutOfBounds):
        xb.xband.shard_tasks(pool, bad, ds.k, 2, locality=True)

"""§8(f) item 2: the reference's input formats parsed natively (csrc/
xb_ingest.cpp) against the reference's own parsers (proj/src/io.cpp:58-196):
identical records, names, tasks, error kinds, lines and messages; seeded fuzz
and multi-threaded large inputs against the live reference (oracle/_ref)."""
import os
import random
import sys

import numpy as np
import pytest

from helpers import load_json
from ingest_cases import FASTA, OVERLAPS, SEEDS

import paper_2304_08662_b200 as xb
from paper_2304_08662_b200 import capi

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "oracle"))
from oracle_py import REF_SO  # noqa: E402

GOLD = load_json("ingest.json")


def ours_fasta(text, allowed, threads=0):
    try:
        r = xb.FastaRecords(text, allowed, threads)
    except xb.InputError as e:
        return ("error", type(e).__name__, getattr(e, "line", 0), str(e))
    return (r.symbols.tobytes().decode(), r.offsets.tolist(), r.names)


def ours_tasks(text, overlaps):
    try:
        t = (xb.parse_overlaps if overlaps else xb.parse_seeds)(text)
    except xb.InputError as e:
        return ("error", type(e).__name__, getattr(e, "line", 0), str(e))
    return [[int(r["task_id"]), int(r["h_id"]), int(r["v_id"]), int(r["h_seed"]), int(r["v_seed"])] for r in t]


def gold(g):
    if "error" in g:
        return ("error", capi.XB_PARSE_NAMES[g["error"]], g["line"], g["message"])
    if "tasks" in g:
        return g["tasks"]
    return (g["symbols"], g["offsets"], g["names"])


@pytest.mark.parametrize("i", range(len(FASTA)))
def test_fasta_cases_match_reference(i):
    text, allowed = FASTA[i]
    assert ours_fasta(text, allowed) == gold(GOLD["fasta"][i])


@pytest.mark.parametrize("i", range(len(SEEDS)))
def test_seed_list_cases_match_reference(i):
    assert ours_tasks(SEEDS[i], False) == gold(GOLD["seeds"][i])


@pytest.mark.parametrize("i", range(len(OVERLAPS)))
def test_overlap_cases_match_reference(i):
    assert ours_tasks(OVERLAPS[i], True) == gold(GOLD["overlaps"][i])


def ref():
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref not built")
    from oracle_py import Ref
    return Ref()


def ref_fasta(R, text, allowed):
    r = R.parse_fasta(text.encode(), allowed)
    if r[0] == "error":
        return ("error", capi.XB_PARSE_NAMES[r[1]], r[2], r[3])
    return (r[0].decode(), r[1].tolist(), r[2])


def ref_tasks(R, text, overlaps):
    r = R.parse_tasks(text.encode(), overlaps)
    if isinstance(r, tuple):
        return ("error", capi.XB_PARSE_NAMES[r[1]], r[2], r[3])
    return r.tolist()


def random_fasta(rng, n_rec, corrupt):
    lines = []
    for q in range(n_rec):
        lines.append(">" + rng.choice(["", " "]) + f"r{q}" + rng.choice(["", " d e", "\tx"]))
        for _ in range(rng.randint(0 if corrupt else 1, 4)):
            lines.append("".join(rng.choice("ACGTNacgtn \t") for _ in range(rng.randint(0, 70))))
        if rng.random() < 0.2:
            lines.append("")
    text = rng.choice(["\n", "\r\n"]).join(lines) + rng.choice(["", "\n"])
    if corrupt and text:
        k = rng.randrange(len(text))
        text = text[:k] + rng.choice("X>#\n>z") + text[k:]
    return text


def test_fasta_fuzz_against_live_reference():
    R = ref()
    rng = random.Random(20231)
    for it in range(400):
        text = random_fasta(rng, rng.randint(0, 6), corrupt=it % 2 == 1)
        assert ours_fasta(text, "ACGTN") == ref_fasta(R, text, "ACGTN"), repr(text)


def test_task_list_fuzz_against_live_reference():
    R = ref()
    rng = random.Random(20232)
    toks = ["0", "1", "7", "-1", "+2", "x", "1.5", "99999999999999999999", "#", "%", "3", "12"]
    for it in range(400):
        rows = []
        for _ in range(rng.randint(0, 6)):
            rows.append(" ".join(rng.choice(toks) for _ in range(rng.choice([2, 4, 4, 4, 3, 5]))))
        seeds = "\n".join(rows) + rng.choice(["", "\n"])
        assert ours_tasks(seeds, False) == ref_tasks(R, seeds, False), repr(seeds)
        banner = rng.choice(["%%MatrixMarket matrix coordinate integer general",
                             "%%MatrixMarket matrix coordinate pattern general",
                             "%%MatrixMarket matrix coordinate real general"])
        ov = "\n".join([banner, rng.choice(["", "%c"]), f"{rng.randint(1, 9)} {rng.randint(1, 9)} {len(rows)}"]
                       + rows)
        assert ours_tasks(ov, True) == ref_tasks(R, ov, True), repr(ov)


def big_fasta(n_rec, seed):
    rng = np.random.default_rng(seed)
    lens = rng.integers(1, 5000, n_rec)
    sym = rng.choice(np.frombuffer(b"ACGTacgtN", dtype=np.uint8), int(lens.sum()))
    out, pos = [], 0
    for q, L in enumerate(lens):
        s = sym[pos:pos + L].tobytes().decode()
        pos += L
        out.append(f">read{q} len={L}\n" + "\n".join(s[i:i + 80] for i in range(0, len(s), 80)))
    return "\n".join(out) + "\n"


def test_fasta_threads_match_sequential_and_reference():
    """Chunked parsing (cuts at "\\n>") equals one thread and the reference,
    including errors placed at chunk boundaries."""
    text = big_fasta(6000, 3)  # ~15 MB: several 4 MB chunks
    one = ours_fasta(text, "ACGTN", threads=1)
    many = ours_fasta(text, "ACGTN", threads=16)
    assert one == many and one[0] != "error"
    if os.path.exists(REF_SO):
        assert ref_fasta(ref(), text, "ACGTN") == one
    cut = text.find("\n>", len(text) // 4)
    for bad in (text[:cut + 1] + ">empty\n" + text[cut + 1:],          # empty record at a cut
                text[:cut] + "X" + text[cut:],                           # invalid symbol before a cut
                text[:len(text) // 2] + "\n\n" + text[len(text) // 2:].replace(">", "!", 1)):
        e1 = ours_fasta(bad, "ACGTN", threads=1)
        e16 = ours_fasta(bad, "ACGTN", threads=16)
        assert e1 == e16 and e1[0] == "error"
        if os.path.exists(REF_SO):
            assert ref_fasta(ref(), bad, "ACGTN") == e1


def test_pool_from_fasta_equals_pool_from_buffers():
    text = ">a\nACGTACGT\n>b\nacgtnn\n"
    s = xb.ScoringScheme.match_mismatch(1, -1, -1, 5)
    p = xb.DevicePool.from_fasta(text, s)
    assert p.n == 2 and p.bits_per_symbol == 5  # N present: 5-bit codes
    p2 = xb.DevicePool.from_fasta(">a\nACGT\n", s)
    assert p2.bits_per_symbol == 2

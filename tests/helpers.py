"""Shared test helpers: loading golden vectors and comparing result records."""
from __future__ import annotations

import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_json(name: str):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def blosum62():
    m = load_json("blosum62.json")
    return m["alphabet"], m["cells"]


def expect_tuple(e: dict):
    """Comparable tuple of a golden result record."""
    if e["status"]:
        return ("band", e["spread"], e["cells"])
    return (e["score"], e["h_ext"], e["v_ext"], e["cells"], e["delta_w"])


def rec_tuple(r) -> tuple:
    """Same tuple from a ctypes result or a structured numpy row."""
    get = (lambda k: int(r[k])) if isinstance(r, (np.void, np.ndarray)) else (lambda k: int(getattr(r, k)))
    if get("status"):
        return ("band", get("spread"), get("cells"))
    return (get("score"), get("h_ext"), get("v_ext"), get("cells"), get("delta_w"))


def result_rows_equal(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Per-row equality of two RESULT_DTYPE arrays (all fields that the
    reference defines for the row's status)."""
    ok = a["status"] == b["status"]
    good = a["status"] == 0
    for f in ("score", "h_ext", "v_ext", "delta_w"):
        ok &= np.where(good, a[f] == b[f], True)
    ok &= a["cells"] == b["cells"]
    ok &= np.where(good, True, a["spread"] == b["spread"])
    return ok


def oracle_scheme(oracle, spec, alphabet=None, cells=None):
    if spec[0] == "BLOSUM62":
        a, c = blosum62()
        return oracle.scheme_matrix(a, c, spec[1], spec[2])
    return oracle.scheme_mm(*spec)

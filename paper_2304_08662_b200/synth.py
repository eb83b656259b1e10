"""The five BASELINE.json configs as deterministic synthetic inputs (C++ generator,
csrc/xb_synth.cpp).  Returns the pool as (symbols uint8, offsets int64) plus
tasks (n, 4) int64 = (h_id, v_id, h_seed, v_seed)."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import blosum62
from .capi import check, lib


def blosum62_text() -> str:
    """NCBI-format BLOSUM62 text (the package constant, blosum62.py)."""
    return blosum62.text()


@dataclass
class Dataset:
    cfg: int
    symbols: np.ndarray
    offsets: np.ndarray
    tasks: np.ndarray
    k: int
    x: int
    band: int

    @property
    def n_tasks(self) -> int:
        return len(self.tasks)

    def seq(self, i: int) -> bytes:
        return self.symbols[self.offsets[i]:self.offsets[i + 1]].tobytes()

    def paper_products(self) -> float:
        """sum over tasks of |H| * |V| (pipeline.cpp:156-162)."""
        ln = np.diff(self.offsets).astype(np.float64)
        return float(np.sum(ln[self.tasks[:, 0]] * ln[self.tasks[:, 1]]))


def make(cfg: int, scale: float = 1.0, seed: int = 0, threads: int = 0) -> Dataset:
    L = lib()
    err = C.c_int(0)
    mtext = blosum62_text().encode() if cfg == 3 else None
    h = L.xb_synth_make(cfg, scale, seed, mtext, threads, C.byref(err))
    check(err.value, "xb_synth_make")
    try:
        z = (C.c_int64 * 6)()
        L.xb_synth_sizes(h, z)
        n_seqs, total, n_tasks, k, x, band = (int(v) for v in z)
        sym = np.empty(total, dtype=np.uint8)
        off = np.empty(n_seqs + 1, dtype=np.int64)
        tasks = np.empty((n_tasks, 4), dtype=np.int64)
        L.xb_synth_copy(h, sym.ctypes.data, off.ctypes.data, tasks.ctypes.data)
    finally:
        L.xb_synth_free(h)
    return Dataset(cfg, sym, off, tasks, k, x, band)


def pairs(n_pairs: int, length: int, p_match: float, k: int = 17, seed: int = 42,
          uniform_seed: bool = False):
    """The reference's generate_synthetic (proj/src/io.cpp:198-255) through the
    C ABI: (symbols uint8, offsets int64, tasks (n, 4) int64), byte-identical
    to the reference for the same SynthParams."""
    L = lib()
    err = C.c_int(0)
    h = L.xb_synth_pairs(n_pairs, length, p_match, k, int(uniform_seed), seed, C.byref(err))
    from .xband import _raise  # the reference's InputError for k < 1 or k > length
    _raise(err.value, "generate_synthetic")
    try:
        z = (C.c_int64 * 6)()
        L.xb_synth_sizes(h, z)
        n_seqs, total, n_tasks = int(z[0]), int(z[1]), int(z[2])
        sym = np.empty(total, dtype=np.uint8)
        off = np.empty(n_seqs + 1, dtype=np.int64)
        tasks = np.empty((n_tasks, 4), dtype=np.int64)
        L.xb_synth_copy(h, sym.ctypes.data, off.ctypes.data, tasks.ctypes.data)
    finally:
        L.xb_synth_free(h)
    return sym, off, tasks

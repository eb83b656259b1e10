"""Host-side mirror of the reference xband C++ API, running on the sm_100a engine.

Same names, argument meaning and error behaviour as the reference
(proj/include/xband/*.hpp) so callers and tests read like the reference's
own, e.g. proj/tests/test_align.cpp:

    s = ScoringScheme.match_mismatch(1, -1, -1, 3)
    a = Sequence(0, "s", "ACGT")
    r = xdrop_extend(full(a), full(a), s, 16)        # -> ExtensionResult(4, 4, 4, 23, 4)

Every extension goes through the C-ABI (include/xdrop_b200.h) to the CUDA
kernels; there is no CPU fallback.  Batches use ``extend_batch`` (the
pipeline loop, proj/src/pipeline.cpp:103-136) or ``extend_tasks`` for numpy
inputs.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from enum import IntEnum

import numpy as np

from . import capi
from .capi import RESULT_DTYPE, TASK_DTYPE, UNIT_DTYPE, XbError, check, lib

Score = int


# ---------------------------------------------------------------- errors ----
# proj/include/xband/errors.hpp:14-93

class InputError(RuntimeError):
    pass


class InternalError(RuntimeError):
    pass


class UnknownSymbol(InputError):
    def __init__(self, symbol: str = "?"):
        super().__init__(f"symbol not in scoring alphabet: '{symbol}'")
        self.symbol = symbol


class OutOfRange(InputError):
    pass


class SeedOutOfBounds(InputError):
    pass


class DanglingReference(InputError):
    pass


class NonSquare(InputError):
    pass


class DeviceError(InternalError):
    pass


# parser errors (errors.hpp:54-82), each naming the offending line where the
# reference does
class MissingHeader(InputError):
    pass


class EmptyRecord(InputError):
    pass


class InvalidSymbol(InputError):
    def __init__(self, line: int, msg: str):
        super().__init__(msg)
        self.line = line


class MalformedLine(InputError):
    def __init__(self, line: int, msg: str):
        super().__init__(msg)
        self.line = line


class NegativeIndex(InputError):
    pass


class BadHeader(InputError):
    pass


class IndexOutOfDeclaredShape(InputError):
    pass


def _raise_parse(e) -> None:
    msg = e.message.decode()
    if e.kind == 1:
        raise MissingHeader(msg)
    if e.kind == 2:
        raise EmptyRecord(msg)
    if e.kind == 3:
        raise InvalidSymbol(int(e.line), msg)
    if e.kind == 4:
        raise MalformedLine(int(e.line), msg)
    if e.kind == 5:
        raise NegativeIndex(msg)
    if e.kind == 6:
        raise BadHeader(msg)
    if e.kind == 7:
        raise IndexOutOfDeclaredShape(msg)
    raise InputError(msg or "invalid argument")


class BandExceededError(RuntimeError):
    """Retry signal (errors.hpp:80-93): the live spread outgrew the band."""

    def __init__(self, spread: int, cells: int, side: str = "?"):
        super().__init__(f"antidiagonal spread {spread} exceeds allocated band")
        self.observed_spread = spread
        self.cells = cells
        self.side = side


def _raise(code: int, what: str, index=None):
    if code == capi.XB_OK:
        return
    if code == capi.XB_E_DANGLING:
        raise DanglingReference(f"{what}: task {index} references an unknown sequence")
    if code == capi.XB_E_SEED_OOB:
        raise SeedOutOfBounds(f"{what}: seed of task {index} does not fit inside its sequences")
    if code == capi.XB_E_UNKNOWN_SYMBOL:
        raise UnknownSymbol()
    if code == capi.XB_E_OUT_OF_RANGE:
        raise OutOfRange(f"{what}: view out of range")
    if code in (capi.XB_E_BAD_PARAM, capi.XB_E_PARSE):
        raise InputError(f"{what}: {lib().xb_strerror(code).decode()}")
    raise DeviceError(f"{what}: {lib().xb_strerror(code).decode()} (code {code})")


# --------------------------------------------------------------- scoring ----
# proj/include/xband/scoring.hpp:13-56

@dataclass
class SubMatrix:
    alphabet: str
    cells: list

    def at(self, a: str, b: str) -> int:
        ia, ib = self.alphabet.find(a), self.alphabet.find(b)
        if ia < 0:
            raise UnknownSymbol(a)
        if ib < 0:
            raise UnknownSymbol(b)
        return self.cells[ia * len(self.alphabet) + ib]


def parse_submatrix(text: str) -> SubMatrix:
    """NCBI-format matrix (scoring.cpp:61-105)."""
    alpha = C.create_string_buffer(64)
    cells = (C.c_int * (64 * 64))()
    n = lib().xb_parse_submatrix(text.encode(), alpha, 64, cells, 64 * 64)
    if n < 0:
        raise NonSquare("malformed substitution matrix") if -n == capi.XB_E_PARSE else InputError(
            "substitution matrix too large")
    return SubMatrix(alpha.value.decode(), [cells[i] for i in range(n * n)])


class ScoringScheme:
    """Pairwise similarity + gap/x-drop parameters (scoring.hpp:28-54)."""

    def __init__(self, handle, gap: int, x: int, desc):
        self._h = handle
        self.gap = gap
        self.x = x
        self.desc = desc

    @staticmethod
    def match_mismatch(match: int, mismatch: int, gap: int, x: int) -> "ScoringScheme":
        err = C.c_int(0)
        h = lib().xb_scheme_match_mismatch(match, mismatch, gap, x, C.byref(err))
        if not h:
            raise InputError("invalid match/mismatch/gap/x")
        return ScoringScheme(h, gap, x, ("mm", match, mismatch, gap, x))

    @staticmethod
    def from_matrix(m: SubMatrix, gap: int, x: int) -> "ScoringScheme":
        n = len(m.alphabet)
        arr = (C.c_int * (n * n))(*m.cells)
        err = C.c_int(0)
        h = lib().xb_scheme_from_matrix(m.alphabet.encode(), n, arr, gap, x, C.byref(err))
        if not h:
            raise InputError("invalid matrix scheme")
        return ScoringScheme(h, gap, x, ("mx", m.alphabet, tuple(m.cells), gap, x))

    def sim(self, a: str, b: str) -> int:
        out = C.c_int(0)
        if lib().xb_scheme_sim(self._h, a.encode(), b.encode(), C.byref(out)) != 0:
            raise UnknownSymbol(a)
        return out.value

    def __del__(self):
        try:
            if self._h:
                lib().xb_scheme_free(self._h)
        except Exception:
            pass


def sim(scheme: ScoringScheme, a: str, b: str) -> int:
    """Checked similarity (scoring.cpp:55-59)."""
    return scheme.sim(a, b)


# ------------------------------------------------------- pool and views ----
# proj/include/xband/sequence.hpp:13-45

class Dir(IntEnum):
    Left = 0
    Right = 1


@dataclass
class Sequence:
    id: int
    name: str
    symbols: str


class SequenceStore(list):
    """Detached sequence pool: list of Sequence with dense ids."""


@dataclass
class SeqView:
    seq: Sequence
    origin: int
    dir: Dir
    length: int

    def at(self, i: int) -> str:
        return self.seq.symbols[self.origin + i] if self.dir == Dir.Right else \
            self.seq.symbols[self.origin - 1 - i]


def make_view(s: Sequence, origin: int, dir: Dir, length: int) -> SeqView:
    if origin > len(s.symbols):
        raise OutOfRange(f"view origin {origin} past end of sequence {s.id}")
    room = len(s.symbols) - origin if dir == Dir.Right else origin
    if length > room:
        raise OutOfRange(f"view length {length} exceeds the {room} symbols available")
    return SeqView(s, origin, dir, length)


def full(s: Sequence) -> SeqView:
    return make_view(s, 0, Dir.Right, len(s.symbols))


class DevicePool:
    """A packed, device-resident copy of sequences for one scheme (xb_pool)."""

    def __init__(self, scheme: ScoringScheme, symbols: np.ndarray | bytes,
                 offsets: np.ndarray):
        err = C.c_int(0)
        self.scheme = scheme
        self._h = lib().xb_pool_create(scheme._h, C.byref(err))
        check(err.value, "xb_pool_create")
        sym = np.frombuffer(symbols, dtype=np.uint8) if isinstance(symbols, (bytes, bytearray)) \
            else np.ascontiguousarray(symbols).view(np.uint8)
        off = np.ascontiguousarray(offsets, dtype=np.int64)
        n = len(off) - 1
        if n > 0:
            r = lib().xb_pool_add_bulk(self._h, sym.ctypes.data, off.ctypes.data, n)
            if r < 0:
                _raise(int(-r), "xb_pool_add_bulk")
        self.n = n

    @staticmethod
    def from_fasta(text_or_records, scheme: ScoringScheme, allowed: str = "ACGTN") -> "DevicePool":
        """FASTA text (or FastaRecords) straight into a packed pool: records in
        file order are sequence ids 0..n-1 (parse_fasta + SequenceStore)."""
        rec = text_or_records if isinstance(text_or_records, FastaRecords) else \
            FastaRecords(text_or_records, allowed)
        p = DevicePool(scheme, b"", np.zeros(1, dtype=np.int64))
        r = lib().xb_pool_add_fasta(p._h, rec._h)
        if r < 0:
            _raise(int(-r), "xb_pool_add_fasta")
        p.n = len(rec)
        return p

    @staticmethod
    def from_store(store, scheme: ScoringScheme) -> "DevicePool":
        data = b"".join(s.symbols.encode() for s in store)
        off = np.zeros(len(store) + 1, dtype=np.int64)
        np.cumsum([len(s.symbols) for s in store], out=off[1:])
        return DevicePool(scheme, data, off)

    def add(self, symbols: bytes | str) -> int:
        """Appends one sequence (SequenceStore push_back); returns its id.
        A pool may grow after it was uploaded: the next batch re-uploads it."""
        b = symbols.encode() if isinstance(symbols, str) else bytes(symbols)
        buf = C.create_string_buffer(b, len(b) + 1)
        r = lib().xb_pool_add(self._h, buf, len(b))
        if r < 0:
            _raise(int(-r), "xb_pool_add")
        self.n += 1
        return int(r)

    @property
    def bits_per_symbol(self) -> int:
        return lib().xb_pool_bits_per_symbol(self._h)

    def evict(self):
        lib().xb_pool_evict(self._h)

    def __del__(self):
        try:
            if self._h:
                lib().xb_pool_free(self._h)
        except Exception:
            pass


# -------------------------------------------------------- result types ----
# proj/include/xband/align.hpp:16-51

@dataclass
class ExtensionTask:
    task_id: int = 0
    h_id: int = 0
    v_id: int = 0
    h_seed: int = 0
    v_seed: int = 0


@dataclass(frozen=True)
class ExtensionResult:
    score: int = 0
    h_ext: int = 0
    v_ext: int = 0
    cells: int = 0
    delta_w: int = 0


@dataclass
class SeedAlignment:
    task_id: int = 0
    left: ExtensionResult = field(default_factory=ExtensionResult)
    right: ExtensionResult = field(default_factory=ExtensionResult)
    seed_score: int = 0
    total: int = 0


@dataclass
class FailedUnit:
    task_id: int
    side: str
    observed_spread: int


def _result(r) -> ExtensionResult:
    return ExtensionResult(int(r["score"]), int(r["h_ext"]), int(r["v_ext"]), int(r["cells"]),
                           int(r["delta_w"]))


# ------------------------------------------------------------- kernels ----

def _store_of(*views):
    """Pool the sequences behind a set of views (dedup by object identity)."""
    seqs, index = [], {}
    for v in views:
        if id(v.seq) not in index:
            index[id(v.seq)] = len(seqs)
            seqs.append(v.seq)
    return seqs, index


def xdrop_extend(h: SeqView, v: SeqView, scheme: ScoringScheme, band: int,
                 scratch=None, exec_flags: int = 0) -> ExtensionResult:
    """X-drop extension of v against h (align.hpp:53-59, align.cpp:165-177).

    Raises BandExceededError when the live spread outgrows ``band``.  The
    ``scratch`` argument of the reference has no device analogue; a
    BandBuffers whose width differs from ``band`` raises InputError as in the
    reference (align.cpp:168-172)."""
    if scratch is not None and getattr(scratch, "width", band) != band:
        raise InputError(f"scratch buffers sized for band {scratch.width}, kernel asked for {band}")
    if band < 1:
        raise InputError("band width must be at least 1")
    seqs, index = _store_of(h, v)
    pool = DevicePool.from_store(seqs, scheme)
    u = np.zeros(1, dtype=UNIT_DTYPE)
    u["h_id"], u["v_id"] = index[id(h.seq)], index[id(v.seq)]
    u["h_dir"], u["v_dir"] = int(h.dir), int(v.dir)
    u["h_origin"], u["v_origin"] = h.origin, v.origin
    u["h_len"], u["v_len"] = h.length, v.length
    out = extend_units(pool, u, band, exec_flags=exec_flags)
    r = out[0]
    if r["status"] == capi.XB_SIDE_BAND_EXCEEDED:
        raise BandExceededError(int(r["spread"]), int(r["cells"]))
    return _result(r)


class BandBuffers:
    """Reference storage object (align.hpp:26-34).  The engine keeps the band
    in registers / device scratch; this only mirrors the reference contract
    (two rows of exactly ``width`` cells, width >= 1)."""

    def __init__(self, delta_b: int):
        if delta_b < 1:
            raise InputError("band width must be at least 1")
        self.width = delta_b
        self.rows = (np.zeros(delta_b, np.int32), np.zeros(delta_b, np.int32))
        self.lower = self.upper = 0

    def cell_capacity(self) -> int:
        return 2 * self.width


def extend_units(pool: DevicePool, units: np.ndarray, band: int, exec_flags: int = 0,
                 n_devices: int = 1, device_ids=None) -> np.ndarray:
    """One xdrop_extend per row of ``units`` (UNIT_DTYPE) -> RESULT_DTYPE rows."""
    units = np.ascontiguousarray(units, dtype=UNIT_DTYPE)
    out = np.zeros(len(units), dtype=RESULT_DTYPE)
    bad = C.c_int64(-1)
    ex = capi.make_exec(n_devices, device_ids, None, exec_flags)
    rc = lib().xb_extend_units(pool._h, units.ctypes.data, len(units), band, out.ctypes.data,
                               C.byref(bad), C.byref(ex))
    _raise(rc, "xb_extend_units", bad.value)
    return out


def tasks_array(tasks) -> np.ndarray:
    """ExtensionTask list or an (n, 4) int array -> TASK_DTYPE."""
    if isinstance(tasks, np.ndarray) and tasks.dtype == TASK_DTYPE:
        return tasks
    if isinstance(tasks, np.ndarray):
        t = np.asarray(tasks, dtype=np.int64).reshape(-1, 4)
        out = np.zeros(len(t), dtype=TASK_DTYPE)
        out["task_id"] = np.arange(len(t))
        out["h_id"], out["v_id"], out["h_seed"], out["v_seed"] = t[:, 0], t[:, 1], t[:, 2], t[:, 3]
        return out
    out = np.zeros(len(tasks), dtype=TASK_DTYPE)
    for q, t in enumerate(tasks):
        out[q] = (t.task_id, t.h_id, t.v_id, 0, t.h_seed, t.v_seed)
    return out


def extend_tasks(pool: DevicePool, tasks, k: int, band: int, exec_flags: int = 0,
                 n_devices: int = 1, device_ids=None, stream=None):
    """The batch C-ABI: returns (results[2n] RESULT_DTYPE, seed_score[n])."""
    t = tasks_array(tasks)
    out = np.zeros(2 * len(t), dtype=RESULT_DTYPE)
    ss = np.zeros(len(t), dtype=np.int32)
    bad = C.c_int64(-1)
    ex = capi.make_exec(n_devices, device_ids, stream, exec_flags)
    rc = lib().xb_extend_batch(pool._h, t.ctypes.data, len(t), k, band, out.ctypes.data,
                               ss.ctypes.data, C.byref(bad), C.byref(ex))
    _raise(rc, "xb_extend_batch", bad.value)
    return out, ss


def shard_tasks(pool: DevicePool, tasks, k: int, n_shards: int, locality: bool = False) -> np.ndarray:
    """xb_shard_tasks: shard index (int32) of every task, one shard per GPU.
    LPT on estimated cost, or locality-aware (a breadth-first sweep of the
    sequence graph cut into equal-cost runs, so a shard references a compact
    part of the pool, which is all its device uploads)."""
    t = tasks_array(tasks)
    out = np.zeros(len(t), dtype=np.int32)
    bad = C.c_int64(-1)
    rc = lib().xb_shard_tasks(pool._h, t.ctypes.data, len(t), k, n_shards,
                              capi.XB_SHARD_LOCALITY if locality else capi.XB_SHARD_LPT,
                              out.ctypes.data, C.byref(bad))
    _raise(rc, "xb_shard_tasks", bad.value)
    return out


def extend_batches(batches, k: int, band: int, exec_flags: int = 0, n_devices: int = 1,
                   device_ids=None, reupload: bool = False, stats: list | None = None):
    """A stream of batches through the device-resident batch C-ABI
    (xb_batch_create / run / fetch), one batch in flight ahead of the host:
    batch i+1's uploads (pool if not resident, tasks) and planning overlap
    batch i's kernels, and batch i's rows are copied out while batch i+1
    runs.  `batches` yields (DevicePool, tasks); yields (results[2n],
    seed_score[n]) per batch, in order.  reupload=True drops each batch's
    device pool copy before its upload (xb_pool_evict), so every batch's
    inputs cross PCIe -- consecutive batches must then use distinct pools,
    since batch i may still read its pool while batch i+1 uploads.  `stats`,
    if given, receives each batch's xb_stats dict."""
    L = lib()
    ex = capi.make_exec(n_devices, device_ids, None, exec_flags)
    prev = None  # (handle, pool, results, seeds)

    def finish(p):
        h, _, out, ss = p
        try:
            _raise(L.xb_batch_fetch(h, out.ctypes.data, ss.ctypes.data), "xb_batch_fetch")
            if stats is not None:
                st = capi.XbStats()
                _raise(L.xb_batch_stats(h, C.byref(st)), "xb_batch_stats")
                stats.append(st.as_dict())
        finally:
            L.xb_batch_free(h)
        return out, ss

    try:
        for pool, tasks in batches:
            if reupload:
                if prev is not None and prev[1] is pool:
                    raise ValueError("reupload: consecutive batches need distinct pools")
                pool.evict()
            t = tasks_array(tasks)
            err, bad = C.c_int(0), C.c_int64(-1)
            h = L.xb_batch_create(pool._h, t.ctypes.data, len(t), k, band, C.byref(ex),
                                  C.byref(bad), C.byref(err))
            _raise(err.value, "xb_batch_create", bad.value)
            cur = (h, pool, np.zeros(2 * len(t), dtype=RESULT_DTYPE), np.zeros(len(t), dtype=np.int32))
            rc = L.xb_batch_run(h)
            if rc:
                L.xb_batch_free(h)
                _raise(rc, "xb_batch_run")
            if prev is not None:
                p, prev = prev, None
                yield finish(p)
            prev = cur
        if prev is not None:
            p, prev = prev, None
            yield finish(p)
    finally:
        if prev is not None:
            L.xb_batch_free(prev[0])


# ---------------------------------------------------------------- ingest ----
# proj/src/io.cpp:58-196, native (csrc/xb_ingest.cpp)

def _text(t) -> bytes:
    return t.encode() if isinstance(t, str) else bytes(t)


class FastaRecords:
    """parse_fasta output as contiguous buffers: symbols (uint8), offsets,
    names; `handle` can feed a DevicePool without another copy."""

    def __init__(self, text, allowed: str = "ACGTN", threads: int = 0):
        b = _text(text)
        err = capi.XbParseError()
        self._h = lib().xb_fasta_parse(b, len(b), allowed.encode(), threads, C.byref(err))
        if not self._h:
            _raise_parse(err)
        z = (C.c_int64 * 3)()
        lib().xb_fasta_sizes(self._h, z)
        n, ns, nb = int(z[0]), int(z[1]), int(z[2])
        self.symbols = np.empty(ns, dtype=np.uint8)
        self.offsets = np.empty(n + 1, dtype=np.int64)
        names = np.empty(nb, dtype=np.uint8)
        noff = np.empty(n + 1, dtype=np.int64)
        lib().xb_fasta_copy(self._h, self.symbols.ctypes.data, self.offsets.ctypes.data,
                            names.ctypes.data, noff.ctypes.data)
        nbytes = names.tobytes()
        self.names = [nbytes[noff[i]:noff[i + 1]].decode() for i in range(n)]

    def __len__(self):
        return len(self.names)

    def __del__(self):
        try:
            if self._h:
                lib().xb_fasta_free(self._h)
        except Exception:
            pass


def parse_fasta(text, allowed: str = "ACGTN") -> SequenceStore:
    """parse_fasta (io.cpp:58-96): records with upper-cased symbols checked
    against `allowed`; MissingHeader / EmptyRecord / InvalidSymbol as there."""
    r = FastaRecords(text, allowed)
    st = SequenceStore()
    sym = r.symbols.tobytes()
    for i, name in enumerate(r.names):
        st.append(Sequence(i, name, sym[r.offsets[i]:r.offsets[i + 1]].decode()))
    return st


def _parse_tasks(fn, text) -> np.ndarray:
    b = _text(text)
    err = capi.XbParseError()
    n = fn(b, len(b), None, 0, C.byref(err))
    if n < 0:
        _raise_parse(err)
    out = np.zeros(int(n), dtype=TASK_DTYPE)
    if n:
        fn(b, len(b), out.ctypes.data, int(n), C.byref(err))
    return out


def parse_seeds(text) -> np.ndarray:
    """parse_seeds (io.cpp:98-127): TASK_DTYPE rows in input order."""
    return _parse_tasks(lib().xb_parse_seeds, text)


def parse_overlaps(text) -> np.ndarray:
    """parse_overlaps (io.cpp:129-196): Matrix Market coordinate overlaps."""
    return _parse_tasks(lib().xb_parse_overlaps, text)


def sweep_band(length: int, xs, p_grid, rng_seed: int = 42, n_devices: int = 1,
               device_ids=None) -> str:
    """The band survey of proj/src/pipeline.cpp:181-208 (declared at
    pipeline.hpp:58): for every X and p, one synthetic pair of `length`
    (generate_synthetic, centred 17-mer seed) extended over the full views
    with band length + 1; returns the reference's TSV byte for byte."""
    xa = np.ascontiguousarray(list(xs), dtype=np.int32)
    pa = np.ascontiguousarray(list(p_grid), dtype=np.float64)
    dw = np.zeros(len(xa) * len(pa), dtype=np.int32)
    ex = capi.make_exec(n_devices, device_ids, None, 0)
    rc = lib().xb_sweep_band(length, xa.ctypes.data, len(xa), pa.ctypes.data, len(pa), rng_seed,
                             dw.ctypes.data, C.byref(ex))
    _raise(rc, "xb_sweep_band", -1)
    rows = ["x\terror_rate\tdelta_w\n"]
    for a, x in enumerate(xa):
        for b, p in enumerate(pa):
            rows.append("%d\t%.2f\t%d\n" % (int(x), 1.0 - float(p), int(dw[a * len(pa) + b])))
    return "".join(rows)


def last_stats() -> dict:
    st = capi.XbStats()
    lib().xb_last_stats(C.byref(st))
    return st.as_dict()


def extend_seed(t: ExtensionTask, store: SequenceStore, k: int, scheme: ScoringScheme,
                band: int, scratch=None) -> SeedAlignment:
    """Seed extension in both directions (align.cpp:268-309); band failures
    are raised with the failing side attributed, left before right."""
    if scratch is not None and scratch.width != band:
        raise InputError(f"scratch buffers sized for band {scratch.width}, kernel asked for {band}")
    pool = DevicePool.from_store(store, scheme)
    out, ss = extend_tasks(pool, [t], k, band)
    for side, r in (("L", out[0]), ("R", out[1])):
        if r["status"] == capi.XB_SIDE_BAND_EXCEEDED:
            raise BandExceededError(int(r["spread"]), int(r["cells"]), side)
    a = SeedAlignment(t.task_id, _result(out[0]), _result(out[1]), int(ss[0]))
    a.total = a.left.score + a.seed_score + a.right.score
    return a


def extend_batch(store: SequenceStore, tasks, k: int, scheme: ScoringScheme, band: int):
    """Drop-in for the batch loop at pipeline.cpp:103-136: every task's two
    sides always run; a task is kept only if both succeed, else each failing
    side becomes a FailedUnit.  Returns (alignments in task order, failed,
    unit_cells {unit_id: cells})."""
    pool = DevicePool.from_store(store, scheme)
    out, ss = extend_tasks(pool, tasks, k, band)
    alignments, failed, unit_cells = [], [], {}
    for q, t in enumerate(tasks):
        ok = True
        for s, side in ((0, "L"), (1, "R")):
            r = out[2 * q + s]
            unit_cells[2 * t.task_id + s] = int(r["cells"])
            if r["status"] == capi.XB_SIDE_BAND_EXCEEDED:
                failed.append(FailedUnit(t.task_id, side, int(r["spread"])))
                ok = False
        if ok:
            a = SeedAlignment(t.task_id, _result(out[2 * q]), _result(out[2 * q + 1]), int(ss[q]))
            a.total = a.left.score + a.seed_score + a.right.score
            alignments.append(a)
    return alignments, failed, unit_cells


# ---------------------------------------------------- work decomposition ----
# proj/src/partition.cpp:45-81 (host-side mirror; the engine does the same
# split on the device)

@dataclass
class WorkUnit:
    unit_id: int
    task_id: int
    side: str
    h_id: int
    v_id: int
    h_origin: int
    v_origin: int
    h_len: int
    v_len: int
    est_cost: int


def estimate_cost(u: WorkUnit) -> int:
    return u.h_len * u.v_len


def split_lr(t: ExtensionTask, store: SequenceStore, k: int):
    if t.h_id >= len(store) or t.v_id >= len(store):
        raise DanglingReference(f"task {t.task_id} references an unknown sequence")
    hn, vn = len(store[t.h_id].symbols), len(store[t.v_id].symbols)
    if t.h_seed + k > hn or t.v_seed + k > vn:
        raise SeedOutOfBounds(f"seed of task {t.task_id} does not fit inside its sequences")
    l = WorkUnit(2 * t.task_id, t.task_id, "L", t.h_id, t.v_id, t.h_seed, t.v_seed, t.h_seed,
                 t.v_seed, 0)
    l.est_cost = estimate_cost(l)
    r = WorkUnit(2 * t.task_id + 1, t.task_id, "R", t.h_id, t.v_id, t.h_seed + k, t.v_seed + k,
                 hn - t.h_seed - k, vn - t.v_seed - k, 0)
    r.est_cost = estimate_cost(r)
    return l, r


def gcups(h_len: float, v_len: float, seconds: float) -> float:
    """Paper GCUPS for one h x v problem in t seconds (pipeline.cpp:51-54)."""
    if seconds <= 0:
        raise InputError("cannot rate work done in zero time")
    return h_len * v_len / seconds / 1e9

"""TEST INFRASTRUCTURE ONLY -- ctypes bindings for the CPU checkers.

* ``Oracle``: the C restatement (oracle/liboracle.so, xdrop_oracle.c).
* ``Ref``: the unmodified reference library (oracle/_ref/libxband_ref.so,
  built from /root/reference/proj/src by oracle/Makefile).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libxband_ref.so")

# xo_result / RefResult / xb_side_result layout
RESULT_DTYPE = np.dtype([("score", "<i4"), ("h_ext", "<i4"), ("v_ext", "<i4"),
                         ("delta_w", "<i4"), ("cells", "<i8"), ("status", "<i4"),
                         ("spread", "<i4")])


class XoScheme(C.Structure):
    _fields_ = [("table", C.c_int16 * (256 * 256)), ("valid", C.c_ubyte * 256),
                ("gap", C.c_int), ("x", C.c_int)]


class XoResult(C.Structure):
    _fields_ = [("score", C.c_int32), ("h_ext", C.c_int32), ("v_ext", C.c_int32),
                ("delta_w", C.c_int32), ("cells", C.c_int64), ("status", C.c_int32),
                ("spread", C.c_int32)]

    def tuple(self):
        return (self.score, self.h_ext, self.v_ext, self.cells, self.delta_w)


class XoView(C.Structure):
    _fields_ = [("origin", C.c_void_p), ("length", C.c_int64), ("dir", C.c_int32)]


def build(quiet: bool = True) -> None:
    """Compile liboracle.so (and oracle/_ref when the reference is present)."""
    import subprocess
    out = subprocess.DEVNULL if quiet else None
    subprocess.check_call(["make", "-s", "-C", HERE, "liboracle.so"], stdout=out)
    if os.path.isdir("/root/reference/proj/src"):
        subprocess.check_call(["make", "-s", "-C", HERE, "ref"], stdout=out)


def _buf(b: bytes):
    return C.create_string_buffer(b, len(b) + 1)


class Oracle:
    """The C restatement."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        self.lib = C.CDLL(path)
        L = self.lib
        L.xo_scheme_match_mismatch.argtypes = [C.POINTER(XoScheme), C.c_int, C.c_int, C.c_int, C.c_int]
        L.xo_scheme_from_matrix.argtypes = [C.POINTER(XoScheme), C.c_char_p, C.c_int,
                                            C.POINTER(C.c_int), C.c_int, C.c_int]
        L.xo_xdrop_extend.argtypes = [XoView, XoView, C.POINTER(XoScheme), C.c_int, C.POINTER(XoResult)]
        L.xo_full_oracle.argtypes = [XoView, XoView, C.POINTER(XoScheme), C.POINTER(XoResult)]
        L.xo_extend_batch.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                                      C.c_int, C.POINTER(XoScheme), C.c_int, C.c_void_p,
                                      C.c_void_p, C.POINTER(C.c_int64), C.c_int]

    def scheme_mm(self, match=1, mismatch=-1, gap=-1, x=15):
        s = XoScheme()
        if self.lib.xo_scheme_match_mismatch(C.byref(s), match, mismatch, gap, x) != 0:
            raise ValueError("invalid match/mismatch scheme")
        return s

    def scheme_matrix(self, alphabet: str, cells, gap=-1, x=20):
        s = XoScheme()
        n = len(alphabet)
        arr = (C.c_int * (n * n))(*[int(c) for c in np.asarray(cells).ravel()])
        if self.lib.xo_scheme_from_matrix(C.byref(s), alphabet.encode(), n, arr, gap, x) != 0:
            raise ValueError("invalid matrix scheme")
        return s

    def _views(self, h: bytes, h_origin, h_dir, h_len, v: bytes, v_origin, v_dir, v_len):
        hb, vb = _buf(h), _buf(v)
        hv = XoView(C.addressof(hb) + h_origin, h_len, h_dir)
        vv = XoView(C.addressof(vb) + v_origin, v_len, v_dir)
        return hb, vb, hv, vv

    def extend(self, h: bytes, v: bytes, scheme, band, h_origin=0, v_origin=0, h_dir=1,
               v_dir=1, h_len=None, v_len=None) -> XoResult:
        if h_len is None:
            h_len = len(h) - h_origin if h_dir else h_origin
        if v_len is None:
            v_len = len(v) - v_origin if v_dir else v_origin
        hb, vb, hv, vv = self._views(h, h_origin, h_dir, h_len, v, v_origin, v_dir, v_len)
        r = XoResult()
        if self.lib.xo_xdrop_extend(hv, vv, C.byref(scheme), band, C.byref(r)) != 0:
            raise ValueError("band must be at least 1")
        return r

    def full(self, h: bytes, v: bytes, scheme) -> XoResult:
        hb, vb, hv, vv = self._views(h, 0, 1, len(h), v, 0, 1, len(v))
        r = XoResult()
        self.lib.xo_full_oracle(hv, vv, C.byref(scheme), C.byref(r))
        return r

    def extend_batch(self, pool: np.ndarray, offsets: np.ndarray, tasks: np.ndarray, k: int,
                     scheme, band: int, threads: int = 1):
        """pool: uint8 concatenated symbols; offsets: int64 (n_seqs+1);
        tasks: int64 (n,4).  Returns (results[2n], seed_scores[n])."""
        pool = np.ascontiguousarray(pool, dtype=np.uint8)
        offsets = np.ascontiguousarray(offsets, dtype=np.int64)
        tasks = np.ascontiguousarray(tasks, dtype=np.int64).reshape(-1, 4)
        n = tasks.shape[0]
        out = np.zeros(2 * n, dtype=RESULT_DTYPE)
        ss = np.zeros(n, dtype=np.int32)
        bad = C.c_int64(-1)
        rc = self.lib.xo_extend_batch(pool.ctypes.data, offsets.ctypes.data, len(offsets) - 1,
                                      tasks.ctypes.data, n, k, C.byref(scheme), band,
                                      out.ctypes.data, ss.ctypes.data, C.byref(bad), threads)
        if rc != 0:
            raise ValueError(f"oracle batch error {rc} at task {bad.value}")
        return out, ss


class RefResult(XoResult):
    pass


class Ref:
    """The unmodified reference library (oracle/_ref/libxband_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.lib = C.CDLL(path)
        L = self.lib
        L.ref_scheme_mm.restype = C.c_void_p
        L.ref_scheme_mm.argtypes = [C.c_int] * 4
        L.ref_scheme_matrix.restype = C.c_void_p
        L.ref_scheme_matrix.argtypes = [C.c_char_p, C.c_int, C.c_int]
        L.ref_scheme_free.argtypes = [C.c_void_p]
        L.ref_parse_matrix.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.POINTER(C.c_int)]
        L.ref_xdrop_extend.argtypes = [C.c_char_p, C.c_int64, C.c_int64, C.c_int, C.c_int64,
                                       C.c_char_p, C.c_int64, C.c_int64, C.c_int, C.c_int64,
                                       C.c_void_p, C.c_int, C.POINTER(XoResult)]
        L.ref_full_oracle.argtypes = [C.c_char_p, C.c_int64, C.c_char_p, C.c_int64, C.c_void_p,
                                      C.POINTER(XoResult)]
        L.ref_extend_seed.argtypes = [C.c_char_p, C.c_int64, C.c_char_p, C.c_int64, C.c_int64,
                                      C.c_int64, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int,
                                      C.POINTER(XoResult), C.POINTER(XoResult),
                                      C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                      C.c_char_p, C.POINTER(C.c_int32)]
        L.ref_pool_create.restype = C.c_void_p
        L.ref_pool_create.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
        L.ref_pool_free.argtypes = [C.c_void_p]
        L.ref_extend_batch.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p,
                                       C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                                       C.POINTER(C.c_int64)]
        L.ref_pipeline_synth.restype = C.c_int64
        L.ref_pipeline_synth.argtypes = [C.c_int64, C.c_int64, C.c_double, C.c_int, C.c_int,
                                         C.c_int, C.c_uint64, C.c_int, C.c_char_p, C.c_int64,
                                         C.POINTER(C.c_int)]
        L.ref_generate_synthetic.restype = C.c_int64
        L.ref_generate_synthetic.argtypes = [C.c_int64, C.c_int64, C.c_double, C.c_int,
                                             C.c_uint64, C.c_int, C.c_void_p, C.c_void_p,
                                             C.c_void_p]

    def scheme_mm(self, match=1, mismatch=-1, gap=-1, x=15):
        p = self.lib.ref_scheme_mm(match, mismatch, gap, x)
        if not p:
            raise ValueError("reference rejected the scheme")
        return p

    def scheme_matrix(self, text: str, gap=-1, x=20):
        p = self.lib.ref_scheme_matrix(text.encode(), gap, x)
        if not p:
            raise ValueError("reference rejected the matrix")
        return p

    def parse_matrix(self, text: str):
        alpha = C.create_string_buffer(300)
        cells = (C.c_int * (256 * 256))()
        n = self.lib.ref_parse_matrix(text.encode(), alpha, 256 * 256, cells)
        if n < 0:
            raise ValueError("reference rejected the matrix")
        return alpha.value.decode(), np.array(cells[: n * n], dtype=np.int32).reshape(n, n)

    def extend(self, h: bytes, v: bytes, scheme, band, h_origin=0, v_origin=0, h_dir=1,
               v_dir=1, h_len=None, v_len=None):
        if h_len is None:
            h_len = len(h) - h_origin if h_dir else h_origin
        if v_len is None:
            v_len = len(v) - v_origin if v_dir else v_origin
        r = XoResult()
        rc = self.lib.ref_xdrop_extend(h, len(h), h_origin, h_dir, h_len, v, len(v), v_origin,
                                       v_dir, v_len, scheme, band, C.byref(r))
        if rc == 2:
            raise ValueError("reference input error")
        return r

    def full(self, h: bytes, v: bytes, scheme):
        r = XoResult()
        self.lib.ref_full_oracle(h, len(h), v, len(v), scheme, C.byref(r))
        return r

    def extend_seed(self, h: bytes, v: bytes, h_seed, v_seed, k, scheme, band, h_id=0, v_id=1):
        L, R = XoResult(), XoResult()
        ss, tot, sp = C.c_int32(), C.c_int32(), C.c_int32()
        side = C.create_string_buffer(2)
        rc = self.lib.ref_extend_seed(h, len(h), v, len(v), h_seed, v_seed, h_id, v_id, k, scheme,
                                      band, C.byref(L), C.byref(R), C.byref(ss), C.byref(tot),
                                      side, C.byref(sp))
        return rc, L, R, ss.value, tot.value, side.value.decode(errors="replace"), sp.value

    def pool(self, pool: np.ndarray, offsets: np.ndarray):
        pool = np.ascontiguousarray(pool, dtype=np.uint8)
        offsets = np.ascontiguousarray(offsets, dtype=np.int64)
        return self.lib.ref_pool_create(pool.ctypes.data, offsets.ctypes.data, len(offsets) - 1)

    def extend_batch(self, pool_handle, scheme, tasks: np.ndarray, k: int, band: int,
                     threads: int = 1, order: np.ndarray | None = None):
        tasks = np.ascontiguousarray(tasks, dtype=np.int64).reshape(-1, 4)
        n = tasks.shape[0]
        out = np.zeros(2 * n, dtype=RESULT_DTYPE)
        ss = np.zeros(n, dtype=np.int32)
        bad = C.c_int64(-1)
        optr = None
        if order is not None:
            order = np.ascontiguousarray(order, dtype=np.int64)
            optr = order.ctypes.data
        rc = self.lib.ref_extend_batch(pool_handle, scheme, tasks.ctypes.data, n, optr, k, band,
                                       threads, out.ctypes.data, ss.ctypes.data, C.byref(bad))
        if rc != 0:
            raise ValueError(f"reference batch error {rc} at task {bad.value}")
        return out, ss

    def pipeline_synth(self, pairs, length, p_match, x=15, band=1024, k=17, seed=42,
                       uniform_seed=False):
        cap = 1 << 24
        buf = C.create_string_buffer(cap)
        ec = C.c_int()
        n = self.lib.ref_pipeline_synth(pairs, length, p_match, x, band, k, seed,
                                        int(uniform_seed), buf, cap, C.byref(ec))
        return ec.value, buf.raw[:n].decode()

    def parse_fasta(self, text: bytes, allowed: str = "ACGTN"):
        """The reference's parse_fasta: (symbols bytes, offsets, names) or
        ("error", kind, line, message) with kind as XB_PARSE_*."""
        n = len(text)
        nrec = text.count(b">") + 2  # records <= headers
        sym = C.create_string_buffer(n + 1)
        off = np.zeros(nrec, dtype=np.int64)
        names = C.create_string_buffer(n + 1)
        noff = np.zeros(nrec, dtype=np.int64)
        kind, line, msg = C.c_int(0), C.c_int64(0), C.create_string_buffer(256)
        f = self.lib.ref_parse_fasta
        f.restype = C.c_int64
        f.argtypes = [C.c_char_p, C.c_int64, C.c_char_p] + [C.c_void_p] * 4 + [C.c_void_p] * 3
        r = f(text, n, allowed.encode(), sym, off.ctypes.data, names, noff.ctypes.data,
              C.byref(kind), C.byref(line), msg)
        if r < 0:
            return ("error", kind.value, line.value, msg.value.decode())
        r = int(r)
        raw = names.raw  # one copy (every .raw access copies the whole buffer)
        return (sym.raw[: off[r]], off[: r + 1].copy(),
                [raw[noff[i]:noff[i + 1]].decode() for i in range(r)])

    def parse_tasks(self, text: bytes, overlaps: bool):
        """The reference's parse_seeds / parse_overlaps: (n, 5) int64
        (task_id, h, v, h_seed, v_seed) or ("error", kind, line, message)."""
        cap = text.count(b"\n") + 2  # tasks <= lines
        tasks = np.zeros((cap, 5), dtype=np.int64)
        kind, line, msg = C.c_int(0), C.c_int64(0), C.create_string_buffer(256)
        f = self.lib.ref_parse_tasks
        f.restype = C.c_int64
        f.argtypes = [C.c_int, C.c_char_p, C.c_int64, C.c_void_p, C.c_int64] + [C.c_void_p] * 3
        r = f(int(overlaps), text, len(text), tasks.ctypes.data, cap, C.byref(kind), C.byref(line), msg)
        if r < 0:
            return ("error", kind.value, line.value, msg.value.decode())
        return tasks[: int(r)].copy()

    def sweep_band(self, length, xs, ps, seed=42) -> str:
        """The reference's band survey TSV (pipeline.cpp:181-208)."""
        xa = np.ascontiguousarray(xs, dtype=np.int32)
        pa = np.ascontiguousarray(ps, dtype=np.float64)
        f = self.lib.ref_sweep_band
        f.restype = C.c_int64
        f.argtypes = [C.c_int64, C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_uint64, C.c_void_p,
                      C.c_int64]
        n = f(length, xa.ctypes.data, len(xa), pa.ctypes.data, len(pa), seed, None, 0)
        buf = C.create_string_buffer(int(n) + 1)
        f(length, xa.ctypes.data, len(xa), pa.ctypes.data, len(pa), seed, buf, n)
        return buf.raw[:n].decode()

    def generate_synthetic(self, pairs, length, p_match, k=17, seed=42, uniform_seed=False):
        sym = np.zeros(2 * pairs * length + 1, dtype=np.uint8)
        off = np.zeros(2 * pairs + 1, dtype=np.int64)
        tasks = np.zeros((pairs, 4), dtype=np.int64)
        self.lib.ref_generate_synthetic(pairs, length, p_match, k, seed, int(uniform_seed),
                                        sym.ctypes.data, off.ctypes.data, tasks.ctypes.data)
        return sym[: off[-1]], off, tasks

"""ctypes binding of the C-ABI in include/xdrop_b200.h.

The shared library is built in-tree (``make lib`` or ``__graft_entry__.build()``)
at paper_2304_08662_b200/_lib/libxdrop_b200.so.  There is no Python or CPU
fallback for the extension path: if the library or a CUDA device is missing,
the calls fail loudly (XB_E_NO_DEVICE / ImportError).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("XB_LIB_PATH") or os.path.join(HERE, "_lib", "libxdrop_b200.so")

XB_OK = 0
XB_E_BAD_PARAM = 1
XB_E_DANGLING = 2
XB_E_SEED_OOB = 3
XB_E_UNKNOWN_SYMBOL = 4
XB_E_OUT_OF_RANGE = 5
XB_E_CUDA = 6
XB_E_NO_DEVICE = 7
XB_E_PARSE = 8

XB_SIDE_OK = 0
XB_SIDE_BAND_EXCEEDED = 1

XB_FLAG_NO_SORT = 1
XB_FLAG_GENERIC_ONLY = 2
XB_FLAG_FORCE_TIER = 8
XB_FLAG_ESC_TO_WARP = 16
XB_FLAG_GROUP = 32
XB_FLAG_NO_GROUP = 64
XB_FLAG_THROUGHPUT = 128
XB_FLAG_SERIAL_TAIL = 4096
XB_FLAG_LOCALITY = 8192
XB_FLAG_LANES = 16384
XB_FLAG_NO_LANES = 32768

XB_SHARD_LPT = 0
XB_SHARD_LOCALITY = 1


def force_tier(t: int) -> int:
    return XB_FLAG_FORCE_TIER | (t << 8)

# numpy views of the C structs
TASK_DTYPE = np.dtype([("task_id", "<i4"), ("h_id", "<u4"), ("v_id", "<u4"), ("pad", "<u4"),
                       ("h_seed", "<u8"), ("v_seed", "<u8")])
RESULT_DTYPE = np.dtype([("score", "<i4"), ("h_ext", "<i4"), ("v_ext", "<i4"),
                         ("delta_w", "<i4"), ("cells", "<i8"), ("status", "<i4"),
                         ("spread", "<i4")])
UNIT_DTYPE = np.dtype([("h_id", "<u4"), ("v_id", "<u4"), ("h_dir", "<i4"), ("v_dir", "<i4"),
                       ("h_origin", "<u8"), ("v_origin", "<u8"), ("h_len", "<u8"),
                       ("v_len", "<u8")])
assert TASK_DTYPE.itemsize == 32 and RESULT_DTYPE.itemsize == 32 and UNIT_DTYPE.itemsize == 48


class XbExec(C.Structure):
    _fields_ = [("n_devices", C.c_int32), ("device_ids", C.POINTER(C.c_int32)),
                ("stream", C.c_void_p), ("flags", C.c_int32)]


# tiers 0-4: thread / lane-group register bands; 5-9: wide (8-32 lanes per unit); 10: warp tier
TIER_WIDTHS = [16, 24, 32, 48, 64, 96, 128, 256, 512, 1024]
TIER_NAMES = [f"thread_k{w}" for w in TIER_WIDTHS[:5]] + [f"wide_k{w}" for w in TIER_WIDTHS[5:]] + ["warp"]
NUM_TIERS = len(TIER_NAMES)
WIDE_FIRST = 5
WARP_TIER = NUM_TIERS - 1


def tier_kernel_name(t: int, stats: dict, flags: int = 0) -> str:
    """Kernel that served tier t in a run: the start tier runs one thread per
    unit unless the batch was latency-bound (lane groups); wider tiers take
    their escalations on lane groups (xb_engine.cu, run_cascade)."""
    if t >= len(TIER_WIDTHS):
        return "warp"
    if t >= WIDE_FIRST:
        return f"wide_k{TIER_WIDTHS[t]}"
    s = stats.get("start_tier", -1)
    group = bool(flags & 32) or (t == s and stats.get("start_lane_groups")) or (t > s >= 0 and not flags & 64)
    lanes = group and (stats.get("start_lane_groups") == 2 or flags & XB_FLAG_LANES)
    return f"{'lane' if lanes else 'group' if group else 'thread'}_k{TIER_WIDTHS[t]}"


class XbStats(C.Structure):
    _fields_ = [("n_devices", C.c_int32), ("launches", C.c_int32), ("ms_total", C.c_double),
                ("ms_prep", C.c_double), ("ms_pilot", C.c_double),
                ("ms_tier", C.c_double * NUM_TIERS), ("units_tier", C.c_int64 * NUM_TIERS),
                ("cells_tier", C.c_int64 * NUM_TIERS), ("escalated", C.c_int64 * NUM_TIERS), ("h2d_bytes", C.c_int64), ("d2h_bytes", C.c_int64),
                ("sm_count", C.c_int32), ("start_tier", C.c_int32), ("dbg", C.c_int64 * 6),
                ("start_lane_groups", C.c_int32), ("reserved", C.c_int32)]

    def as_dict(self) -> dict:
        return {"n_devices": self.n_devices, "launches": self.launches,
                "ms_total": self.ms_total, "ms_prep": self.ms_prep, "ms_pilot": self.ms_pilot,
                "ms_tier": list(self.ms_tier), "units_tier": list(self.units_tier),
                "cells_tier": list(self.cells_tier), "escalated": list(self.escalated),
                "h2d_bytes": self.h2d_bytes, "d2h_bytes": self.d2h_bytes,
                "sm_count": self.sm_count, "start_tier": self.start_tier,
                "dbg": list(self.dbg), "start_lane_groups": int(self.start_lane_groups)}


_lib = None


def lib() -> C.CDLL:
    """Load (once) and type the shared library; raises if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: run `make lib` or __graft_entry__.build()")
    L = C.CDLL(LIB_PATH)
    P, I, I64, V = C.c_void_p, C.c_int, C.c_int64, None
    sig = {
        "xb_version": (C.c_char_p, []),
        "xb_strerror": (C.c_char_p, [I]),
        "xb_device_count": (I, []),
        "xb_scheme_match_mismatch": (P, [I, I, I, I, C.POINTER(I)]),
        "xb_scheme_from_matrix": (P, [C.c_char_p, I, C.POINTER(I), I, I, C.POINTER(I)]),
        "xb_parse_submatrix": (I, [C.c_char_p, C.c_char_p, I, C.POINTER(I), I]),
        "xb_scheme_sim": (I, [P, C.c_char, C.c_char, C.POINTER(I)]),
        "xb_scheme_free": (V, [P]),
        "xb_pool_create": (P, [P, C.POINTER(I)]),
        "xb_pool_add": (I64, [P, C.c_char_p, I64]),
        "xb_pool_add_bulk": (I64, [P, P, P, I64]),
        "xb_pool_size": (I64, [P]),
        "xb_pool_seq_len": (I64, [P, I64]),
        "xb_pool_bits_per_symbol": (I, [P]),
        "xb_pool_evict": (V, [P]),
        "xb_pool_free": (V, [P]),
        "xb_extend_batch": (I, [P, P, I64, I, I, P, P, C.POINTER(I64), C.POINTER(XbExec)]),
        "xb_extend_units": (I, [P, P, I64, I, P, C.POINTER(I64), C.POINTER(XbExec)]),
        "xb_batch_create": (P, [P, P, I64, I, I, C.POINTER(XbExec), C.POINTER(I64), C.POINTER(I)]),
        "xb_batch_run": (I, [P]),
        "xb_batch_sync": (I, [P]),
        "xb_batch_fetch": (I, [P, P, P]),
        "xb_batch_stats": (I, [P, C.POINTER(XbStats)]),
        "xb_batch_free": (V, [P]),
        "xb_last_stats": (I, [C.POINTER(XbStats)]),
        "xb_shard_tasks": (I, [P, P, I64, I, I, I, P, C.POINTER(I64)]),
        "xb_debug_checks": (I, [I, C.POINTER(C.c_uint32)]),
        "xb_plan_group_family": (I, [I, I, I64, C.c_double, C.c_double]),
        "xb_measure_int32_peak": (I, [I, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                      C.POINTER(C.c_double), C.POINTER(I)]),
        "xb_synth_make": (P, [I, C.c_double, C.c_uint64, C.c_char_p, I, C.POINTER(I)]),
        "xb_synth_sizes": (V, [P, C.POINTER(I64)]),
        "xb_synth_copy": (V, [P, P, P, P]),
        "xb_synth_free": (V, [P]),
        "xb_fasta_parse": (P, [P, I64, C.c_char_p, I, P]),
        "xb_fasta_sizes": (V, [P, P]),
        "xb_fasta_copy": (V, [P, P, P, P, P]),
        "xb_pool_add_fasta": (I64, [P, P]),
        "xb_fasta_free": (V, [P]),
        "xb_parse_seeds": (I64, [P, I64, P, I64, P]),
        "xb_parse_overlaps": (I64, [P, I64, P, I64, P]),
        "xb_synth_pairs": (P, [C.c_uint64, C.c_uint64, C.c_double, I, I, C.c_uint64, C.POINTER(I)]),
        "xb_sweep_band": (I, [C.c_uint64, P, C.c_int32, P, C.c_int32, C.c_uint64, P, C.POINTER(XbExec)]),
    }
    for name, (res, args) in sig.items():
        if not hasattr(L, name):  # an older build (A/B runs); tests check the full export list
            continue
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


# every symbol include/xdrop_b200.h declares (checked by the CPU test-suite)
EXPORTED = ["xb_version", "xb_strerror", "xb_device_count", "xb_scheme_match_mismatch",
            "xb_scheme_from_matrix", "xb_parse_submatrix", "xb_scheme_sim", "xb_scheme_free",
            "xb_pool_create", "xb_pool_add", "xb_pool_add_bulk", "xb_pool_size",
            "xb_pool_seq_len", "xb_pool_bits_per_symbol", "xb_pool_evict", "xb_pool_free",
            "xb_extend_batch", "xb_extend_units", "xb_batch_create", "xb_batch_run",
            "xb_batch_sync", "xb_batch_fetch", "xb_batch_stats", "xb_batch_free",
            "xb_last_stats", "xb_measure_int32_peak", "xb_synth_make", "xb_synth_sizes",
            "xb_synth_copy", "xb_synth_free", "xb_synth_pairs", "xb_sweep_band", "xb_fasta_parse",
            "xb_fasta_sizes", "xb_fasta_copy", "xb_pool_add_fasta", "xb_fasta_free", "xb_parse_seeds",
            "xb_parse_overlaps", "xb_shard_tasks", "xb_debug_checks", "xb_plan_group_family"]


class XbParseError(C.Structure):
    _fields_ = [("kind", C.c_int32), ("reserved", C.c_int32), ("line", C.c_int64),
                ("message", C.c_char * 256)]


XB_PARSE_NAMES = ["ok", "MissingHeader", "EmptyRecord", "InvalidSymbol", "MalformedLine",
                  "NegativeIndex", "BadHeader", "IndexOutOfDeclaredShape", "BadArgument"]


class XbError(RuntimeError):
    def __init__(self, code: int, what: str = "", index: int | None = None):
        msg = lib().xb_strerror(code).decode()
        super().__init__(f"{what}: {msg} (code {code})" + (f" at {index}" if index is not None else ""))
        self.code = code
        self.index = index


def check(code: int, what: str = "", index: int | None = None) -> None:
    if code != XB_OK:
        raise XbError(code, what, index)


def make_exec(n_devices: int = 1, device_ids=None, stream=None, flags: int = 0):
    ex = XbExec()
    ex.n_devices = n_devices
    if device_ids is not None:
        arr = (C.c_int32 * len(device_ids))(*device_ids)
        ex.device_ids = arr
        ex._keep = arr  # keep alive
    ex.stream = stream
    ex.flags = flags
    return ex

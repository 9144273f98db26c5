"""ctypes binding of the engine library ``_lib/libbf_gbs.so`` (include/bf_gbs.h).

The library is built in-tree by ``__graft_entry__.build()`` (nvcc, sm_100a).
There is no fallback: if the shared object is missing or no sm_100 device is
present, calls raise immediately.
"""
from __future__ import annotations

import ctypes
import os
import pathlib
import threading

from .errors import BudgetError

LIB_PATH = pathlib.Path(os.environ.get(
    "BF_GBS_LIB", pathlib.Path(__file__).resolve().parent / "_lib" / "libbf_gbs.so"))

BF_OK, BF_EINVAL, BF_ENOMEM, BF_ECUDA, BF_ENODEV, BF_EBUDGET, BF_EIO = range(7)
PRECISION = {"fp32": 0, "fp64": 1}

# Every symbol include/bf_gbs.h declares.
EXPORTS = (
    "bf_version", "bf_last_error", "bf_device_count", "bf_launch_count",
    "bf_gbs_accumulate", "bf_gbs_accumulate_dev", "bf_nearest_on_segments",
    "bf_trace_range_dev", "bf_field_finalize_dev", "bf_plan_chunks", "bf_last_stats",
    "bf_tile_size", "bf_tile_order_dev", "bf_probe_peaks", "bf_last_path_stats", "bf_worklist",
    "bf_last_pair_stats", "bf_write_field_csv", "bf_set_memory_budget", "bf_rows_create",
    "bf_rows_destroy", "bf_rows_info", "bf_rows_append_dev", "bf_gbs_accumulate_rows_dev",
    "bf_set_kernel_timing",
)
FLAG_OBS_PRESORTED = 1
TRACE_EXHAUSTIVE = 1

_lock = threading.Lock()
_lib = None

D = ctypes.POINTER(ctypes.c_double)
I32 = ctypes.POINTER(ctypes.c_int32)
I64P = ctypes.POINTER(ctypes.c_int64)
I64 = ctypes.c_int64
F64 = ctypes.c_double
INT = ctypes.c_int
VP = ctypes.c_void_p


class EngineError(RuntimeError):
    """CUDA / device failure inside the engine library."""


def _declare(lib):
    lib.bf_version.restype = ctypes.c_char_p
    lib.bf_last_error.restype = ctypes.c_char_p
    lib.bf_device_count.restype = INT
    lib.bf_launch_count.restype = ctypes.c_uint64
    gbs_args = [VP] * 7 + [VP, I64, I64, VP, VP, I64, VP, I64, F64, F64, F64, INT, VP, VP,
                           I64, I64, I64, I64, INT, INT]
    lib.bf_gbs_accumulate.argtypes = gbs_args
    lib.bf_gbs_accumulate_dev.argtypes = gbs_args[:-1] + [INT, INT, VP]
    lib.bf_tile_order_dev.argtypes = [VP, I64, VP, INT, VP]
    lib.bf_nearest_on_segments.argtypes = [VP] * 7 + [VP, I64, I64, VP, I64, VP, VP, I64, VP,
                                                      INT]
    lib.bf_trace_range_dev.argtypes = ([VP, VP, VP, VP, I64, VP, F64, VP, VP, VP, VP, F64, I64,
                                        I64] + [VP] * 9 + [I64, I64, I64, INT, INT, VP])
    lib.bf_set_memory_budget.argtypes = [INT, I64]
    lib.bf_set_kernel_timing.argtypes = [INT]
    lib.bf_rows_create.argtypes = [INT, ctypes.POINTER(VP)]
    lib.bf_rows_destroy.argtypes = [VP]
    lib.bf_rows_info.argtypes = [VP, I64P, I64P]
    lib.bf_rows_append_dev.argtypes = [VP] * 8 + [I64, I64, F64, F64, VP]
    lib.bf_gbs_accumulate_rows_dev.argtypes = [VP, VP, I64, VP, I64, F64, INT, VP, VP, I64, I64,
                                               I64, I64, INT, VP]
    lib.bf_field_finalize_dev.argtypes = [VP, I64, F64, VP, VP, INT, VP]
    lib.bf_plan_chunks.argtypes = [I64, I64, I64, I64P, I64, I64P]
    lib.bf_last_stats.argtypes = [I64P, I64P, I64P, I64P, I64P, D, I64P]
    lib.bf_probe_peaks.argtypes = [INT, D, D]
    lib.bf_last_path_stats.argtypes = [I64P] * 4
    lib.bf_last_pair_stats.argtypes = [I64P] * 6
    lib.bf_write_field_csv.argtypes = [ctypes.c_char_p, VP, I64, VP, I64, VP, VP, INT]
    lib.bf_worklist.argtypes = [VP, VP, VP, VP, VP, I64, I64, VP, I64, VP, I64, F64, F64, INT,
                                VP, VP, VP, VP, VP, I64, I64P, INT]
    for name in EXPORTS:
        if name not in ("bf_version", "bf_last_error", "bf_device_count", "bf_launch_count"):
            getattr(lib, name).restype = INT


def load():
    """Load (once) and return the engine library; raises if it was not built."""
    global _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise ImportError(
                    f"engine library {LIB_PATH} is missing: run __graft_entry__.build() "
                    "(there is no CPU fallback)")
            lib = ctypes.CDLL(str(LIB_PATH))
            _declare(lib)
            _lib = lib
    return _lib


def check(status: int) -> None:
    """Map a bf_status to the reference's exception types (errors.py)."""
    if status == BF_OK:
        return
    msg = load().bf_last_error().decode(errors="replace")
    if status == BF_EINVAL:
        raise ValueError(msg)
    if status == BF_ENOMEM:
        raise MemoryError(msg)
    if status == BF_EBUDGET:
        raise BudgetError(msg)
    if status == BF_EIO:
        raise OSError(msg)
    raise EngineError(f"[bf_status {status}] {msg}")


def set_memory_budget(device: int, nbytes: int) -> None:
    """Beam-group workspace budget of the summation on `device` (0 = automatic).

    Changes how a call is grouped, never its results (bf_set_memory_budget)."""
    check(load().bf_set_memory_budget(int(device), int(nbytes)))


def set_kernel_timing(on: bool) -> None:
    """Record kernel_ms (last_stats) for later fp32 calls; off by default (it costs
    ~10 us of graph-node latency per small call)."""
    check(load().bf_set_kernel_timing(1 if on else 0))


def launch_count() -> int:
    return int(load().bf_launch_count())


def last_stats() -> dict:
    """Statistics of the last fp32 summation on this thread (bf_last_stats)."""
    vals = [ctypes.c_int64(0) for _ in range(5)]
    ms = ctypes.c_double(0.0)
    cps = ctypes.c_int64(0)
    check(load().bf_last_stats(*[ctypes.byref(v) for v in vals], ctypes.byref(ms),
                               ctypes.byref(cps)))
    cand, total, ties, tiles, nbp = (v.value for v in vals)
    paths = [ctypes.c_int64(0) for _ in range(4)]
    check(load().bf_last_path_stats(*[ctypes.byref(v) for v in paths]))
    pairs = [ctypes.c_int64(0) for _ in range(6)]
    check(load().bf_last_pair_stats(*[ctypes.byref(v) for v in pairs]))
    a9p, a9s, tp, ts, lp, ls = (v.value for v in pairs)
    return {"candidate_pairs": cand, "total_pairs": total, "tie_pairs": ties, "n_tiles": tiles,
            "tight_pairs": tp, "tight_pair_segs": ts, "live_pairs": lp, "live_pair_segs": ls,
            "nonbehind_pairs": nbp, "kernel_ms": ms.value, "candidate_pair_segs": cps.value,
            "patch_beams": dict(zip(("culled", "single", "wedge", "multi"),
                                    (v.value for v in paths)))}


def probe_peaks(device: int = 0) -> dict:
    """Measured FFMA (TFLOP/s) and MUFU ex2 (Tops/s) throughput (bf_probe_peaks)."""
    f, m = ctypes.c_double(0.0), ctypes.c_double(0.0)
    check(load().bf_probe_peaks(int(device), ctypes.byref(f), ctypes.byref(m)))
    return {"fp32_tflops": f.value, "mufu_tops": m.value}

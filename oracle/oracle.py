"""ctypes front end of the C oracle (gbs_oracle.c) -- TEST INFRASTRUCTURE ONLY.

`gbs_accumulate` has the reference signature (kernels.py:352-355) and its
in-place semantics; `threads` adds the reference's flat observer-block
scheduler (parallel.py:108-140).
"""
from __future__ import annotations

import ctypes
import os
import pathlib
import subprocess

import numpy as np

_DIR = pathlib.Path(__file__).resolve().parent
_LIB = _DIR / "liboracle_gbs.so"
_lib = None

_d = ctypes.POINTER(ctypes.c_double)
_i32 = ctypes.POINTER(ctypes.c_int32)
_i64p = ctypes.POINTER(ctypes.c_int64)
_i64 = ctypes.c_int64


def build() -> pathlib.Path:
    """Compile the oracle with the committed Makefile (gcc, no FMA)."""
    subprocess.run(["make", "-s", "-C", str(_DIR)], check=True)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        if not _LIB.exists():
            build()
        lib = ctypes.CDLL(str(_LIB))
        lib.oracle_gbs_accumulate.argtypes = [
            _d, _d, _d, _d, _d, _d, _d, _i32, _i64, _d, _d, _d, _i64,
            ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_int,
            _d, _i64p, _i64, _i64, _i64, _i64, ctypes.c_int]
        lib.oracle_gbs_accumulate.restype = ctypes.c_int
        lib.oracle_nearest_on_segments.argtypes = [
            _d, _d, _d, _d, _d, _d, _d, _i64, _i64, ctypes.c_double, ctypes.c_double,
            ctypes.c_double, _d]
        lib.oracle_nearest_on_segments.restype = None
        _lib = lib
    return _lib


def _p(a, t=_d):
    return a.ctypes.data_as(t)


def _f64(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a


def gbs_accumulate(seg_origin, seg_dir, seg_e1, seg_e2, seg_len, seg_s0, seg_refl,
                   n_segs, max_seg, weights, obs, omegas, c, width_b, phi_amp,
                   use_cutoff, acc, evals, obs_lo, obs_hi, beam_lo, beam_hi, threads=1):
    lib = _load()
    arrs = [_f64(x) for x in (seg_origin, seg_dir, seg_e1, seg_e2, seg_len, seg_s0,
                              seg_refl)]
    n_segs = np.ascontiguousarray(n_segs, dtype=np.int32)
    weights = _f64(weights)
    obs = _f64(obs)
    omegas = _f64(np.atleast_1d(omegas))
    if acc.dtype != np.complex128 or not acc.flags.c_contiguous:
        raise TypeError("acc must be C-contiguous complex128")
    if evals.dtype != np.int64 or not evals.flags.c_contiguous:
        raise TypeError("evals must be C-contiguous int64")
    rc = lib.oracle_gbs_accumulate(
        *[_p(a) for a in arrs], _p(n_segs, _i32), int(max_seg), _p(weights), _p(obs),
        _p(omegas), omegas.shape[0], float(c), float(width_b), float(phi_amp),
        int(bool(use_cutoff)), acc.ctypes.data_as(_d), _p(evals, _i64p), int(obs_lo),
        int(obs_hi), int(beam_lo), int(beam_hi), int(threads))
    if rc != 0:
        raise MemoryError("oracle thread allocation failed")


def nearest_on_segments(seg_origin, seg_dir, seg_e1, seg_e2, seg_len, seg_s0, seg_refl,
                        base, n_seg, px, py, pz):
    lib = _load()
    out = np.zeros(6)
    arrs = [_f64(x) for x in (seg_origin, seg_dir, seg_e1, seg_e2, seg_len, seg_s0,
                              seg_refl)]
    lib.oracle_nearest_on_segments(*[_p(a) for a in arrs], int(base), int(n_seg),
                                   float(px), float(py), float(pz), _p(out))
    return int(out[0]), out[1], out[2], out[3], out[4], bool(out[5])


def load_bundle(path):
    """Rebuild the padded reference PathBundle arrays from a golden npz.

    Returns a dict with the padded (n_beams*max_seg, ...) arrays exactly as
    allocate_bundle (beamtrace.py:274-288) lays them out, plus the case data.
    """
    z = np.load(path, allow_pickle=False)
    d = {k: z[k] for k in z.files}
    n_segs = d["n_segs"].astype(np.int32)
    S = int(d["max_seg"])
    nb = n_segs.shape[0]
    rows = nb * S
    idx = np.concatenate([np.arange(i * S, i * S + int(n)) for i, n in enumerate(n_segs)])
    out = dict(d)
    for name, width in (("origin", 3), ("dir", 3), ("e1", 3), ("e2", 3)):
        a = np.zeros((rows, width))
        a[idx] = d["v_" + name]
        out["seg_" + name] = a
    for name, fill in (("len", 0.0), ("s0", 0.0), ("refl", 1.0)):
        a = np.full(rows, fill)
        a[idx] = d["v_" + name]
        out["seg_" + name] = a
    out["n_segs"] = n_segs
    out["max_seg"] = S
    return out


def trace(v0, v1, v2, refl, bounds, diameter, origin, dirs, e1s, e2s, length_cap, r_max,
          threads=1):
    """C restatement of trace_range over all rays (trace_oracle.c); padded bundle dict."""
    lib = _load()
    if not hasattr(lib, "_trace_declared"):
        lib.oracle_trace.argtypes = ([_d, _d, _d, _d, _i64, _d, ctypes.c_double, _d, _d, _d, _d,
                                      _i64, ctypes.c_double, _i64, _i64] + [_d] * 7 +
                                     [_i32, _i32, ctypes.c_int])
        lib.oracle_trace.restype = ctypes.c_int
        lib._trace_declared = True
    f = lambda a: np.ascontiguousarray(a, dtype=np.float64)  # noqa: E731
    v0, v1, v2, refl, bounds = f(v0), f(v1), f(v2), f(refl), f(bounds).reshape(-1)
    origin, dirs, e1s, e2s = f(origin), f(dirs), f(e1s), f(e2s)
    n = dirs.shape[0]
    S = int(r_max) + 1
    rows = n * S
    out = dict(seg_origin=np.zeros((rows, 3)), seg_dir=np.zeros((rows, 3)),
               seg_e1=np.zeros((rows, 3)), seg_e2=np.zeros((rows, 3)), seg_len=np.zeros(rows),
               seg_s0=np.zeros(rows), seg_refl=np.ones(rows), n_segs=np.zeros(n, np.int32),
               n_refls=np.zeros(n, np.int32), max_seg=S)
    rc = lib.oracle_trace(_p(v0), _p(v1), _p(v2), _p(refl), v0.shape[0], _p(bounds),
                          float(diameter), _p(origin), _p(dirs), _p(e1s), _p(e2s), n,
                          float(length_cap), int(r_max), S,
                          *[_p(out[k]) for k in ("seg_origin", "seg_dir", "seg_e1", "seg_e2",
                                                 "seg_len", "seg_s0", "seg_refl")],
                          _p(out["n_segs"], _i32), _p(out["n_refls"], _i32), int(threads))
    if rc != 0:
        raise MemoryError("oracle thread allocation failed")
    return out


def worklist(seg_origin, seg_dir, seg_len, seg_s0, n_segs, max_seg, centre, c, width_b,
             omega_min, use_cutoff=True, tight=False, box=None):
    """Tile-level candidate bitmask (worklist_oracle.c); centre is (n_tiles, 4).
    tight=True: the tight list the fp32 kernel walks (subset of the a9 list); needs the
    tiles' bounding-box half extents box (n_tiles, 4: hx, hy, hz, R_T)."""
    lib = _load()
    if not hasattr(lib, "_wl_declared"):
        lib.oracle_worklist.argtypes = [_d, _d, _d, _d, _i32, _i64, _i64, _d, _d, _i64,
                                        ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                        ctypes.c_int, ctypes.c_int,
                                        ctypes.POINTER(ctypes.c_uint32)]
        lib.oracle_worklist.restype = None
        lib._wl_declared = True
    f = lambda a: np.ascontiguousarray(a, dtype=np.float64)  # noqa: E731
    so, sd, sl, ss0, centre = f(seg_origin), f(seg_dir), f(seg_len), f(seg_s0), f(centre)
    n_segs = np.ascontiguousarray(n_segs, dtype=np.int32)
    nb = n_segs.shape[0]
    nt = centre.reshape(-1, 4).shape[0]
    if tight and box is None:
        raise ValueError("the tight list needs the tiles' bounding boxes")
    bx = f(box).reshape(nt, 4) if box is not None else None
    bits = np.zeros((nt, (nb + 31) // 32), np.uint32)
    lib.oracle_worklist(_p(so), _p(sd), _p(sl), _p(ss0), _p(n_segs, _i32), nb, int(max_seg),
                        _p(centre), _p(bx) if bx is not None else None, nt, float(c),
                        float(width_b), float(omega_min), int(bool(use_cutoff)),
                        int(bool(tight)), bits.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)))
    return bits

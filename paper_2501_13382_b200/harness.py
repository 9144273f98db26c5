"""Field writers of the GBS stage (mirror of ``beamfield.harness``).

Reference: /root/reference/pkg/src/beamfield/harness.py.  Kept names, files and bytes:
``write_field_csv`` (harness.py:197-208) writes the same CSV -- header
``x,y,z,freq_hz,re_p,im_p,spl_db``, observer-major rows, numbers as ``format(x,
".17g")`` (harness.py:39-40) -- through the native multithreaded formatter
``bf_write_field_csv``; ``emit_heatmap`` (harness.py:224-255) writes the same 8-bit
grayscale SPL raster and ``.txt`` sidecar.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib

FIELD_CSV_HEADER = "x,y,z,freq_hz,re_p,im_p,spl_db"


def _g(x) -> str:
    return format(float(x), ".17g")


def write_field_csv(path, observers, freqs, field, threads: int = 0) -> None:
    """One row per (observer, frequency), observer index major (harness.py:197-208)."""
    pts = np.ascontiguousarray(getattr(observers, "points", observers), dtype=np.float64)
    fr = np.ascontiguousarray(np.atleast_1d(freqs), dtype=np.float64)
    p = np.ascontiguousarray(field.pressure, dtype=np.complex128)
    s = np.ascontiguousarray(field.spl, dtype=np.float64)
    n = pts.shape[0]
    if p.shape != (n, fr.shape[0]) or s.shape != p.shape:
        raise ValueError("field shape does not match observers x frequencies")
    vp = lambda a: ctypes.c_void_p(a.ctypes.data)  # noqa: E731
    _lib.check(_lib.load().bf_write_field_csv(str(path).encode(), vp(pts), n, vp(fr),
                                              fr.shape[0], vp(p), vp(s), int(threads)))


def emit_heatmap(spl_values, grid_spec, out_path) -> dict:
    """8-bit grayscale raster of the SPL grid (row-major n2 x n1): [min, max] of the
    finite values mapped linearly onto [0, 255] (rounded half to even), non-finite
    (null) points 0; sidecar ``<out_path>.txt`` records the scale (harness.py:224-255)."""
    from PIL import Image

    n1, n2 = int(grid_spec.n1), int(grid_spec.n2)
    v = np.asarray(spl_values, dtype=np.float64).reshape(n2, n1)
    ok = np.isfinite(v)
    nulls = int(v.size - np.count_nonzero(ok))
    lo, hi = (float(v[ok].min()), float(v[ok].max())) if ok.any() else (0.0, 0.0)
    img = np.zeros(v.shape, dtype=np.uint8)
    if hi > lo:
        img = np.rint(np.clip((v - lo) / (hi - lo), 0.0, 1.0) * 255.0).astype(np.uint8)
    img[~ok] = 0
    Image.fromarray(img, mode="L").save(out_path)
    with open(str(out_path) + ".txt", "w", encoding="utf-8") as fh:
        fh.write(f"width={n1}\nheight={n2}\n")
        fh.write(f"spl_min_db={_g(lo)}\nspl_max_db={_g(hi)}\n")
        fh.write(f"null_points={nulls}\n")
        fh.write("mapping=linear [spl_min_db, spl_max_db] -> [0, 255], row-major\n")
    return {"width": n1, "height": n2, "spl_min_db": lo, "spl_max_db": hi,
            "null_points": nulls}

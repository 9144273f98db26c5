"""Field-reconstruction API of the GBS stage (mirror of reference ``beamfield.gbs``).

/root/reference/pkg/src/beamfield/gbs.py.  The summation itself always runs on
the B200 (kernels.gbs_accumulate -> libbf_gbs); this module keeps the
reference's types, argument meanings and error behaviour:

* ``spl``            gbs.py:39-46   20 log10(|p| / 2e-5), -inf at |p| = 0
* ``ObserverSet``    gbs.py:62-76   (N, 3) finite fp64, N >= 1
* ``FieldResult``    gbs.py:79-88
* ``bundle_from_paths`` gbs.py:91-126 (vectorised packing, same layout)
* ``sum_at_observer``   gbs.py:176-205
* ``calibrate_phi``     gbs.py:208-256 (26 probes batched into ONE device call)
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import kernels
from .beamtrace import Atmosphere, BeamPath, PathBundle, SourceSpec
from .errors import CalibrationError, DegenerateBeamError

P_REF = 2e-5
CALIBRATION_RADIUS = 10.0
CALIBRATION_MIN_RAYS = 64 * 64


def spl(pressure):
    """Sound pressure level re 20 uPa; zero magnitude maps to -inf."""
    mag = np.abs(pressure)
    with np.errstate(divide="ignore"):
        out = 20.0 * np.log10(mag / P_REF)
    if np.isscalar(pressure) or np.asarray(pressure).ndim == 0:
        return float(out)
    return out


def continuous_sqrt(values) -> np.ndarray:
    """Square root with the branch followed continuously along a sampled path."""
    values = np.asarray(values, dtype=np.complex128)
    return np.sqrt(np.abs(values)) * np.exp(0.5j * np.unwrap(np.angle(values)))


@dataclass(frozen=True)
class ObserverSet:
    points: np.ndarray

    def __post_init__(self):
        pts = np.ascontiguousarray(self.points, dtype=np.float64).reshape(-1, 3)
        if pts.shape[0] < 1:
            raise ValueError("observer set must contain at least one point")
        if not np.all(np.isfinite(pts)):
            raise ValueError("observer coordinates must be finite")
        object.__setattr__(self, "points", pts)

    @property
    def count(self) -> int:
        return self.points.shape[0]


@dataclass
class FieldResult:
    """Complex pressure and SPL per (observer, frequency)."""
    pressure: np.ndarray
    spl: np.ndarray
    calibration: float

    @classmethod
    def from_pressure(cls, pressure: np.ndarray, calibration: float) -> "FieldResult":
        return cls(pressure=pressure, spl=spl(pressure), calibration=calibration)


def bundle_from_paths(paths, atmosphere: Atmosphere | None = None) -> PathBundle:
    """Pack BeamPath objects into the padded PathBundle layout (gbs.py:91-126)."""
    paths = list(paths)
    if not paths:
        raise ValueError("empty path list")
    c, imb, phi = paths[0].c, paths[0].beam_param_im, paths[0].amplitude_phi
    for p in paths:
        if p.c != c or p.beam_param_im != imb or p.amplitude_phi != phi:
            raise ValueError("paths in one bundle must share launch constants")
    S = max(len(p.segments) for p in paths)
    n = len(paths)
    counts = np.array([len(p.segments) for p in paths], dtype=np.int32)
    rows = (np.repeat(np.arange(n) * S, counts)
            + np.concatenate([np.arange(k) for k in counts]) if counts.sum() else
            np.zeros(0, np.int64))
    segs = [s for p in paths for s in p.segments]

    def col(get, width):
        out = np.zeros((n * S, width)) if width > 1 else np.zeros(n * S)
        if segs:
            out[rows] = np.array([get(s) for s in segs], dtype=np.float64)
        return out

    refl = np.ones(n * S)
    if segs:
        refl[rows] = [s.cum_reflection for s in segs]
    return PathBundle(
        seg_origin=col(lambda s: s.origin, 3), seg_dir=col(lambda s: s.direction, 3),
        seg_e1=col(lambda s: s.e1, 3), seg_e2=col(lambda s: s.e2, 3),
        seg_len=col(lambda s: s.length, 1), seg_s0=col(lambda s: s.s_start, 1), seg_refl=refl,
        n_segs=counts, n_refls=np.array([p.n_reflections for p in paths], dtype=np.int32),
        max_seg=S, weights=np.array([p.weight_dgamma for p in paths]),
        gamma1=np.array([p.gamma1 for p in paths]), gamma2=np.array([p.gamma2 for p in paths]),
        c=c, beam_param_im=imb, amplitude_phi=phi)


def _as_bundle(paths) -> PathBundle:
    return paths if hasattr(paths, "seg_origin") else bundle_from_paths(paths)


def nearest_on_path(observer, path: BeamPath):
    """Closest polyline point (segment index, s*, q 2-vector) -- gbs.py:133-145."""
    b = bundle_from_paths([path])
    px, py, pz = np.asarray(observer, dtype=np.float64)
    k, s, q1, q2, _refl, _behind = kernels.nearest_on_segments(
        b.seg_origin, b.seg_dir, b.seg_e1, b.seg_e2, b.seg_len, b.seg_s0, b.seg_refl,
        0, int(b.n_segs[0]), px, py, pz)
    return int(k), float(s), np.array([q1, q2])


def beam_pressure(path: BeamPath, s_star: float, q, omega: float, atmosphere: Atmosphere,
                  source: SourceSpec) -> complex:
    """Single-beam field at ray-centred coordinates (gbs.py:148-173), scalar."""
    imb = path.beam_param_im
    if not imb < 0:
        raise DegenerateBeamError("beam envelope matrix is not decaying (Im(PQ^-1) not positive)")
    c = atmosphere.sound_speed
    qs = s_star + 1j * imb
    if qs == 0:
        raise DegenerateBeamError("det Q vanished along the beam")
    r_acc = 1.0
    for seg in path.segments:
        if seg.s_start <= s_star or math.isclose(seg.s_start, s_star):
            r_acc = seg.cum_reflection
    q = np.asarray(q, dtype=np.float64)
    expo = 1j * omega * (s_star / c) + 1j * omega * float(q @ q) / (2.0 * c * qs)
    return complex(source.amplitude_phi * np.sqrt(c) / qs * r_acc * np.exp(expo))


def _sum_many(points, bundle: PathBundle, omegas, use_cutoff, precision=None, device=None):
    obs = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
    acc = np.zeros((obs.shape[0], omegas.shape[0]), dtype=np.complex128)
    evals = np.zeros(obs.shape[0], dtype=np.int64)
    kernels.gbs_accumulate(
        bundle.seg_origin, bundle.seg_dir, bundle.seg_e1, bundle.seg_e2, bundle.seg_len,
        bundle.seg_s0, bundle.seg_refl, bundle.n_segs, bundle.max_seg, bundle.weights, obs,
        omegas, bundle.c, -bundle.beam_param_im, bundle.amplitude_phi, use_cutoff, acc, evals,
        0, obs.shape[0], 0, bundle.n_paths, precision=precision, device=device)
    return acc


def sum_at_observer(observer, paths, omega, atmosphere: Atmosphere, source: SourceSpec,
                    calibration: float = 1.0, use_cutoff: bool = True, *, precision=None,
                    device=None):
    """Calibrated beam sum at one observer, beams ascending (gbs.py:176-205)."""
    scalar = np.isscalar(omega) or np.asarray(omega).ndim == 0
    omegas = np.atleast_1d(np.asarray(omega, dtype=np.float64))
    if not hasattr(paths, "seg_origin") and len(paths) == 0:
        return 0j if scalar else np.zeros(omegas.shape[0], dtype=np.complex128)
    bundle = _as_bundle(paths)
    if not bundle.beam_param_im < 0:
        raise DegenerateBeamError("bundle carries a non-decaying beam parameter")
    out = calibration * _sum_many(np.asarray(observer, dtype=np.float64).reshape(1, 3), bundle,
                                  omegas, use_cutoff, precision, device)[0]
    return complex(out[0]) if scalar else out


def calibration_probes(radius: float = CALIBRATION_RADIUS) -> np.ndarray:
    """The 26 lattice directions x radius, in the reference's loop order (gbs.py:228-236)."""
    probes = []
    for i in (-1, 0, 1):
        for j in (-1, 0, 1):
            for k in (-1, 0, 1):
                if i == j == k == 0:
                    continue
                v = np.array([i, j, k], dtype=np.float64)
                probes.append(radius * (v / np.linalg.norm(v)))
    return np.asarray(probes)


def calibrate_phi(paths, atmosphere: Atmosphere, source: SourceSpec, omegas=None,
                  probe_radius: float = CALIBRATION_RADIUS, *, precision=None,
                  device=None) -> float:
    """Fit the real summation scale against the free-field monopole (gbs.py:208-256).

    Probes sit around the WORLD ORIGIN exactly as in the reference (a known
    reference defect for sources off the origin); all 26 probes
    and all frequencies are summed in one device call.
    """
    bundle = _as_bundle(paths)
    if bundle.n_paths < CALIBRATION_MIN_RAYS:
        raise CalibrationError(
            f"calibration needs a full-sphere launch of at least {CALIBRATION_MIN_RAYS} rays")
    if int(np.max(bundle.n_refls, initial=0)) > 0:
        raise CalibrationError("calibration requires free-field paths (no reflections)")
    if not bundle.beam_param_im < 0:
        raise DegenerateBeamError("bundle carries a non-decaying beam parameter")
    omegas = source.omegas if omegas is None else omegas
    omegas = np.atleast_1d(np.asarray(omegas, dtype=np.float64))
    probes = calibration_probes(1.0)
    pts = probe_radius * probes
    mags_all = np.abs(_sum_many(pts, bundle, omegas, True, precision, device))  # (26, F)
    target = 1.0 / (4.0 * np.pi * probe_radius)
    scales = []
    for f in range(omegas.shape[0]):
        mags = mags_all[:, f]
        if np.any(mags == 0.0):
            raise CalibrationError("calibration probe saw a null field")
        spread_db = 20.0 * np.log10(mags.max() / mags.min())
        if spread_db > 1.0:
            raise CalibrationError(
                f"calibration did not converge: {spread_db:.2f} dB spread over probe directions")
        scales.append(target / mags.mean())
    scales = np.asarray(scales)
    drift = np.abs(20.0 * np.log10(scales / scales[0]))
    if drift.max() > 0.5:
        raise CalibrationError(
            f"calibration scale varies {drift.max():.2f} dB across frequencies")
    return float(scales[0])

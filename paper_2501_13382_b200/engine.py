"""Device-resident GBS engine: HBM buffers owned by torch, compute in libbf_gbs.

This is the layer ``parallel.run_pipeline`` drives (the reference's per-chunk
trace -> sum loop, parallel.py:297-338, moved onto the B200):

* :class:`DeviceScene` -- triangle soup in HBM for the tracer;
* :func:`trace_device_rows` -- sm_100a tracer into a padded device bundle
  (the reference PathBundle layout, beamtrace.py:274-288);
* :class:`DeviceBundle` -- a device PathBundle (torch tensors) + upload from a
  host PathBundle (pinned, async);
* :func:`accumulate` -- ``bf_gbs_accumulate_dev`` on device buffers;
* :class:`SegmentRows` -- compact segment rows resident in HBM (``bf_rows_*``):
  traced chunks are appended (68 B per segment, no padding) and every ray is
  summed in one call, independent of the chunk plan.

Host-resident bundles larger than the device budget need no Python streaming:
the host-buffer ABI (``bf_gbs_accumulate``) streams beam groups through pinned
staging itself, copy of group g+1 overlapping the summation of group g.

PyTorch is used for allocation, streams and events only.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib

SEG_FIELDS = ("seg_origin", "seg_dir", "seg_e1", "seg_e2", "seg_len", "seg_s0", "seg_refl")


def _torch():
    import torch
    return torch


def _vp(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


CUDA_STREAM_LEGACY = 0x1  # cudaStreamLegacy (cuda_runtime_api.h)


def _stream_ptr(stream, device=None):
    """The cudaStream_t of `stream`; None -> torch's current stream on `device`, so the
    engine's work is ordered after the torch kernels that produced its inputs.  torch's
    default stream has handle 0, which the C ABI reads as "the engine's own stream,
    synchronous"; it is passed as cudaStreamLegacy instead (the same stream, explicitly)."""
    if stream is None:
        torch = _torch()
        stream = torch.cuda.current_stream(device)
    return ctypes.c_void_p(stream.cuda_stream or CUDA_STREAM_LEGACY)


@dataclass
class DeviceScene:
    v0: object
    v1: object
    v2: object
    refl: object
    bounds: object  # (6,) bmin xyz, bmax xyz
    diameter: float
    n_tri: int

    @classmethod
    def from_scene(cls, scene, device) -> "DeviceScene":
        torch = _torch()

        def f64(a, shape):
            a = np.ascontiguousarray(np.asarray(a, dtype=np.float64).reshape(shape))
            return torch.from_numpy(a).to(device)

        n = int(np.asarray(scene.v0).reshape(-1, 3).shape[0])
        return cls(v0=f64(scene.v0, (-1, 3)), v1=f64(scene.v1, (-1, 3)),
                   v2=f64(scene.v2, (-1, 3)), refl=f64(scene.refl, (-1,)),
                   bounds=f64(scene.bounds, (6,)), diameter=float(scene.diameter), n_tri=n)


@dataclass
class DeviceBundle:
    """Padded PathBundle in HBM (same layout as beamtrace.PathBundle)."""
    seg_origin: object
    seg_dir: object
    seg_e1: object
    seg_e2: object
    seg_len: object
    seg_s0: object
    seg_refl: object
    n_segs: object
    n_refls: object
    weights: object
    max_seg: int
    c: float
    beam_param_im: float
    amplitude_phi: float

    @property
    def n_paths(self) -> int:
        return int(self.n_segs.numel())

    @classmethod
    def empty(cls, n_rays, max_seg, device, c, beam_param_im, amplitude_phi, weights=None):
        torch = _torch()
        rows = n_rays * max_seg
        z = dict(dtype=torch.float64, device=device)
        return cls(seg_origin=torch.zeros((rows, 3), **z), seg_dir=torch.zeros((rows, 3), **z),
                   seg_e1=torch.zeros((rows, 3), **z), seg_e2=torch.zeros((rows, 3), **z),
                   seg_len=torch.zeros(rows, **z), seg_s0=torch.zeros(rows, **z),
                   seg_refl=torch.ones(rows, **z),
                   n_segs=torch.zeros(n_rays, dtype=torch.int32, device=device),
                   n_refls=torch.zeros(n_rays, dtype=torch.int32, device=device),
                   weights=(weights if weights is not None else torch.zeros(n_rays, **z)),
                   max_seg=max_seg, c=c, beam_param_im=beam_param_im,
                   amplitude_phi=amplitude_phi)

    @classmethod
    def from_host(cls, b, device, with_frame=True, non_blocking=False) -> "DeviceBundle":
        """Upload a host PathBundle (or reference PathBundle) to HBM."""
        torch = _torch()

        def up(a, dtype):
            t = torch.from_numpy(np.ascontiguousarray(a, dtype=dtype))
            if non_blocking:
                t = t.pin_memory()
            return t.to(device, non_blocking=non_blocking)

        f = np.float64
        return cls(seg_origin=up(b.seg_origin, f), seg_dir=up(b.seg_dir, f),
                   seg_e1=up(b.seg_e1, f) if with_frame else None,
                   seg_e2=up(b.seg_e2, f) if with_frame else None,
                   seg_len=up(b.seg_len, f), seg_s0=up(b.seg_s0, f), seg_refl=up(b.seg_refl, f),
                   n_segs=up(b.n_segs, np.int32), n_refls=up(b.n_refls, np.int32),
                   weights=up(b.weights, f), max_seg=int(b.max_seg), c=float(b.c),
                   beam_param_im=float(b.beam_param_im),
                   amplitude_phi=float(b.amplitude_phi))

    def to_host(self):
        from .beamtrace import PathBundle
        g = lambda t: None if t is None else t.cpu().numpy()  # noqa: E731
        n = self.n_paths
        return PathBundle(seg_origin=g(self.seg_origin), seg_dir=g(self.seg_dir),
                          seg_e1=g(self.seg_e1), seg_e2=g(self.seg_e2), seg_len=g(self.seg_len),
                          seg_s0=g(self.seg_s0), seg_refl=g(self.seg_refl),
                          n_segs=g(self.n_segs), n_refls=g(self.n_refls), max_seg=self.max_seg,
                          weights=g(self.weights), gamma1=np.zeros(n), gamma2=np.zeros(n),
                          c=self.c, beam_param_im=self.beam_param_im,
                          amplitude_phi=self.amplitude_phi)


def trace_device_rows(dscene: DeviceScene, source, launch, cfg, c, lo, hi, device,
                      row_base=None, out: DeviceBundle | None = None, stream=None,
                      exhaustive=False):
    """Trace launch rays [lo, hi) on the GPU (kernels.trace_range, kernels.py:282-301).

    Fills ``out`` (allocated when None) rows [(lo-row_base)*S, (hi-row_base)*S).
    Returns a dict of the device arrays (and 'max_seg').
    """
    torch = _torch()
    lib = _lib.load()
    row_base = lo if row_base is None else row_base
    S = cfg.r_max + 1
    n = hi - row_base
    if out is None:
        w = torch.from_numpy(np.ascontiguousarray(launch.weights[row_base:hi])).to(device)
        out = DeviceBundle.empty(n, S, device, c, source.beam_param_im, source.amplitude_phi,
                                 weights=w)
    f64 = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(device)  # noqa
    dirs = f64(launch.directions[row_base:hi])
    e1s = f64(launch.e1[row_base:hi])
    e2s = f64(launch.e2[row_base:hi])
    origin = f64(source.position)
    # Rays are indexed relative to row_base inside the launch slices passed down.
    _lib.check(lib.bf_trace_range_dev(
        _vp(dscene.v0), _vp(dscene.v1), _vp(dscene.v2), _vp(dscene.refl), dscene.n_tri,
        _vp(dscene.bounds), dscene.diameter, _vp(origin), _vp(dirs), _vp(e1s), _vp(e2s),
        float(cfg.length_cap(c)), int(cfg.r_max), S, _vp(out.seg_origin), _vp(out.seg_dir),
        _vp(out.seg_e1), _vp(out.seg_e2), _vp(out.seg_len), _vp(out.seg_s0),
        _vp(out.seg_refl), _vp(out.n_segs), _vp(out.n_refls), lo - row_base, hi - row_base, 0,
        _lib.TRACE_EXHAUSTIVE if exhaustive else 0, device.index or 0,
        _stream_ptr(stream, device)))
    d = {k: getattr(out, k) for k in SEG_FIELDS + ("n_segs", "n_refls", "weights")}
    d["max_seg"] = S
    d["bundle"] = out
    return d


def accumulate(bundle: DeviceBundle, obs, omegas, width_b, use_cutoff, acc, evals,
               obs_lo=0, obs_hi=None, beam_lo=0, beam_hi=None, precision="fp32", stream=None,
               presorted=False):
    """bf_gbs_accumulate_dev on a DeviceBundle (kernels.py:352-399 semantics)."""
    lib = _lib.load()
    n_obs = obs.numel() // 3
    obs_hi = n_obs if obs_hi is None else obs_hi
    beam_hi = bundle.n_paths if beam_hi is None else beam_hi
    om = np.ascontiguousarray(np.atleast_1d(omegas), dtype=np.float64)
    prec = _lib.PRECISION[precision]
    if prec == 1 and bundle.seg_e1 is None:
        raise ValueError("fp64 mode needs the segment frames (seg_e1/seg_e2)")
    _lib.check(lib.bf_gbs_accumulate_dev(
        _vp(bundle.seg_origin), _vp(bundle.seg_dir), _vp(bundle.seg_e1), _vp(bundle.seg_e2),
        _vp(bundle.seg_len), _vp(bundle.seg_s0), _vp(bundle.seg_refl), _vp(bundle.n_segs),
        bundle.n_paths, bundle.max_seg, _vp(bundle.weights), _vp(obs), n_obs,
        ctypes.c_void_p(om.ctypes.data), om.shape[0], float(bundle.c), float(width_b),
        float(bundle.amplitude_phi), int(bool(use_cutoff)), _vp(acc), _vp(evals), int(obs_lo),
        int(obs_hi), int(beam_lo), int(beam_hi), prec,
        _lib.FLAG_OBS_PRESORTED if presorted else 0, obs.device.index or 0,
        _stream_ptr(stream, obs.device)))


def finalize(acc, calibration, stream=None):
    """pressure = calibration*acc and SPL on the device (parallel.py:343, gbs.py:39-46)."""
    torch = _torch()
    lib = _lib.load()
    pressure = torch.empty_like(acc)
    spl = torch.empty(acc.shape, dtype=torch.float64, device=acc.device)
    _lib.check(lib.bf_field_finalize_dev(_vp(acc), acc.numel(), float(calibration),
                                         _vp(pressure), _vp(spl), acc.device.index or 0,
                                         _stream_ptr(stream, acc.device)))
    return pressure, spl


class SegmentRows:
    """Compact segment rows resident on one device (bf_rows_*, include/bf_gbs.h).

    ``append`` packs the valid rows of a padded DeviceBundle (the reference PathBundle
    layout) behind the rows appended so far; ``accumulate`` runs the fp32 summation over
    all (or a range of) the appended beams -- the same bits as one
    ``bf_gbs_accumulate_dev`` call over the concatenated bundle.
    """

    def __init__(self, device):
        torch = _torch()
        self.device = torch.device(device)
        self._lib = _lib.load()
        h = ctypes.c_void_p()
        _lib.check(self._lib.bf_rows_create(self.device.index or 0, ctypes.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            _lib.check(self._lib.bf_rows_destroy(self._h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 (interpreter shutdown)
            pass

    @property
    def n_beams(self) -> int:
        nb, nr = ctypes.c_int64(0), ctypes.c_int64(0)
        _lib.check(self._lib.bf_rows_info(self._h, ctypes.byref(nb), ctypes.byref(nr)))
        return nb.value

    @property
    def n_rows(self) -> int:
        nb, nr = ctypes.c_int64(0), ctypes.c_int64(0)
        _lib.check(self._lib.bf_rows_info(self._h, ctypes.byref(nb), ctypes.byref(nr)))
        return nr.value

    def append(self, bundle: DeviceBundle, n_beams=None, stream=None):
        n = bundle.n_paths if n_beams is None else int(n_beams)
        _lib.check(self._lib.bf_rows_append_dev(
            self._h, _vp(bundle.seg_origin), _vp(bundle.seg_dir), _vp(bundle.seg_len),
            _vp(bundle.seg_s0), _vp(bundle.seg_refl), _vp(bundle.n_segs), _vp(bundle.weights),
            n, int(bundle.max_seg), float(bundle.c), float(bundle.amplitude_phi),
            _stream_ptr(stream, self.device)))

    def accumulate(self, obs, omegas, width_b, use_cutoff, acc, evals, obs_lo=0, obs_hi=None,
                   beam_lo=0, beam_hi=None, stream=None, presorted=False):
        n_obs = obs.numel() // 3
        obs_hi = n_obs if obs_hi is None else obs_hi
        beam_hi = self.n_beams if beam_hi is None else beam_hi
        om = np.ascontiguousarray(np.atleast_1d(omegas), dtype=np.float64)
        _lib.check(self._lib.bf_gbs_accumulate_rows_dev(
            self._h, _vp(obs), n_obs, ctypes.c_void_p(om.ctypes.data), om.shape[0],
            float(width_b), int(bool(use_cutoff)), _vp(acc), _vp(evals), int(obs_lo),
            int(obs_hi), int(beam_lo), int(beam_hi),
            _lib.FLAG_OBS_PRESORTED if presorted else 0, _stream_ptr(stream, obs.device)))

"""Drop-in operator surface of the reference ``beamfield.kernels`` GBS path.

``gbs_accumulate`` keeps the reference signature and in-place semantics
(/root/reference/pkg/src/beamfield/kernels.py:352-399): positional fp64
arrays in the PathBundle layout, ``acc`` (n_obs, F) complex128 and ``evals``
(n_obs,) int64 continued in place over ``[obs_lo, obs_hi)``, beams
``[beam_lo, beam_hi)`` visited in ascending order per observer.

It runs on the B200 through the C ABI (include/bf_gbs.h):

* numpy arguments  -> ``bf_gbs_accumulate`` (host buffers; the library copies
  the beam/observer ranges to HBM, sums, copies acc/evals back);
* torch CUDA tensors -> ``bf_gbs_accumulate_dev`` (device-resident, no copies).

``precision="fp64"`` (the default of this operator-level drop-in) follows the
reference operation order without FMA: like the reference it is bit-identical
under any split of the beam or observer ranges (the reference's sequential /
flat / dynamic schedulers, parallel.py:108-181, call it on disjoint observer
blocks) and within 1e-12 of the reference's values (libm vs CUDA exp/sincos).
``precision="fp32"`` is the fast FP32/MUFU kernel with fp64 tie re-decision and
fp64-anchored phase (relL2 <= 1e-4, dTL <= 0.01 dB against the reference); its
bits depend on the call's beam and observer sets (patch-local fp32 geometry),
not on memory budgets, host vs device inputs or the number of ranks.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib

# kernels.py:14,18
EPS_HIT = 1e-6
CUTOFF_EXPONENT = -36.0

# operator-level default: the mode whose results do not depend on how a caller splits
# its ranges (see the module docstring); the pipeline API defaults to fp32
DEFAULT_PRECISION = "fp64"
PIPELINE_PRECISION = "fp32"


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def _np_in(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def _ptr(a):
    if a is None:
        return None
    if _is_torch(a):
        return ctypes.c_void_p(a.data_ptr())
    return ctypes.c_void_p(a.ctypes.data)


def _precision(precision):
    p = DEFAULT_PRECISION if precision is None else precision
    if p not in _lib.PRECISION:
        raise ValueError(f"unknown precision {p!r} (expected 'fp32' or 'fp64')")
    return _lib.PRECISION[p]


def gbs_accumulate(seg_origin, seg_dir, seg_e1, seg_e2, seg_len, seg_s0, seg_refl,
                   n_segs, max_seg, weights, obs, omegas, c, width_b, phi_amp,
                   use_cutoff, acc, evals, obs_lo, obs_hi, beam_lo, beam_hi, *,
                   precision=None, device=None, stream=None):
    """Accumulate beam contributions into acc[obs, freq], beams in index order.

    Same contract as the reference (kernels.py:352-361).  width_b is the
    magnitude of the (negative) imaginary launch parameter.
    """
    lib = _lib.load()
    prec = _precision(precision)
    max_seg = int(max_seg)
    if _is_torch(acc):
        return _gbs_dev(lib, seg_origin, seg_dir, seg_e1, seg_e2, seg_len, seg_s0, seg_refl,
                        n_segs, max_seg, weights, obs, omegas, c, width_b, phi_amp,
                        use_cutoff, acc, evals, obs_lo, obs_hi, beam_lo, beam_hi, prec,
                        stream)
    if not (isinstance(acc, np.ndarray) and acc.dtype == np.complex128
            and acc.flags.c_contiguous and acc.ndim == 2):
        raise TypeError("acc must be a C-contiguous (n_obs, n_freq) complex128 array")
    if not (isinstance(evals, np.ndarray) and evals.dtype == np.int64
            and evals.flags.c_contiguous):
        raise TypeError("evals must be a C-contiguous int64 array")
    n_segs = _np_in(n_segs, np.int32)
    n_beams = n_segs.shape[0]
    rows = n_beams * max_seg
    geo = [_np_in(a, np.float64) for a in (seg_origin, seg_dir, seg_len, seg_s0, seg_refl)]
    if geo[0].size < 3 * rows or geo[1].size < 3 * rows or min(g.size for g in geo[2:]) < rows:
        raise ValueError("segment arrays shorter than n_beams * max_seg rows")
    e1 = _np_in(seg_e1, np.float64) if prec == 1 else None
    e2 = _np_in(seg_e2, np.float64) if prec == 1 else None
    weights = _np_in(weights, np.float64)
    obs = _np_in(obs, np.float64).reshape(-1, 3)
    omegas = _np_in(np.atleast_1d(omegas), np.float64)
    nf = omegas.shape[0]
    if acc.shape != (obs.shape[0], nf):
        raise ValueError(f"acc shape {acc.shape} != (n_obs, n_freq) = {(obs.shape[0], nf)}")
    if evals.shape[0] != obs.shape[0]:
        raise ValueError("evals length != n_obs")
    dev = 0 if device is None else int(device)
    _lib.check(lib.bf_gbs_accumulate(
        _ptr(geo[0]), _ptr(geo[1]), _ptr(e1), _ptr(e2), _ptr(geo[2]), _ptr(geo[3]),
        _ptr(geo[4]), _ptr(n_segs), n_beams, max_seg, _ptr(weights), _ptr(obs),
        obs.shape[0], _ptr(omegas), nf, float(c), float(width_b), float(phi_amp),
        int(bool(use_cutoff)), _ptr(acc), _ptr(evals), int(obs_lo), int(obs_hi),
        int(beam_lo), int(beam_hi), prec, dev))


def _gbs_dev(lib, seg_origin, seg_dir, seg_e1, seg_e2, seg_len, seg_s0, seg_refl, n_segs,
             max_seg, weights, obs, omegas, c, width_b, phi_amp, use_cutoff, acc, evals,
             obs_lo, obs_hi, beam_lo, beam_hi, prec, stream):
    import torch
    dev = acc.device
    if dev.type != "cuda":
        raise TypeError("torch path needs CUDA tensors (there is no CPU fallback)")
    f64 = [seg_origin, seg_dir, seg_len, seg_s0, seg_refl, weights, obs]
    if prec == 1:
        f64 += [seg_e1, seg_e2]
    for t in f64:
        if t.dtype != torch.float64 or not t.is_contiguous() or t.device != dev:
            raise TypeError("device arrays must be contiguous float64 CUDA tensors on one device")
    if n_segs.dtype != torch.int32 or not n_segs.is_contiguous():
        raise TypeError("n_segs must be a contiguous int32 CUDA tensor")
    if acc.dtype != torch.complex128 or not acc.is_contiguous() or acc.dim() != 2:
        raise TypeError("acc must be a contiguous (n_obs, n_freq) complex128 CUDA tensor")
    if evals.dtype != torch.int64 or not evals.is_contiguous():
        raise TypeError("evals must be a contiguous int64 CUDA tensor")
    om = np.ascontiguousarray(np.atleast_1d(
        omegas.detach().cpu().numpy() if _is_torch(omegas) else omegas), dtype=np.float64)
    nf = om.shape[0]
    n_obs = obs.numel() // 3
    if tuple(acc.shape) != (n_obs, nf):
        raise ValueError(f"acc shape {tuple(acc.shape)} != {(n_obs, nf)}")
    if stream is None:
        stream = torch.cuda.current_stream(dev)  # ordered after the producers of the inputs
    # torch's default stream (handle 0) goes as cudaStreamLegacy: asynchronous and ordered
    # on it (a bare 0 would ask the C ABI for its own stream and a synchronous call)
    st = ctypes.c_void_p((stream.cuda_stream or 0x1) if hasattr(stream, "cuda_stream")
                         else int(stream))
    _lib.check(lib.bf_gbs_accumulate_dev(
        _ptr(seg_origin), _ptr(seg_dir), _ptr(seg_e1) if prec == 1 else None,
        _ptr(seg_e2) if prec == 1 else None, _ptr(seg_len), _ptr(seg_s0), _ptr(seg_refl),
        _ptr(n_segs), n_segs.numel(), int(max_seg), _ptr(weights), _ptr(obs), n_obs,
        _ptr(om), nf, float(c), float(width_b), float(phi_amp), int(bool(use_cutoff)),
        _ptr(acc), _ptr(evals), int(obs_lo), int(obs_hi), int(beam_lo), int(beam_hi), prec,
        0, dev.index or 0, st))


def nearest_batch(seg_origin, seg_dir, seg_e1, seg_e2, seg_len, seg_s0, seg_refl, n_segs,
                  max_seg, obs, q_obs, q_beam, device=0):
    """nearest_on_segments (kernels.py:304-349) for many (observer, beam) pairs.

    Returns an (n, 6) array: k, s, q1, q2, refl, behind (k = -1 for empty beams).
    """
    lib = _lib.load()
    n_segs = _np_in(n_segs, np.int32)
    arrs = [_np_in(a, np.float64) for a in (seg_origin, seg_dir, seg_e1, seg_e2, seg_len,
                                            seg_s0, seg_refl)]
    obs = _np_in(obs, np.float64).reshape(-1, 3)
    q_obs = _np_in(q_obs, np.int64)
    q_beam = _np_in(q_beam, np.int64)
    out = np.zeros((q_obs.shape[0], 6))
    _lib.check(lib.bf_nearest_on_segments(
        *[_ptr(a) for a in arrs], _ptr(n_segs), n_segs.shape[0], int(max_seg), _ptr(obs),
        obs.shape[0], _ptr(q_obs), _ptr(q_beam), q_obs.shape[0], _ptr(out), int(device)))
    return out


def nearest_on_segments(seg_origin, seg_dir, seg_e1, seg_e2, seg_len, seg_s0, seg_refl,
                        base, n_seg, px, py, pz):
    """Reference signature (kernels.py:304-306); evaluated on the device in fp64."""
    if n_seg <= 0:
        return -1, 0.0, 0.0, 0.0, 1.0, False
    sl = slice(int(base), int(base) + int(n_seg))
    out = nearest_batch(np.asarray(seg_origin)[sl], np.asarray(seg_dir)[sl],
                        np.asarray(seg_e1)[sl], np.asarray(seg_e2)[sl],
                        np.asarray(seg_len)[sl], np.asarray(seg_s0)[sl],
                        np.asarray(seg_refl)[sl], np.array([n_seg], np.int32), int(n_seg),
                        np.array([[px, py, pz]], float), np.zeros(1, np.int64),
                        np.zeros(1, np.int64))[0]
    return int(out[0]), float(out[1]), float(out[2]), float(out[3]), float(out[4]), bool(out[5])

#!/usr/bin/env python3
"""Generate the golden fixtures by EXECUTING the reference `beamfield` package.

Test infrastructure only.  Runs in the build container (where the read-only
reference lives at /root/reference); the GPU box never runs this script, it
only reads the committed `*.npz` outputs.

    NUMBA_CACHE_DIR=/tmp/nb python tests/golden/make_golden.py

Every case records
  * the traced PathBundle (valid rows only, fp64 bit patterns) produced by the
    reference tracer `beamtrace.trace_into` (beamtrace.py:291-306), together
    with the scene/launch parameters that produced it (tracer golden);
  * the reference `kernels.gbs_accumulate` (kernels.py:352-399) output
    `acc` (complex128) and `evals` (int64) for the stated call sequence
    (GBS golden; uncalibrated, calibration = 1.0 as in harness.cmd_bench);
  * (k, s, q1, q2, refl, behind) from the reference
    `kernels.nearest_on_segments` (kernels.py:304-349) for a deterministic
    sample of (observer, beam) pairs (nearest-segment golden).
"""

from __future__ import annotations

import os
import zlib
import pathlib
import sys

import numpy as np

REF = pathlib.Path("/root/reference/pkg/src")
OUT = pathlib.Path(__file__).resolve().parent

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
sys.path.insert(0, str(REF))

from beamfield import kernels  # noqa: E402
from beamfield.beamtrace import (Atmosphere, LaunchGrid, SourceSpec,  # noqa: E402
                                 TraceConfig, allocate_bundle,
                                 launch_directions, trace_into)
from beamfield.gbs import calibrate_phi, sum_at_observer  # noqa: E402
from beamfield.scene import make_city, make_ground_plane  # noqa: E402


def grid_points(origin, axis1, axis2, n1, n2):
    """Same ordering as config.ObserverGridSpec.points (config.py:39-46)."""
    o = np.asarray(origin, float)
    a1 = np.asarray(axis1, float)
    a2 = np.asarray(axis2, float)
    pts = (o[None, None, :] + np.arange(n1)[None, :, None] * a1[None, None, :]
           + np.arange(n2)[:, None, None] * a2[None, None, :])
    return np.ascontiguousarray(pts.reshape(-1, 3))


def trace_bundle(scene, source, grid, tcfg, atmo):
    launch = launch_directions(grid)
    c = atmo.sound_speed
    b = allocate_bundle(len(launch), launch, 0, source, tcfg, c)
    trace_into(scene, source, launch, tcfg, c, b, 0, 0, len(launch))
    return launch, b


def pack_valid(b):
    """Valid rows of the padded bundle, in (beam, segment) order."""
    rows = np.concatenate([np.arange(i * b.max_seg, i * b.max_seg + int(n))
                           for i, n in enumerate(b.n_segs)]) if b.n_segs.sum() else np.zeros(0, int)
    return dict(
        v_origin=b.seg_origin[rows], v_dir=b.seg_dir[rows], v_e1=b.seg_e1[rows],
        v_e2=b.seg_e2[rows], v_len=b.seg_len[rows], v_s0=b.seg_s0[rows],
        v_refl=b.seg_refl[rows], n_segs=b.n_segs.copy(), n_refls=b.n_refls.copy(),
        max_seg=np.int64(b.max_seg), weights=b.weights.copy(),
        gamma1=b.gamma1.copy(), gamma2=b.gamma2.copy(), c=np.float64(b.c),
        beam_param_im=np.float64(b.beam_param_im),
        amplitude_phi=np.float64(b.amplitude_phi))


def gbs(b, obs, omegas, use_cutoff, calls):
    acc = np.zeros((obs.shape[0], omegas.shape[0]), np.complex128)
    evals = np.zeros(obs.shape[0], np.int64)
    for (olo, ohi, blo, bhi) in calls:
        kernels.gbs_accumulate(b.seg_origin, b.seg_dir, b.seg_e1, b.seg_e2, b.seg_len,
                               b.seg_s0, b.seg_refl, b.n_segs, b.max_seg, b.weights,
                               obs, omegas, b.c, -b.beam_param_im, b.amplitude_phi,
                               use_cutoff, acc, evals, olo, ohi, blo, bhi)
    return acc, evals


def nearest_samples(b, obs, n_samples, seed):
    rng = np.random.default_rng(seed)
    oi = rng.integers(0, obs.shape[0], n_samples)
    bi = rng.integers(0, b.n_paths, n_samples)
    out = np.zeros((n_samples, 6))
    for j in range(n_samples):
        ns = int(b.n_segs[bi[j]])
        if ns == 0:
            out[j] = (-1, 0, 0, 0, 1, 0)
            continue
        p = obs[oi[j]]
        k, s, q1, q2, refl, behind = kernels.nearest_on_segments(
            b.seg_origin, b.seg_dir, b.seg_e1, b.seg_e2, b.seg_len, b.seg_s0, b.seg_refl,
            int(bi[j]) * b.max_seg, ns, p[0], p[1], p[2])
        out[j] = (k, s, q1, q2, refl, float(behind))
    return dict(ns_obs=oi, ns_beam=bi, ns_k=out[:, 0].astype(np.int64), ns_s=out[:, 1],
                ns_q1=out[:, 2], ns_q2=out[:, 3], ns_refl=out[:, 4],
                ns_behind=out[:, 5].astype(np.int8))


def make_case(name, scene_kind, scene_args, src, freqs, im_b, n_theta, n_phi,
              n_steps, r_max, grid, use_cutoff=True, calls=None, n_samples=4000):
    atmo = Atmosphere(20.0)
    scene = make_ground_plane(*scene_args) if scene_kind == "plane" else make_city(*scene_args)
    source = SourceSpec(position=np.asarray(src, float), frequencies=tuple(freqs),
                        beam_param_im=im_b)
    lg = LaunchGrid(0.0, 180.0, 0.0, 360.0, n_theta, n_phi)
    tcfg = TraceConfig(n_steps=n_steps, dt=1e-4, r_max=r_max)
    launch, b = trace_bundle(scene, source, lg, tcfg, atmo)
    obs = grid_points(*grid)
    omegas = source.omegas
    if calls is None:
        calls = [(0, obs.shape[0], 0, b.n_paths)]
    acc, evals = gbs(b, obs, omegas, use_cutoff, calls)
    d = pack_valid(b)
    d.update(nearest_samples(b, obs, n_samples, seed=zlib.crc32(name.encode())))
    d.update(
        scene_kind=np.array(scene_kind), scene_args=np.asarray(scene_args, float),
        src=np.asarray(src, float), freqs=np.asarray(freqs, float), im_b=np.float64(im_b),
        n_theta=np.int64(n_theta), n_phi=np.int64(n_phi), n_steps=np.int64(n_steps),
        dt=np.float64(1e-4), r_max=np.int64(r_max),
        grid_origin=np.asarray(grid[0], float), grid_axis1=np.asarray(grid[1], float),
        grid_axis2=np.asarray(grid[2], float), grid_n=np.asarray(grid[3:], np.int64),
        obs=obs, omegas=omegas, use_cutoff=np.int8(use_cutoff),
        calls=np.asarray(calls, np.int64), acc=acc, evals=evals,
        launch_dirs=launch.directions, launch_e1=launch.e1, launch_e2=launch.e2,
        launch_weights=launch.weights, scene_v0=scene.v0, scene_v1=scene.v1,
        scene_v2=scene.v2)
    np.savez_compressed(OUT / f"{name}.npz", **d)
    nb = b.n_paths
    print(f"{name}: beams={nb} segs={int(b.n_segs.sum())} obs={obs.shape[0]} "
          f"F={len(freqs)} evals={int(evals.sum())} |acc|max={np.abs(acc).max():.3e}")


def make_calibration():
    """calibrate_phi on a 64x64 full-sphere free-field bundle, source at origin."""
    from beamfield.scene import _assemble
    atmo = Atmosphere(20.0)
    empty = _assemble(np.zeros((0, 3)), np.zeros((0, 3)), np.zeros((0, 3)), [], [])
    source = SourceSpec(position=np.zeros(3), frequencies=(500.0,), beam_param_im=-12.0)
    lg = LaunchGrid(0.0, 180.0, 0.0, 360.0, 64, 64)
    tcfg = TraceConfig(n_steps=2000, dt=1e-4, r_max=4)
    _, b = trace_bundle(empty, source, lg, tcfg, atmo)
    scale = calibrate_phi(b, atmo, source)
    probe = np.array([10.0, 0.0, 0.0])
    p = sum_at_observer(probe, b, source.omegas[0], atmo, source)
    d = pack_valid(b)
    d.update(scale=np.float64(scale), probe=probe, probe_p=np.complex128(p),
             omegas=source.omegas, src=np.zeros(3))
    np.savez_compressed(OUT / "calibration_origin.npz", **d)
    print(f"calibration_origin: scale={scale!r} p={p!r}")


def main():
    # Config 1: open plane, 2048 rays, 128x128 receivers, full field.
    make_case("cfg1_open_plane", "plane", (1000.0,), (0.0, 0.0, 5.0), (500.0,), -12.0,
              32, 64, 2000, 4, ((-32.0, -32.0, 1.5), (0.5, 0, 0), (0, 0.5, 0), 128, 128))
    # Config 1, chunked call sequence: two beam chunks, the second on an observer sub-range.
    make_case("cfg1_chunked", "plane", (1000.0,), (0.0, 0.0, 5.0), (500.0,), -12.0,
              32, 64, 2000, 4, ((-32.0, -32.0, 1.5), (0.5, 0, 0), (0, 0.5, 0), 64, 64),
              calls=[(0, 4096, 0, 1000), (100, 3000, 1000, 2048), (3000, 4096, 1000, 1500)],
              n_samples=200)
    # Config 3 shape (city 5x10, street source), strided receivers, 2048 rays.
    make_case("city_street", "city", (5, 10, 40.0, 20.0, 300.0), (20.0, 0.0, 2.0), (125.0,),
              -10.0, 32, 64, 5000, 8, ((-125.0, -125.0, 1.8), (4.0, 0, 0), (0, 4.0, 0), 64, 64))
    # Same scene, no cutoff.
    make_case("city_street_nocut", "city", (5, 10, 40.0, 20.0, 300.0), (20.0, 0.0, 2.0),
              (125.0,), -10.0, 32, 32, 5000, 8,
              ((-60.0, -60.0, 1.8), (2.0, 0, 0), (0, 2.0, 0), 48, 48), use_cutoff=False,
              n_samples=1000)
    # Source next to a building corner, F = 5 (table2 frequencies), many corner ties.
    make_case("city_corner_f5", "city", (6, 6, 40.0, 20.0, 250.0), (-9.5, -9.5, 2.0),
              (63.0, 125.0, 250.0, 500.0, 1000.0), -10.0, 32, 64, 5000, 8,
              ((-60.0, -60.0, 1.8), (2.0, 0, 0), (0, 2.0, 0), 64, 64))
    # Paper beam parameter (im_b = -45874): the cutoff never fires.
    make_case("open_paper_imb", "plane", (1000.0,), (0.0, 0.0, 5.0), (500.0,), -45874.0,
              32, 32, 2000, 4, ((-16.0, -16.0, 1.5), (1.0, 0, 0), (0, 1.0, 0), 32, 32),
              n_samples=500)
    make_calibration()


if __name__ == "__main__":
    main()

#!/usr/bin/env python3
"""Config 4 of the survey through run_pipeline on one B200: dense city (500 buildings,
5002 triangles), 4M rays traced and summed in 1M-ray chunks (the memory budget forces
the chunk loop), 2000 x 2000 receivers at 0.4 m, 125 Hz, im_b -10, uncalibrated.
Prints phase timings, pairs/s and parity against the C oracle on a strided receiver
sample (all 4M beams, traced once more on the device for the oracle's bundle).

    python scripts/cfg4_pipeline.py [--sample 400]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sample", type=int, default=400)
    args = ap.parse_args()
    import torch

    import oracle
    from paper_2501_13382_b200 import (Atmosphere, ExecPlan, LaunchGrid, ObserverSet,
                                       SourceSpec, TraceConfig, engine, make_city, parallel)
    from paper_2501_13382_b200.beamtrace import launch_directions
    sc = make_city(20, 25, 40.0, 20.0, 600.0)
    src = SourceSpec(position=np.array([0.0, 20.0, 2.0]), frequencies=(125.0,),
                     beam_param_im=-10.0)
    grid = LaunchGrid(0.0, 180.0, 0.0, 360.0, 2000, 2000)
    cfg = TraceConfig(5000, 1e-4, 8)
    atm = Atmosphere(20.0)
    x = -400.0 + 0.4 * np.arange(2000)
    X, Y = np.meshgrid(x, x, indexing="xy")
    pts = np.ascontiguousarray(np.stack([X.ravel(), Y.ravel(), np.full(X.size, 1.8)], 1))
    per_ray = 9 * 120
    plan = ExecPlan(memory_budget=1048576 * per_ray, per_ray_bytes=per_ray)
    parallel.run_pipeline(sc, src, LaunchGrid(0.0, 180.0, 0.0, 360.0, 40, 50), cfg,
                          ObserverSet(pts[:1024]), ExecPlan(), atm, calibration=1.0)  # warm-up
    t0 = time.perf_counter()
    res, t = parallel.run_pipeline(sc, src, grid, cfg, ObserverSet(pts), plan, atm,
                                   calibration=1.0)
    wall = time.perf_counter() - t0
    n_b, n_r = 4_000_000, pts.shape[0]
    out = {"config": "cfg4 (dense city, 4M rays in 4 chunks, 4M receivers, 125 Hz)",
           "chunks": 4, "rt_s": t.rt_seconds, "gbs_s": t.gbs_seconds, "wall_s": wall,
           "pairs_per_s_gbs": n_b * n_r / t.gbs_seconds, "evaluations": t.gbs_evaluations}
    # parity on a strided receiver sample: the oracle over the same (device-traced) bundle
    dev = torch.device("cuda", 0)
    launch = launch_directions(grid)
    tr = engine.trace_device_rows(engine.DeviceScene.from_scene(sc, dev), src, launch, cfg,
                                  atm.sound_speed, 0, len(launch), dev)
    hb = tr["bundle"].to_host()
    idx = np.linspace(0, n_r - 1, args.sample).astype(np.int64)
    obs = np.ascontiguousarray(pts[idx])
    ref = np.zeros((idx.size, 1), np.complex128)
    rev = np.zeros(idx.size, np.int64)
    t1 = time.perf_counter()
    oracle.gbs_accumulate(hb.seg_origin, hb.seg_dir, hb.seg_e1, hb.seg_e2, hb.seg_len,
                          hb.seg_s0, hb.seg_refl, hb.n_segs, hb.max_seg, hb.weights, obs,
                          src.omegas, atm.sound_speed, -src.beam_param_im,
                          src.amplitude_phi, True, ref, rev, 0, idx.size, 0, n_b,
                          threads=len(os.sched_getaffinity(0)))
    cpu_s = time.perf_counter() - t1
    got = res.pressure[idx]
    m = np.abs(ref) > 0
    strong = m & (20 * np.log10(np.maximum(np.abs(ref), 1e-300) / np.abs(ref).max()) > -60)
    out["parity"] = {"receivers": int(idx.size),
                     "rel_l2": float(np.linalg.norm(got - ref) / np.linalg.norm(ref)),
                     "max_dtl_db_above_-60dB": float(np.max(np.abs(20 * np.log10(
                         np.abs(got[strong]) / np.abs(ref[strong]))))),
                     "cpu_pairs_per_s": n_b * idx.size / cpu_s,
                     "cpu_threads": len(os.sched_getaffinity(0))}
    print(json.dumps(out))


if __name__ == "__main__":
    main()

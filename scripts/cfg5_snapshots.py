#!/usr/bin/env python3
"""Config 5 of the survey on one B200: drone noise map, 16 moving-source snapshots
(-300 + 40k, 20, 50), k = 0..15, each 1000 x 1000 rays over the dense city (500
buildings), 2000 x 1000 receivers at 0.5 m, 125 Hz, im_b -10, uncalibrated; per-snapshot
fields and the energy-mean SPL map through run_snapshots.  Parity of snapshot 0 and 15
against the C oracle on a strided receiver sample.

    python scripts/cfg5_snapshots.py [--sample 300]
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
    ap.add_argument("--sample", type=int, default=300)
    args = ap.parse_args()
    import torch

    import oracle
    from paper_2501_13382_b200 import (Atmosphere, ExecPlan, LaunchGrid, ObserverSet,
                                       SourceSpec, TraceConfig, engine, make_city, parallel)
    from paper_2501_13382_b200.beamtrace import launch_directions
    sc = make_city(20, 25, 40.0, 20.0, 600.0)
    srcs = [SourceSpec(position=np.array([-300.0 + 40.0 * k, 20.0, 50.0]), frequencies=(125.0,),
                       beam_param_im=-10.0) for k in range(16)]
    grid = LaunchGrid(0.0, 180.0, 0.0, 360.0, 1000, 1000)
    cfg = TraceConfig(5000, 1e-4, 8)
    atm = Atmosphere(20.0)
    x = -500.0 + 0.5 * np.arange(2000)
    y = -250.0 + 0.5 * np.arange(1000)
    X, Y = np.meshgrid(x, y, indexing="xy")
    pts = np.ascontiguousarray(np.stack([X.ravel(), Y.ravel(), np.full(X.size, 1.8)], 1))
    parallel.run_pipeline(sc, srcs[0], LaunchGrid(0.0, 180.0, 0.0, 360.0, 40, 50), cfg,
                          ObserverSet(pts[:1024]), ExecPlan(), atm, calibration=1.0)  # warm-up
    t0 = time.perf_counter()
    fields, spl_mean, tims = parallel.run_snapshots(sc, srcs, grid, cfg, ObserverSet(pts),
                                                    ExecPlan(), atm, calibration=1.0)
    wall = time.perf_counter() - t0
    n_b, n_r = 1_000_000, pts.shape[0]
    gbs = sum(t.gbs_seconds for t in tims)
    out = {"config": "cfg5 (16 snapshots x 1M rays, dense city, 2M receivers, 125 Hz)",
           "rt_s": sum(t.rt_seconds for t in tims), "gbs_s": gbs, "wall_s": wall,
           "pairs_per_s_gbs": 16 * n_b * n_r / gbs,
           "spl_mean_db_range": [float(np.nanmin(spl_mean[np.isfinite(spl_mean)])),
                                 float(np.nanmax(spl_mean))]}
    dev = torch.device("cuda", 0)
    launch = launch_directions(grid)
    dscene = engine.DeviceScene.from_scene(sc, dev)
    idx = np.linspace(0, n_r - 1, args.sample).astype(np.int64)
    obs = np.ascontiguousarray(pts[idx])
    par = {}
    for k in (0, 15):
        tr = engine.trace_device_rows(dscene, srcs[k], launch, cfg, atm.sound_speed, 0,
                                      len(launch), dev)
        hb = tr["bundle"].to_host()
        ref = np.zeros((idx.size, 1), np.complex128)
        rev = np.zeros(idx.size, np.int64)
        oracle.gbs_accumulate(hb.seg_origin, hb.seg_dir, hb.seg_e1, hb.seg_e2, hb.seg_len,
                              hb.seg_s0, hb.seg_refl, hb.n_segs, hb.max_seg, hb.weights, obs,
                              srcs[k].omegas, atm.sound_speed, -srcs[k].beam_param_im,
                              srcs[k].amplitude_phi, True, ref, rev, 0, idx.size, 0, n_b,
                              threads=len(os.sched_getaffinity(0)))
        got = fields[k].pressure[idx]
        m = np.abs(ref) > 0
        strong = m & (20 * np.log10(np.maximum(np.abs(ref), 1e-300) / np.abs(ref).max()) > -60)
        par[f"snapshot_{k}"] = {
            "rel_l2": float(np.linalg.norm(got - ref) / np.linalg.norm(ref)),
            "max_dtl_db_above_-60dB": float(np.max(np.abs(20 * np.log10(
                np.abs(got[strong]) / np.abs(ref[strong])))))}
    out["parity"] = par
    print(json.dumps(out))


if __name__ == "__main__":
    main()

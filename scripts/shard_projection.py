"""Per-rank cost of the receiver-tile partition, measured on ONE GPU.

For W in (1, 2, 4, 8) and every rank r < W this times exactly the work rank r does
under `torchrun bench.py --gpus W` (its round-robin tiles, presorted, all beams), one
rank after another on the same device, and prints max / mean per-rank time and the
projected strong-scaling efficiency T1 / (W * max_r T_r).  The gather to rank 0
(16 B x receivers over NVLink, well under 1 ms) is not included.  This is a
projection from single-GPU timings, not a multi-GPU measurement.

    python scripts/shard_projection.py [--config cfg3] [--reps 3] [--out file.json]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--worlds", default="1,2,4,8")
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    import torch

    import bench
    from paper_2501_13382_b200 import _lib, engine, shard
    _lib.set_kernel_timing(True)  # kernel_ms below
    dev = torch.device("cuda", 0)
    cfg = bench.CONFIGS[args.config]
    sc, src, launch, tcfg, c, obs_np = bench.make_inputs(cfg)
    omegas, nf, width_b = src.omegas, src.omegas.shape[0], -src.beam_param_im
    dscene = engine.DeviceScene.from_scene(sc, dev)
    bundle = engine.trace_device_rows(dscene, src, launch, tcfg, c, 0, len(launch), dev)["bundle"]
    obs_all = torch.from_numpy(obs_np).to(dev)
    order = shard.tile_order(obs_all)
    flush = torch.zeros(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    def time_rank(rank, world):
        obs = obs_all.index_select(0, shard.rank_indices(order, rank, world)).contiguous()
        acc = torch.zeros((obs.shape[0], nf), dtype=torch.complex128, device=dev)
        ev = torch.zeros(obs.shape[0], dtype=torch.int64, device=dev)
        best, kern = float("inf"), float("inf")
        for i in range(args.reps + 1):
            flush.add_(1.0)  # 256 MiB write > 126 MB L2
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            acc.zero_()
            ev.zero_()
            e0.record(stream)
            engine.accumulate(bundle, obs, omegas, width_b, True, acc, ev, stream=stream,
                              presorted=True)
            e1.record(stream)
            e1.synchronize()
            if i > 0:  # first call warms the workspaces
                best = min(best, e0.elapsed_time(e1))
                kern = min(kern, _lib.last_stats()["kernel_ms"])
        return best, kern

    out = {"config": args.config, "receivers": int(obs_all.shape[0]), "beams": bundle.n_paths,
           "note": "per-rank shares timed one after another on one B200; projection only",
           "worlds": {}}
    t1 = None
    for w in map(int, args.worlds.split(",")):
        per = [time_rank(r, w) for r in range(w)]
        ms = [p[0] for p in per]
        mx, mean = max(ms), sum(ms) / len(ms)
        if w == 1:
            t1 = mx
        row = {"rank_ms": [round(x, 3) for x in ms], "rank_kernel_ms": [round(p[1], 3) for p in per],
               "max_ms": round(mx, 3), "mean_ms": round(mean, 3),
               "imbalance_max_over_mean": round(mx / mean, 4)}
        if t1:
            row["projected_efficiency"] = round(t1 / (w * mx), 4)
        out["worlds"][str(w)] = row
        print(w, json.dumps(row), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()

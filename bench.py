#!/usr/bin/env python3
"""GBS stage benchmark: beam-receiver evaluations/s on B200 vs the CPU reference path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg3] [--impl ours|reference]

A step is one pass of the hot path -- kernels.gbs_accumulate over ALL beams x
ALL receivers of the workload -- on synthetic inputs traced
on the device from the named scene.  Default workload: config 3 (city block,
50 buildings, 500k rays, 1000x1000 receivers, 125 Hz).  `value` = N_beams x
N_receivers / device time per step (max over ranks), inputs resident in HBM;
`e2e` = the same metric through the reference-facing host-buffer call
(kernels.gbs_accumulate on pageable numpy arrays -> bf_gbs_accumulate: host
packing, H2D, kernels and D2H inside the timed region).  With N > 1 each rank
sums its receiver tiles (shard.py) and the field is gathered to rank 0 inside
the timed region (strong scaling: the problem is fixed).  `--gpus N` without
torchrun re-launches itself under torch.distributed.run with N ranks.

The same JSON line carries two more measurements of the same metric:
`north_star_shape` (config 4: dense city, 4M rays x 4M receivers, the
north-star shape, with its own roofline / e2e / CPU baseline / parity sample)
and `fp64_oracle_mode` (the headline workload in the fp64 oracle mode).

`--impl reference` times the reference algorithm's CPU implementation (the C
oracle restatement in oracle/, bit-exact with the reference) on all host
threads on a bounded receiver sample of the same workload; rank 0 only.
"""
from __future__ import annotations

import argparse
import glob
import json
import os
import socket
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "beam-receiver evals/sec and GBS wall time at 1/2/4/8 B200 vs CPU ref (cores stated)"

CITY3 = (5, 10, 40.0, 20.0, 300.0)
CITY4 = (20, 25, 40.0, 20.0, 600.0)
CONFIGS = {
    "cfg1": dict(desc="open plane, 2k rays, 128x128 receivers (config 1)", scene="plane",
                 scene_args=(1000.0,), src=(0.0, 0.0, 5.0), freqs=(500.0,), im_b=-12.0,
                 n_theta=32, n_phi=64, n_steps=2000, r_max=4,
                 grid=((-32.0, -32.0, 1.5), 0.5, 128, 128)),
    "cfg2": dict(desc="open plane, 100k rays, 1024x1024 receivers (config 2)", scene="plane",
                 scene_args=(2000.0,), src=(0.0, 0.0, 10.0), freqs=(500.0,), im_b=-10.0,
                 n_theta=250, n_phi=400, n_steps=8000, r_max=4,
                 grid=((-256.0, -256.0, 1.5), 0.5, 1024, 1024)),
    "cfg3": dict(desc="city block, 50 buildings, 500k rays, 1000x1000 receivers (config 3)",
                 scene="city", scene_args=CITY3, src=(20.0, 0.0, 2.0),
                 freqs=(125.0,), im_b=-10.0, n_theta=500, n_phi=1000, n_steps=5000, r_max=8,
                 grid=((-125.0, -125.0, 1.8), 0.25, 1000, 1000)),
    "cfg4": dict(desc="dense city, 500 buildings, 4M rays, 2000x2000 receivers (config 4)",
                 scene="city", scene_args=CITY4, src=(0.0, 20.0, 2.0), freqs=(125.0,),
                 im_b=-10.0, n_theta=2000, n_phi=2000, n_steps=5000, r_max=8,
                 grid=((-400.0, -400.0, 1.8), 0.4, 2000, 2000)),
    # config-3 variant with the five-frequency set of the survey (63-1000 Hz)
    "cfg3s_f5": dict(desc="city block, 50 buildings, 20k rays, 1000x1000 receivers, F=5 "
                          "(63-1000 Hz variant)", scene="city", scene_args=CITY3,
                     src=(20.0, 0.0, 2.0), freqs=(63.0, 125.0, 250.0, 500.0, 1000.0), im_b=-10.0,
                     n_theta=100, n_phi=200, n_steps=5000, r_max=8,
                     grid=((-125.0, -125.0, 1.8), 0.25, 1000, 1000)),
    # config-3 variant with the paper's beam parameter (im_b = -45874): the cutoff never
    # fires, so every non-behind pair is evaluated (no work-list culling)
    "cfg3s_pb": dict(desc="city block, 50 buildings, 20k rays, 1000x1000 receivers, "
                          "im_b=-45874 (paper beam parameter variant)", scene="city",
                     scene_args=CITY3, src=(20.0, 0.0, 2.0),
                     freqs=(125.0,), im_b=-45874.0, n_theta=100, n_phi=200, n_steps=5000,
                     r_max=8, grid=((-125.0, -125.0, 1.8), 0.25, 1000, 1000)),
    # profiling variant of config 3: same scene/receivers, 20k rays (ncu replays stay short)
    "cfg3s": dict(desc="city block, 50 buildings, 20k rays, 1000x1000 receivers (cfg3 profile "
                       "variant)", scene="city", scene_args=CITY3,
                  src=(20.0, 0.0, 2.0), freqs=(125.0,), im_b=-10.0, n_theta=100, n_phi=200,
                  n_steps=5000, r_max=8, grid=((-125.0, -125.0, 1.8), 0.25, 1000, 1000)),
}


def grid_points(origin, spacing, n1, n2):
    """config.ObserverGridSpec.points ordering (config.py:39-46): j*n1 + i."""
    o = np.asarray(origin, float)
    a1 = np.array([spacing, 0.0, 0.0])
    a2 = np.array([0.0, spacing, 0.0])
    pts = (o[None, None, :] + np.arange(n1)[None, :, None] * a1[None, None, :]
           + np.arange(n2)[:, None, None] * a2[None, None, :])
    return np.ascontiguousarray(pts.reshape(-1, 3))


def make_inputs(cfg):
    from paper_2501_13382_b200 import beamtrace, scene
    sc = (scene.make_ground_plane(*cfg["scene_args"]) if cfg["scene"] == "plane"
          else scene.make_city(*cfg["scene_args"]))
    src = beamtrace.SourceSpec(position=np.array(cfg["src"]), frequencies=cfg["freqs"],
                               beam_param_im=cfg["im_b"])
    launch = beamtrace.launch_directions(beamtrace.LaunchGrid(
        0.0, 180.0, 0.0, 360.0, cfg["n_theta"], cfg["n_phi"]))
    tcfg = beamtrace.TraceConfig(cfg["n_steps"], 1e-4, cfg["r_max"])
    c = beamtrace.Atmosphere(20.0).sound_speed
    obs = grid_points(*cfg["grid"])
    return sc, src, launch, tcfg, c, obs


def cpu_threads():
    return len(os.sched_getaffinity(0))


def time_oracle_sample(bundle, obs, omegas, c, width_b, phi, budget_s, threads):
    """Oracle (C port of kernels.gbs_accumulate) on a strided receiver subset sized
    for ~budget_s seconds of all-thread CPU work.  Returns (pairs/s, sample, idx, acc)."""
    import oracle
    nb = bundle["n_segs"].shape[0]
    args = [bundle[k] for k in ("seg_origin", "seg_dir", "seg_e1", "seg_e2", "seg_len",
                                "seg_s0", "seg_refl")]

    def run(idx):
        o = np.ascontiguousarray(obs[idx])
        acc = np.zeros((o.shape[0], omegas.shape[0]), np.complex128)
        ev = np.zeros(o.shape[0], np.int64)
        t0 = time.perf_counter()
        oracle.gbs_accumulate(*args, bundle["n_segs"], bundle["max_seg"], bundle["weights"], o,
                              omegas, c, width_b, phi, True, acc, ev, 0, o.shape[0], 0, nb,
                              threads=threads)
        return time.perf_counter() - t0, acc, ev

    probe = np.linspace(0, obs.shape[0] - 1, max(threads, 16)).astype(np.int64)
    dt, _, _ = run(probe)
    rate = probe.size * nb / max(dt, 1e-6)
    n_sub = int(np.clip(rate * budget_s / nb, threads, obs.shape[0]))
    stride = max(1, obs.shape[0] // n_sub)
    idx = np.arange(0, obs.shape[0], stride)
    dt, acc, ev = run(idx)
    sample = (f"all {nb} beams x {idx.size} receivers (every {stride}th of {obs.shape[0]}), "
              f"{threads} threads, {dt:.1f} s")
    return idx.size * nb / dt, sample, idx, acc, ev, dt


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out = ""
            self.out = out
        return False

    def summary(self):
        if self.proc is None or not getattr(self, "out", ""):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        rows = [r.split(",") for r in self.out.strip().splitlines() if r.count(",") >= 6]
        sm = [float(r[0]) for r in rows if r[0].strip().replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4)
                          if r[3 + i].strip().lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows)}


def flop_model(total_pairs_segs, p_nb, evals, nf):
    """Algorithmic FLOP / MUFU of SURVEY.md 8(d) for the pairs evaluated."""
    flop = 19.0 * total_pairs_segs + (16.0 + 5.0 * nf) * p_nb + 22.0 * evals
    mufu = p_nb + 3.0 * evals
    return flop, mufu


class Dist:
    """World of the run: NCCL ranks (one GPU each), or gloo ranks sharing cuda:0
    (BF_BENCH_SHARE_DEVICE=1, a functional check of the multi-rank path)."""

    def __init__(self, gpus):
        import torch
        import torch.distributed as dist
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        if self.world != gpus:
            raise SystemExit(f"bench.py: --gpus {gpus} but WORLD_SIZE={self.world}")
        self.share = os.environ.get("BF_BENCH_SHARE_DEVICE") == "1"
        if self.share:
            self.local = 0
        if self.world > 1:
            if self.share:
                dist.init_process_group("gloo")
            else:
                os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator lines in the log
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
        self.dev = torch.device("cuda", self.local)
        self.red_dev = torch.device("cpu") if self.share else self.dev
        torch.cuda.set_device(self.dev)

    def barrier(self):
        import torch.distributed as dist
        if self.world > 1:
            dist.barrier()

    def max(self, *vals):
        import torch
        import torch.distributed as dist
        t = torch.tensor([float(v) for v in vals], dtype=torch.float64, device=self.red_dev)
        if self.world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return [float(x) for x in t]

    def close(self):
        import torch.distributed as dist
        if self.world > 1:
            dist.barrier()
            dist.destroy_process_group()


def measure(D, name, precision, steps, warmup, peaks, cpu_budget, e2e_steps, cpu_sample=None):
    """One workload at one precision on all ranks; the result dict on rank 0."""
    import torch

    from paper_2501_13382_b200 import _lib, engine, kernels, shard
    cfg = CONFIGS[name]
    sc, src, launch, tcfg, c, obs_np = make_inputs(cfg)
    omegas = src.omegas
    nf = omegas.shape[0]
    width_b = -src.beam_param_im
    dev = D.dev

    # ---- inputs: traced on the device by the sm_100a tracer (every rank), in HBM
    dscene = engine.DeviceScene.from_scene(sc, dev)
    tr = engine.trace_device_rows(dscene, src, launch, tcfg, c, 0, len(launch), dev)
    bundle = tr["bundle"]
    torch.cuda.synchronize()
    nb = bundle.n_paths
    sum_segs = int(bundle.n_segs.sum().item())
    obs_all = torch.from_numpy(obs_np).to(dev)
    n_total = obs_all.shape[0]
    order = shard.tile_order(obs_all)
    mine = shard.rank_indices(order, D.rank, D.world)
    obs = obs_all.index_select(0, mine).contiguous()
    n_loc = obs.shape[0]
    acc = torch.zeros((n_loc, nf), dtype=torch.complex128, device=dev)
    evals = torch.zeros(n_loc, dtype=torch.int64, device=dev)
    flush = torch.zeros(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)
    # the gather's index plan is part of the partition, built once (not per step)
    plan = shard.GatherPlan(order, D.world, n_total) if D.world > 1 else None

    def step():
        acc.zero_()
        evals.zero_()
        engine.accumulate(bundle, obs, omegas, width_b, True, acc, evals, precision=precision,
                          stream=stream, presorted=True)
        if D.world > 1:
            shard.gather_field(acc, evals, order, D.rank, D.world, n_total, plan=plan)

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()

    # ---- timed region (device events per step; L2 flushed between steps).  The engine's
    #      kernel timing (kernel_ms, the roofline's denominator) costs ~10 us of graph-node
    #      latency per call: recorded inside the timed steps only for calls of >= 2^28 pairs
    #      (>= ~1 ms), else in separate steps after the timed region
    # (the same decision on every rank: the extra steps below include the field gather)
    inline_timing = float(nb) * float(n_total) / D.world >= 2.0 ** 28
    _lib.set_kernel_timing(inline_timing)
    D.barrier()
    torch.cuda.synchronize()
    launches0 = _lib.launch_count()
    ms_steps, kern_ms, stats = [], [], []
    with ClockSampler(D.local) as clk:
        for _ in range(steps):
            flush.add_(1.0)  # 256 MiB write > 126 MB L2
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step()
            e1.record(stream)
            e1.synchronize()
            ms_steps.append(e0.elapsed_time(e1))
            st = _lib.last_stats()
            kern_ms.append(st["kernel_ms"])
            stats.append(st)
        torch.cuda.synchronize()
    launches = _lib.launch_count() - launches0
    if not inline_timing:
        _lib.set_kernel_timing(True)
        kern_ms = []
        for _ in range(max(3, min(steps, 10))):
            flush.add_(1.0)
            step()
            torch.cuda.synchronize()
            kern_ms.append(_lib.last_stats()["kernel_ms"])
    _lib.set_kernel_timing(False)
    D.barrier()
    ms_max, kern_max = D.max(np.mean(ms_steps), np.mean(kern_ms))
    pairs = float(nb) * float(n_total)
    value = pairs / (ms_max / 1e3)

    # ---- e2e: reference-facing host-buffer call on PAGEABLE numpy arrays
    hb = {k: getattr(bundle, k).cpu().numpy().copy() for k in engine.SEG_FIELDS + (
        "n_segs", "weights")}
    obs_h = obs.cpu().numpy().copy()
    acc_h = np.zeros((n_loc, nf), np.complex128)
    ev_h = np.zeros(n_loc, np.int64)

    def e2e_step():
        kernels.gbs_accumulate(hb["seg_origin"], hb["seg_dir"], hb["seg_e1"],
                               hb["seg_e2"], hb["seg_len"], hb["seg_s0"], hb["seg_refl"],
                               hb["n_segs"], bundle.max_seg, hb["weights"], obs_h, omegas, c,
                               width_b, src.amplitude_phi, True, acc_h, ev_h, 0, n_loc, 0, nb,
                               precision=precision, device=D.local)

    e2e_step()
    e2e_same = bool(np.array_equal(acc_h, acc.cpu().numpy()))
    e2e_t = []
    for _ in range(e2e_steps):
        acc_h[...] = 0  # the caller's fresh field (not part of the call)
        ev_h[...] = 0
        D.barrier()
        t0 = time.perf_counter()
        e2e_step()
        e2e_t.append(time.perf_counter() - t0)
    (e2e_s,) = D.max(np.mean(e2e_t))
    rows = int(bundle.n_segs.sum().item())
    if precision == "fp32":  # compact rows: o, d, len, s0 (fp64) + amplitude (fp32)
        h2d = rows * 68 + nb * 8 + n_loc * (24 + 16 * nf + 8)
    else:  # padded fp64 rows incl. the frames
        h2d = nb * bundle.max_seg * 120 + nb * 12 + n_loc * (24 + 16 * nf + 8)
    d2h = n_loc * (16 * nf + 8)

    out = None
    if D.rank == 0:
        st = stats[-1]
        ev_sum = int(evals.sum().item())
        p_nb = st["nonbehind_pairs"]
        # FLOP model over the pairs of the tight work list the kernel walks
        # (bit-exact, oracle-pinned); the a9 list and the evaluated items are reported too
        flop, mufu = flop_model(float(st["tight_pair_segs"]), p_nb, ev_sum, nf)
        flop_a9, _ = flop_model(float(st["candidate_pair_segs"]), p_nb, ev_sum, nf)
        flop_live, _ = flop_model(float(st["live_pair_segs"]), p_nb, ev_sum, nf)
        kernel_s = kern_max / 1e3
        if precision == "fp64":
            # oracle mode: dense kernel, no work list or kernel statistics -> FLOP model
            # over all pairs (segment scan + evaluations), timed by the step
            flop = flop_a9 = flop_live = 19.0 * n_loc * sum_segs + 22.0 * ev_sum
            mufu = 3.0 * ev_sum
            kernel_s = ms_max / 1e3
        traffic = None  # DRAM bytes of the summation kernel from the committed ncu capture
        for tf in sorted(glob.glob(os.path.join(ROOT, "profiles", "round*", "ncu_*_traffic.json"))):
            with open(tf) as fh:
                tj = json.load(fh)
            if tj.get("config") == name and D.world == 1 and precision == "fp32":
                traffic = tj["dram_read_bytes"] + tj["dram_write_bytes"]
        ach = flop / kernel_s / 1e12
        peak = peaks["fp32_tflops"]
        out = {
            "metric": METRIC, "value": value, "unit": "beam-receiver evals/s",
            "n_gpus": D.world, "steps": steps, "warmup": warmup, "ms_per_step": ms_max,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32" if precision == "fp32" else "f64", "data": "synthetic",
            "config": {"workload": f"{name}: {cfg['desc']}", "beams": nb,
                       "receivers": n_total, "segments": sum_segs, "max_seg": bundle.max_seg,
                       "freqs_hz": list(cfg["freqs"]), "im_b": cfg["im_b"],
                       "precision": precision,
                       "parallelism": f"receiver-tiles x{D.world}" + (
                           " (ranks share cuda:0, gloo)" if D.share else ""),
                       "l2": "flushed (256 MiB write) between timed steps",
                       "inputs": "traced on device by the sm_100a tracer (bit-exact vs "
                                 "reference), on every rank, before the timed region"},
            "gbs_wall_s": ms_max / 1e3,
            "e2e": {"value": pairs / e2e_s, "unit": "beam-receiver evals/s",
                    "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                    "seconds_per_step": e2e_s, "steps": e2e_steps,
                    "equals_device_result_bitwise": e2e_same,
                    "path": "kernels.gbs_accumulate(pageable numpy) -> bf_gbs_accumulate "
                            "(host threads pack compact rows into pinned staging, beam groups "
                            "streamed); per rank, max over ranks, no field gather"},
            "gpu_launches": int(launches),
            "roofline": {"bound": "fp32", "achieved": ach, "peak": peak, "unit": "TFLOP/s",
                         "frac": ach / peak, "traffic": traffic,
                         "work_list": "tight (tile, beam) list walked by the kernel, "
                                      f"tiles of {shard.tile_size()} receivers",
                         "frac_a9_list": flop_a9 / kernel_s / 1e12 / peak,
                         "frac_evaluated_items": flop_live / kernel_s / 1e12 / peak,
                         "traffic_unit": "DRAM bytes per launch (ncu --set full, committed "
                                         "profile of this config)" if traffic else None,
                         "peak_source": peaks["source"],
                         "kernel": "gbs_fp32_kernel" if precision == "fp32" else
                                   "gbs_fp64_kernel (oracle mode, dense; FP32 peak as a "
                                   "common yardstick)",
                         "kernel_ms": kernel_s * 1e3,
                         "flop_per_launch": flop, "mufu_per_launch": mufu,
                         "mufu_tops": mufu / kernel_s / 1e12,
                         "mufu_peak_tops": peaks["mufu_tops"],
                         "mufu_frac": mufu / kernel_s / 1e12 / peaks["mufu_tops"],
                         "algorithmic_model": "SURVEY.md 8(d): 19*sum over work-list pairs of "
                                              "n_segs + (16+5F)*P_nb + 22*E FLOP; P_nb + 3E "
                                              "MUFU",
                         "nonbehind_pairs": p_nb, "evaluations": ev_sum,
                         "tie_pairs": st["tie_pairs"], "patch_beams": st["patch_beams"],
                         "candidate_pairs_a9": st["candidate_pairs"],
                         "candidate_pairs_tight": st["tight_pairs"],
                         "evaluated_item_pairs": st["live_pairs"],
                         "dense_pairs": int(nb) * int(n_loc)},
            "clocks": clk.summary(),
        }
    if D.world == 1 and cpu_budget > 0:
        acc_gpu = acc.cpu().numpy()
        ev_gpu = evals.cpu().numpy()
        order_np = order.cpu().numpy()
        if cpu_sample is None:
            hbf = dict(hb, max_seg=bundle.max_seg)
            th = cpu_threads()
            cpu_sample = time_oracle_sample(hbf, obs_np, omegas, c, width_b, src.amplitude_phi,
                                            cpu_budget, th) + (th,)
        rate, sample, idx, acc_cpu, ev_cpu, dt, th = cpu_sample
        pos = np.empty(n_total, np.int64)
        pos[order_np] = np.arange(n_total)
        mine_acc = acc_gpu[pos[idx]]
        ref = acc_cpu
        m = np.abs(ref) > 0
        strong = m & (20 * np.log10(np.maximum(np.abs(ref), 1e-300) / np.abs(ref).max()) > -60)
        out["cpu_baseline"] = {"value": rate, "unit": "beam-receiver evals/s", "cores": th,
                               "kind": "port", "sample": sample,
                               "impl": "oracle/gbs_oracle.c (bit-exact C restatement of "
                                       "kernels.gbs_accumulate), WorkerPool.flat blocks"}
        out["parity_vs_cpu_sample"] = {
            "receivers": int(idx.size),
            "rel_l2": float(np.linalg.norm(mine_acc - ref) / np.linalg.norm(ref)),
            "max_dtl_db_above_-60dB": float(np.max(np.abs(20 * np.log10(
                np.abs(mine_acc[strong]) / np.abs(ref[strong]))))) if strong.any() else 0.0,
            "max_dtl_db_all": float(np.max(np.abs(20 * np.log10(
                np.abs(mine_acc[m]) / np.abs(ref[m]))))) if m.any() else 0.0,
            "zero_where_reference_nonzero": int(np.sum(m & (np.abs(mine_acc) == 0))),
            "evals_diff": int(np.abs(ev_gpu[pos[idx]] - ev_cpu).sum()),
        }
    del bundle, tr, acc, evals, flush, obs, obs_all, hb
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return out, cpu_sample


def run_ours(args):
    from paper_2501_13382_b200 import _lib
    D = Dist(args.gpus)
    peaks = None
    if D.rank == 0:
        p = _lib.probe_peaks(D.local)
        peaks = {"fp32_tflops": p["fp32_tflops"], "mufu_tops": p["mufu_tops"],
                 "source": "measured FFMA / FFMA2 stream (bf_probe_peaks, the faster of the "
                           "two), this GPU"}
    cpu = 0.0 if args.no_cpu_baseline else args.cpu_budget
    line, sample = measure(D, args.config, args.precision, args.steps, args.warmup, peaks, cpu,
                           e2e_steps=max(1, min(args.steps, 3)))
    if not args.headline_only:
        ns, _ = measure(D, "cfg4", "fp32", min(args.steps, 2), 3, peaks, cpu, e2e_steps=1)
        if D.rank == 0:
            line["north_star_shape"] = ns
        if args.precision == "fp32":
            o64, _ = measure(D, args.config, "fp64", min(args.steps, 2), 3, peaks, cpu,
                             e2e_steps=1, cpu_sample=sample)
            if D.rank == 0:
                line["fp64_oracle_mode"] = o64
    if D.rank == 0:
        print(json.dumps(line), flush=True)
    D.close()


def run_reference(args):
    """Reference arm: the C oracle (bit-exact restatement of the reference numba kernel)
    on all host threads, bounded receiver sample per step; rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    oracle.build()
    cfg = CONFIGS[args.config]
    sc, src, launch, tcfg, c, obs = make_inputs(cfg)
    th = cpu_threads()
    t0 = time.perf_counter()
    b = oracle.trace(sc.v0, sc.v1, sc.v2, sc.refl, sc.bounds, sc.diameter, src.position,
                     launch.directions, launch.e1, launch.e2, tcfg.length_cap(c), tcfg.r_max,
                     threads=th)
    b["weights"] = launch.weights
    t_trace = time.perf_counter() - t0
    nb = b["n_segs"].shape[0]
    per_step = max(2.0, args.ref_budget / max(1, args.steps + args.warmup))
    rates = []
    for i in range(args.warmup + args.steps):
        rate, sample, idx, _, _, dt = time_oracle_sample(
            b, obs, src.omegas, c, -src.beam_param_im, src.amplitude_phi, per_step, th)
        if i >= args.warmup:
            rates.append(rate)
    value = float(np.mean(rates))
    pairs = float(nb) * obs.shape[0]
    out = {"impl": "reference", "metric": METRIC, "value": value,
           "unit": "beam-receiver evals/s", "n_gpus": int(os.environ.get("WORLD_SIZE", "1")),
           "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": pairs / value * 1e3, "higher_is_better": True, "scaling": "strong",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": f"{args.config}: {cfg['desc']}", "beams": nb,
                      "receivers": int(obs.shape[0]), "extrapolated": "full-field time = "
                      "pairs / measured rate (per-receiver cost is independent)",
                      "trace_s": t_trace},
           "cpu_baseline": {"value": value, "unit": "beam-receiver evals/s", "cores": th,
                            "kind": "port", "sample": sample},
           "e2e": {"value": value, "unit": "beam-receiver evals/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg3", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--precision", default="fp32", choices=("fp32", "fp64"))
    ap.add_argument("--cpu-budget", type=float, default=15.0,
                    help="seconds of all-thread CPU work for the cpu_baseline sample")
    ap.add_argument("--ref-budget", type=float, default=60.0,
                    help="total seconds of CPU work for the --impl reference arm")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--headline-only", action="store_true",
                    help="skip the config-4 and fp64 measurements of the same line")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torch.distributed.run
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
               f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
        raise SystemExit(subprocess.call(cmd))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

"""Execution plans and the trace -> sum pipeline on B200 (mirror of ``beamfield.parallel``).

Reference: /root/reference/pkg/src/beamfield/parallel.py.  Kept names and
semantics: ExecPlan (validation), ChunkPlan, PhaseTimings, plan_chunks (greedy
maximal chunks, BudgetError when one ray does not fit), measure,
measure_per_ray_bytes (ray-0 estimate x 1.5, as the reference), run_pipeline,
pipeline_calibration.

What changes: the per-chunk RT and GBS phases run on the GPU (sm_100a tracer
and summation kernels), phase times come from CUDA events, and the CPU
thread-pool modes are replaced by device scheduling -- ``plan.mode`` and
``plan.workers`` are validated and recorded but no longer select a CPU
scheduler.  With ``torch.distributed`` initialised, receivers are partitioned
by spatial tiles across ranks (shard.py) and the field is gathered to rank 0.
"""
from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from .beamtrace import (Atmosphere, LaunchGrid, SourceSpec, TraceConfig, allocate_bundle,
                        launch_directions)
from .errors import BudgetError
from .gbs import FieldResult, ObserverSet, calibrate_phi
from .kernels import PIPELINE_PRECISION

MODES = ("sequential", "flat", "dynamic")
DEFAULT_SPLIT_THRESHOLD = 4096
PER_RAY_SAFETY = 1.5


@dataclass(frozen=True)
class ExecPlan:
    mode: str = "sequential"
    workers: int = 1
    split_threshold: int = DEFAULT_SPLIT_THRESHOLD
    memory_budget: int | None = None
    per_ray_bytes: int | None = None

    def __post_init__(self):
        if self.mode not in MODES:
            raise ValueError(f"unknown execution mode {self.mode!r}")
        if self.workers < 1:
            raise ValueError("worker count must be at least 1")
        if self.split_threshold < 1:
            raise ValueError("split threshold must be at least 1")
        if (self.memory_budget is not None and self.per_ray_bytes is not None
                and self.memory_budget < self.per_ray_bytes):
            raise ValueError("memory budget smaller than one ray")


@dataclass(frozen=True)
class ChunkPlan:
    chunk_sizes: tuple

    def __post_init__(self):
        object.__setattr__(self, "chunk_sizes", tuple(int(c) for c in self.chunk_sizes))
        if any(c <= 0 for c in self.chunk_sizes):
            raise ValueError("chunk sizes must be positive")

    @property
    def n_chunks(self) -> int:
        return len(self.chunk_sizes)

    @property
    def total(self) -> int:
        return sum(self.chunk_sizes)


@dataclass
class PhaseTimings:
    rt_seconds: float
    gbs_seconds: float
    total_seconds: float
    rt_share: float = 0.0
    gbs_share: float = 0.0
    speedup_vs_baseline: float | None = None
    gbs_evaluations: int = 0

    def __post_init__(self):
        if self.total_seconds > 0 and self.rt_share == 0.0 and self.gbs_share == 0.0:
            self.rt_share = self.rt_seconds / self.total_seconds
            self.gbs_share = self.gbs_seconds / self.total_seconds


def plan_chunks(total_rays: int, memory_budget: int, per_ray_bytes: int) -> ChunkPlan:
    """Greedy maximal chunks under the budget (parallel.py:91-105), via bf_plan_chunks."""
    import ctypes
    if total_rays < 1:
        raise ValueError("need at least one ray to plan chunks")
    if per_ray_bytes <= 0:
        raise ValueError("per-ray size must be positive")
    cap = memory_budget // per_ray_bytes
    if cap <= 0:
        raise BudgetError(
            f"memory budget {memory_budget} cannot hold one ray of {per_ray_bytes} bytes")
    n = -(-total_rays // cap)
    sizes = (ctypes.c_int64 * n)()
    got = ctypes.c_int64(0)
    _lib.check(_lib.load().bf_plan_chunks(int(total_rays), int(memory_budget),
                                          int(per_ray_bytes), sizes, n, ctypes.byref(got)))
    return ChunkPlan(tuple(sizes[: got.value]))


def block_partition(n: int, workers: int):
    """Contiguous near-even blocks of [0, n) (parallel.py:108-118)."""
    workers = max(1, workers)
    base, rem = divmod(n, workers)
    out, lo = [], 0
    for w in range(workers):
        size = base + (1 if w < rem else 0)
        out.append((lo, lo + size))
        lo += size
    return out


def measure(run, baseline: PhaseTimings | None = None) -> PhaseTimings:
    """Time a pipeline-style callable (parallel.py:228-246)."""
    t0 = time.perf_counter()
    out = run()
    total = time.perf_counter() - t0
    inner = out[1] if isinstance(out, tuple) else out
    t = PhaseTimings(rt_seconds=inner.rt_seconds, gbs_seconds=inner.gbs_seconds,
                     total_seconds=total,
                     rt_share=inner.rt_seconds / total if total > 0 else 0.0,
                     gbs_share=inner.gbs_seconds / total if total > 0 else 0.0,
                     gbs_evaluations=inner.gbs_evaluations)
    if baseline is not None:
        t.speedup_vs_baseline = baseline.total_seconds / total if total > 0 else None
    return t


def measure_per_ray_bytes(scene, source: SourceSpec, launch, cfg: TraceConfig,
                          atmosphere: Atmosphere, device=None) -> int:
    """Ray-0 estimate x 1.5 with 120 B/row, as the reference (parallel.py:249-257).

    (Reference defect kept for drop-in chunk plans: a padded device row costs
    (r_max+1) x 120 B regardless of ray 0.)
    """
    from .beamtrace import trace_into
    c = atmosphere.sound_speed
    b = allocate_bundle(1, launch, 0, source, cfg, c)
    trace_into(scene, source, launch, cfg, c, b, 0, 0, 1, device=device or 0)
    return int(max(1, int(b.n_segs[0])) * 15 * 8 * PER_RAY_SAFETY)


def _device(device):
    import os

    import torch
    if device is None:
        device = int(os.environ.get("LOCAL_RANK", "0"))
    return torch.device("cuda", int(device)) if not isinstance(device, torch.device) else device


def run_pipeline(scene, source: SourceSpec, grid: LaunchGrid, cfg: TraceConfig,
                 observers: ObserverSet, plan: ExecPlan, atmosphere: Atmosphere,
                 calibration: float | None = None, use_cutoff: bool = True, *,
                 precision: str | None = None, device=None, group=None):
    """Trace-then-sum pipeline on the GPU, chunked to the plan's budget (parallel.py:260-351).

    Returns (FieldResult, PhaseTimings) like the reference.  Under
    torch.distributed (or with ``group``) every rank sums its receiver tiles
    and rank 0 receives the assembled field; other ranks get their local
    PhaseTimings and a FieldResult of None.
    """
    import torch

    from . import engine, shard
    precision = PIPELINE_PRECISION if precision is None else precision
    t_start = time.perf_counter()
    dev = _device(device)
    torch.cuda.set_device(dev)
    c = atmosphere.sound_speed
    launch = launch_directions(grid)
    n_rays = len(launch)
    omegas = source.omegas

    if plan.memory_budget is not None:
        per_ray = plan.per_ray_bytes
        if per_ray is None:
            per_ray = measure_per_ray_bytes(scene, source, launch, cfg, atmosphere, dev.index)
        chunk_plan = plan_chunks(n_rays, plan.memory_budget, per_ray)
    else:
        chunk_plan = ChunkPlan((n_rays,))
    if calibration is None:
        calibration = pipeline_calibration(source, grid, cfg, atmosphere, device=dev.index)

    world, rank = shard.world(group)
    pts = observers.points
    obs_all = torch.from_numpy(pts).to(dev)
    if world > 1:
        order = shard.tile_order(obs_all)
        mine = shard.rank_indices(order, rank, world)
        obs_local = obs_all.index_select(0, mine).contiguous()
    else:
        mine = None
        obs_local = obs_all
    n_local = obs_local.shape[0]
    acc = torch.zeros((n_local, omegas.shape[0]), dtype=torch.complex128, device=dev)
    evals = torch.zeros(n_local, dtype=torch.int64, device=dev)
    dscene = engine.DeviceScene.from_scene(scene, dev)
    stream = torch.cuda.current_stream(dev)
    # fp32: every traced chunk is appended to compact rows resident in HBM (68 B per
    # segment) and all rays are summed in ONE call -- the field does not depend on the
    # chunk plan, and the receivers are tiled once.  fp64 (oracle mode):
    # the chunk's padded bundle is summed per chunk, bit-identical by construction
    # (per-observer ascending beams continue acc in place).
    rows = engine.SegmentRows(dev) if precision == "fp32" else None
    e_start = torch.cuda.Event(enable_timing=True)
    e_rt = torch.cuda.Event(enable_timing=True)
    e_start.record(stream)
    rt_ms, gbs_ms = 0.0, 0.0
    lo = 0
    buf = None
    for n in chunk_plan.chunk_sizes:
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record(stream)
        if buf is None or buf.n_paths < n:
            buf = None
            out = engine.trace_device_rows(dscene, source, launch, cfg, c, lo, lo + n, dev,
                                           row_base=lo, stream=stream)
            buf = out["bundle"]
        else:  # reuse the chunk buffer: rays [lo, lo + n) into its first n rows
            buf.weights[:n].copy_(torch.from_numpy(
                np.ascontiguousarray(launch.weights[lo:lo + n])).to(dev))
            engine.trace_device_rows(dscene, source, launch, cfg, c, lo, lo + n, dev,
                                     row_base=lo, out=buf, stream=stream)
        if rows is not None:
            rows.append(buf, n_beams=n, stream=stream)
        e1.record(stream)
        if n_local and rows is None:
            engine.accumulate(buf, obs_local, omegas, -source.beam_param_im, use_cutoff, acc,
                              evals, beam_hi=n, precision=precision, stream=stream,
                              presorted=world > 1)
        e2.record(stream)
        torch.cuda.synchronize(dev)
        rt_ms += e0.elapsed_time(e1)
        gbs_ms += e1.elapsed_time(e2)
        lo += n
    if rows is not None:
        e_rt.record(stream)
        if n_local:
            rows.accumulate(obs_local, omegas, -source.beam_param_im, use_cutoff, acc, evals,
                            stream=stream, presorted=world > 1)
        e_end = torch.cuda.Event(enable_timing=True)
        e_end.record(stream)
        torch.cuda.synchronize(dev)
        gbs_ms += e_rt.elapsed_time(e_end)
        rows.close()
    torch.cuda.synchronize(dev)
    rt = rt_ms / 1e3
    gbs_t = gbs_ms / 1e3
    if world > 1:
        acc_full, evals_full = shard.gather_field(acc, evals, order, rank, world, pts.shape[0],
                                                  group)
    else:
        acc_full, evals_full = acc, evals
    result = None
    n_eval = int(evals.sum().item())
    if rank == 0:
        pressure = calibration * acc_full.cpu().numpy()
        result = FieldResult.from_pressure(pressure, calibration)
        n_eval = int(evals_full.sum().item())
    total = time.perf_counter() - t_start
    timings = PhaseTimings(rt_seconds=rt, gbs_seconds=gbs_t, total_seconds=total,
                           rt_share=rt / total if total > 0 else 0.0,
                           gbs_share=gbs_t / total if total > 0 else 0.0,
                           gbs_evaluations=n_eval)
    return result, timings


def pipeline_calibration(source: SourceSpec, grid: LaunchGrid, cfg: TraceConfig,
                         atmosphere: Atmosphere, device=None) -> float:
    """Free-field calibration traced on an empty scene (parallel.py:354-368)."""
    import torch

    from . import engine
    from .scene import empty_scene
    dev = _device(device)
    cal_grid = grid
    if (grid.n_rays < 64 * 64 or grid.theta_min > 0 or grid.theta_max < 180
            or grid.phi_min > 0 or grid.phi_max < 360):
        cal_grid = LaunchGrid(0.0, 180.0, 0.0, 360.0, 64, 64)
    launch = launch_directions(cal_grid)
    c = atmosphere.sound_speed
    out = engine.trace_device_rows(engine.DeviceScene.from_scene(empty_scene(), dev), source,
                                   launch, cfg, c, 0, len(launch), dev)
    torch.cuda.synchronize(dev)
    bundle = out["bundle"].to_host()
    # 26 x F single-receiver sums: always in fp64 (oracle) mode, so the scale is the
    # reference's to ~1e-12 whichever precision the field itself is summed in
    return calibrate_phi(bundle, atmosphere, source, precision="fp64", device=dev.index)


def run_snapshots(scene, sources, grid: LaunchGrid, cfg: TraceConfig, observers: ObserverSet,
                  plan: ExecPlan, atmosphere: Atmosphere, calibration: float | None = None,
                  use_cutoff: bool = True, **kw):
    """Moving-source noise map: one run_pipeline field per source
    position (snapshot) and the energy-mean SPL over the snapshots,
    10 log10(mean_k |p_k|^2 / p_ref^2) per receiver and frequency.  Moving sources are a
    reference non-goal; each snapshot is the reference's static problem.

    Returns (fields, spl_energy_mean, timings) on rank 0; fields of other ranks are None.
    """
    from .gbs import P_REF
    fields, timings = [], []
    energy = None
    for src in sources:
        res, t = run_pipeline(scene, src, grid, cfg, observers, plan, atmosphere,
                              calibration=calibration, use_cutoff=use_cutoff, **kw)
        fields.append(res)
        timings.append(t)
        if res is not None:
            e = np.abs(res.pressure) ** 2
            energy = e if energy is None else energy + e
    spl_mean = None
    if energy is not None:
        with np.errstate(divide="ignore"):
            spl_mean = 10.0 * np.log10(energy / len(sources) / P_REF ** 2)
    return fields, spl_mean, timings

"""GPU parity at the benchmark shapes and at the edges of the fp32 range.

* ΔTL on every receiver: no-cutoff scenes whose far receivers sit e^-100 .. e^-700 below
  the field maximum (the fp32 exponent range ends at e^-87): the fp32 path must keep
  the reference's magnitude there too (kernels.py:384-385 with use_cutoff False).
* Config 2 (open plane, 100k rays, 1024 x 1024 receivers) and config 4 (dense city,
  4M rays) at full size against the C oracle on strided receiver samples.
* The device tracer against the C restatement of the reference tracer on ~10k-ray
  strided samples of the config-3 and config-4 launches (bit for bit).
* run_pipeline's distributed branch (2 ranks over gloo sharing cuda:0) == one rank,
  bit for bit; and run_pipeline's ChunkPlan invariance (fp64 bit-exact, fp32 too).
"""
import os
import socket
import sys

import numpy as np
import pytest

import oracle
from conftest import ROOT, rel_l2, tl_db

pytestmark = pytest.mark.gpu

FP32_L2 = 1e-4
FP32_TL_DB = 0.01


def _device_bundle(name, rays=None):
    import torch

    import bench
    from paper_2501_13382_b200 import engine
    cfg = dict(bench.CONFIGS[name])
    sc, src, launch, tcfg, c, obs = bench.make_inputs(cfg)
    dev = torch.device("cuda", 0)
    tr = engine.trace_device_rows(engine.DeviceScene.from_scene(sc, dev), src, launch, tcfg, c,
                                  0, len(launch), dev)
    torch.cuda.synchronize()
    return sc, src, launch, tcfg, c, obs, tr["bundle"]


def _oracle_on(hb, obs, om, c, width_b, phi, threads, use_cutoff=True):
    ref = np.zeros((obs.shape[0], om.shape[0]), np.complex128)
    rev = np.zeros(obs.shape[0], np.int64)
    oracle.gbs_accumulate(hb.seg_origin, hb.seg_dir, hb.seg_e1, hb.seg_e2, hb.seg_len,
                          hb.seg_s0, hb.seg_refl, hb.n_segs, hb.max_seg, hb.weights, obs, om,
                          c, width_b, phi, use_cutoff, ref, rev, 0, obs.shape[0], 0,
                          hb.n_segs.shape[0], threads=threads)
    return ref, rev


@pytest.mark.parametrize("scene,freq,im_b,grid", [
    ("plane", 2000.0, -200.0, (6, 12)),   # down to e^-570 below the maximum
    ("city", 1000.0, -300.0, (8, 16)),    # e^-315
    ("plane", 1000.0, -600.0, (4, 8)),    # e^-290
    ("plane", 4000.0, -80.0, (10, 20))])  # e^-360
def test_fp32_all_receivers_without_cutoff(scene, freq, im_b, grid, threads):
    """No cutoff, sparse beams, receivers up to 300 m away: many receivers get only
    contributions far below the fp32 range; every receiver with a non-zero reference value
    must match within 0.01 dB (the fp32 path redoes such amplitudes in fp64)."""
    import torch

    from paper_2501_13382_b200 import engine, kernels
    from paper_2501_13382_b200.beamtrace import (Atmosphere, LaunchGrid, SourceSpec,
                                                 TraceConfig, launch_directions)
    from paper_2501_13382_b200.scene import make_city, make_ground_plane
    dev = torch.device("cuda", 0)
    sc = make_ground_plane(1000.0) if scene == "plane" else make_city(4, 4, 40.0, 20.0, 300.0)
    src_pos = np.array([0.0, 0.0, 10.0]) if scene == "plane" else np.array([20.0, 3.0, 2.0])
    source = SourceSpec(position=src_pos, frequencies=(freq,), beam_param_im=im_b)
    launch = launch_directions(LaunchGrid(0.0, 180.0, 0.0, 360.0, *grid))
    cfg = TraceConfig(4000, 1e-4, 4)
    c = Atmosphere(20.0).sound_speed
    tr = engine.trace_device_rows(engine.DeviceScene.from_scene(sc, dev), source, launch, cfg,
                                  c, 0, len(launch), dev)
    hb = tr["bundle"].to_host()
    rng = np.random.default_rng(11)
    r = rng.uniform(20.0, 300.0, 3000)
    ph = rng.uniform(0, 2 * np.pi, 3000)
    obs = np.ascontiguousarray(np.stack([src_pos[0] + r * np.cos(ph), src_pos[1] + r * np.sin(ph),
                                         rng.uniform(0.5, 30.0, 3000)], 1))
    om = source.omegas
    ref, rev = _oracle_on(hb, obs, om, float(c), -im_b, 1.0, threads, use_cutoff=False)
    acc = np.zeros_like(ref)
    ev = np.zeros_like(rev)
    kernels.gbs_accumulate(hb.seg_origin, hb.seg_dir, hb.seg_e1, hb.seg_e2, hb.seg_len,
                           hb.seg_s0, hb.seg_refl, hb.n_segs, hb.max_seg, hb.weights, obs, om,
                           float(c), -im_b, 1.0, False, acc, ev, 0, obs.shape[0], 0,
                           hb.n_segs.shape[0], precision="fp32")
    m = np.abs(ref) > 0
    rel = np.abs(ref[m]) / np.abs(ref).max()
    assert (rel < 1e-40).sum() > 100  # the scene does reach far below the fp32 range
    assert not np.any(m & (np.abs(acc) == 0))  # nothing underflows to zero
    assert rel_l2(acc, ref) <= FP32_L2
    assert tl_db(acc, ref) <= FP32_TL_DB  # every receiver with a non-zero reference
    assert np.array_equal(ev, rev) or abs(int(ev.sum()) - int(rev.sum())) <= 10


@pytest.mark.parametrize("name,n_sample", [("cfg2", 1500), ("cfg4", 120)])
def test_full_size_config_vs_oracle(name, n_sample, threads):
    """The benchmark configurations at full size (every beam, every receiver on the GPU)
    against the oracle on a strided receiver sample: config 2 (open plane, 1e11 pairs)
    and config 4 (dense city, 4M rays x 4M receivers, the north-star shape)."""
    import torch

    from paper_2501_13382_b200 import engine, shard
    sc, src, launch, tcfg, c, obs, bundle = _device_bundle(name)
    dev = torch.device("cuda", 0)
    od = torch.from_numpy(obs).to(dev)
    nf = src.omegas.shape[0]
    acc = torch.zeros((obs.shape[0], nf), dtype=torch.complex128, device=dev)
    ev = torch.zeros(obs.shape[0], dtype=torch.int64, device=dev)
    engine.accumulate(bundle, od, src.omegas, -src.beam_param_im, True, acc, ev,
                      precision="fp32")
    idx = np.linspace(0, obs.shape[0] - 1, n_sample).astype(np.int64)
    got = acc.cpu().numpy()[idx]
    gev = ev.cpu().numpy()[idx]
    hb = bundle.to_host()
    del bundle, acc, ev
    torch.cuda.empty_cache()
    ref, rev = _oracle_on(hb, np.ascontiguousarray(obs[idx]), src.omegas, float(c),
                          -src.beam_param_im, 1.0, threads)
    assert rel_l2(got, ref) <= FP32_L2
    assert tl_db(got, ref) <= FP32_TL_DB
    assert abs(int(gev.sum()) - int(rev.sum())) <= 1e-4 * int(rev.sum()) + 10


@pytest.mark.parametrize("name", ["cfg3", "cfg4"])
def test_tracer_at_scale_bitexact(name, threads):
    """sm_100a tracer == C restatement of the reference tracer (kernels.py:143-301), bit
    for bit, on a strided ~10k-ray sample of the benchmark launch (500k / 4M rays)."""
    import torch

    import bench
    from paper_2501_13382_b200 import engine
    from paper_2501_13382_b200.beamtrace import LaunchSet
    sc, src, launch, tcfg, c, obs = bench.make_inputs(bench.CONFIGS[name])
    idx = np.linspace(0, len(launch) - 1, 10007).astype(np.int64)
    sub = LaunchSet(gamma1=launch.gamma1[idx], gamma2=launch.gamma2[idx],
                    directions=np.ascontiguousarray(launch.directions[idx]),
                    weights=launch.weights[idx], e1=np.ascontiguousarray(launch.e1[idx]),
                    e2=np.ascontiguousarray(launch.e2[idx]))
    dev = torch.device("cuda", 0)
    tr = engine.trace_device_rows(engine.DeviceScene.from_scene(sc, dev), src, sub, tcfg, c, 0,
                                  len(sub), dev)
    torch.cuda.synchronize()
    got = tr["bundle"].to_host()
    ref = oracle.trace(sc.v0, sc.v1, sc.v2, sc.refl, sc.bounds, sc.diameter, src.position,
                       sub.directions, sub.e1, sub.e2, tcfg.length_cap(c), tcfg.r_max,
                       threads=threads)
    for f in ("n_segs", "n_refls"):
        assert np.array_equal(getattr(got, f), ref[f]), f
    for f in ("seg_origin", "seg_dir", "seg_e1", "seg_e2", "seg_len", "seg_s0", "seg_refl"):
        a = np.asarray(getattr(got, f))
        assert np.array_equal(a.view(np.uint64), ref[f].view(np.uint64)), f
    assert int(ref["n_refls"].max()) >= 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _pipeline_problem():
    from paper_2501_13382_b200 import (Atmosphere, ExecPlan, LaunchGrid, ObserverSet,
                                       SourceSpec, TraceConfig, make_city)
    sc = make_city(5, 10, 40.0, 20.0, 300.0)
    src = SourceSpec(position=np.array([20.0, 0.0, 2.0]), frequencies=(125.0, 500.0),
                     beam_param_im=-10.0)
    x = -60.0 + 0.5 * np.arange(120)
    X, Y = np.meshgrid(x, x, indexing="xy")
    pts = np.stack([X.ravel(), Y.ravel(), np.full(X.size, 1.8)], 1)
    return (sc, src, LaunchGrid(n_theta=40, n_phi=80), TraceConfig(5000, 1e-4, 8),
            ObserverSet(pts), ExecPlan(memory_budget=1000 * 1080, per_ray_bytes=1080),
            Atmosphere(20.0))


def _pipeline_worker(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, str(ROOT))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2501_13382_b200 import parallel
    res, t = parallel.run_pipeline(*_pipeline_problem(), calibration=1.0, device=0)
    if rank == 0:
        np.savez(out_path, p=res.pressure, ev=t.gbs_evaluations)
    else:
        assert res is None
    dist.barrier()
    dist.destroy_process_group()


def test_run_pipeline_distributed_equals_one_rank(tmp_path):
    """run_pipeline's torch.distributed branch (parallel.py:192-234): two ranks over gloo,
    both on cuda:0, each summing its receiver tiles; rank 0's gathered field equals the
    single-rank field bit for bit (SPEC.md:359 extended to ranks)."""
    import torch.multiprocessing as mp

    from paper_2501_13382_b200 import parallel
    res1, t1 = parallel.run_pipeline(*_pipeline_problem(), calibration=1.0, device=0)
    ctx = mp.get_context("spawn")
    port = _free_port()
    out = str(tmp_path / "w2.npz")
    procs = [ctx.Process(target=_pipeline_worker, args=(r, 2, port, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
    assert all(p.exitcode == 0 for p in procs)
    z = np.load(out)
    assert np.array_equal(z["p"], res1.pressure)
    assert int(z["ev"]) == t1.gbs_evaluations


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_run_pipeline_chunk_plan_invariance(precision):
    """The reference's run_pipeline gives a bit-identical FieldResult for every ChunkPlan
    (SPEC.md:359); so does this one, in both precisions."""
    from paper_2501_13382_b200 import ExecPlan, parallel
    sc, src, grid, cfg, obs, plan, atm = _pipeline_problem()
    fields = []
    for budget in (None, 3200 * 1080, 1000 * 1080, 333 * 1080):
        p = ExecPlan() if budget is None else ExecPlan(memory_budget=budget, per_ray_bytes=1080)
        res, t = parallel.run_pipeline(sc, src, grid, cfg, obs, p, atm, calibration=1.0,
                                       precision=precision)
        fields.append((res.pressure, t.gbs_evaluations))
    for p, e in fields[1:]:
        assert np.array_equal(p, fields[0][0]) and e == fields[0][1]

"""GPU parity of the sm_100a GBS path against the reference golden fixtures and the
C oracle (all calls go through the C ABI in libbf_gbs.so).

Tolerances (BASELINE.json north_star):
  fp64 mode: relL2(acc) <= 1e-12, evals bit-exact, nearest-segment k/behind bit-exact;
  fp32 mode: relL2(acc) <= 1e-4, max dTL <= 0.01 dB over EVERY receiver whose reference
  value is non-zero (and, reported beside it, over receivers within 60 dB of the maximum).
"""
import numpy as np
import pytest

import oracle
from conftest import CASES, gbs_args, load_case, rel_l2, tl_db

pytestmark = pytest.mark.gpu

FP64_TOL = 1e-12
FP32_L2 = 1e-4
FP32_TL_DB = 0.01
FP32_TL_ALL_DB = 0.01


def run(b, precision, obs=None, calls=None):
    from paper_2501_13382_b200 import kernels
    obs = b["obs"] if obs is None else obs
    acc = np.zeros((obs.shape[0], b["omegas"].shape[0]), np.complex128)
    ev = np.zeros(obs.shape[0], np.int64)
    calls = b["calls"] if calls is None else calls
    for olo, ohi, blo, bhi in calls:
        kernels.gbs_accumulate(*gbs_args(b, obs), acc, ev, olo, ohi, blo, bhi,
                               precision=precision)
    return acc, ev


@pytest.mark.parametrize("name", CASES)
def test_fp64_mode_vs_reference(name):
    b = load_case(name)
    acc, ev = run(b, "fp64")
    assert rel_l2(acc, b["acc"]) <= FP64_TOL
    assert np.max(np.abs(acc - b["acc"])) <= FP64_TOL * np.max(np.abs(b["acc"]))
    assert np.array_equal(ev, b["evals"])


@pytest.mark.parametrize("name", CASES)
def test_fp32_mode_vs_reference(name):
    b = load_case(name)
    acc, ev = run(b, "fp32")
    ref = b["acc"]
    assert rel_l2(acc, ref) <= FP32_L2
    assert tl_db(acc, ref, floor_db=-60.0) <= FP32_TL_DB
    assert tl_db(acc, ref) <= FP32_TL_ALL_DB
    # cutoff decisions may flip only at the e^-36 threshold
    assert abs(int(ev.sum()) - int(b["evals"].sum())) <= 1e-4 * int(b["evals"].sum()) + 10


@pytest.mark.parametrize("name", ["cfg1_open_plane", "city_street", "city_corner_f5"])
def test_nearest_segment_bitexact(name):
    from paper_2501_13382_b200 import kernels
    b = load_case(name)
    out = kernels.nearest_batch(b["seg_origin"], b["seg_dir"], b["seg_e1"], b["seg_e2"],
                                b["seg_len"], b["seg_s0"], b["seg_refl"], b["n_segs"],
                                b["max_seg"], b["obs"], b["ns_obs"], b["ns_beam"])
    assert np.array_equal(out[:, 0].astype(np.int64), b["ns_k"])
    assert np.array_equal(out[:, 5].astype(np.int8), b["ns_behind"])
    for col, key in ((1, "ns_s"), (2, "ns_q1"), (3, "ns_q2"), (4, "ns_refl")):
        assert np.array_equal(out[:, col], b[key])


@pytest.mark.parametrize("name", ["cfg1_open_plane", "city_street", "city_corner_f5",
                                  "open_paper_imb"])
def test_tracer_bitexact_vs_reference(name):
    """sm_100a tracer == reference trace_into bundle (beamtrace.py:291-306), bit for bit."""
    import torch

    from paper_2501_13382_b200 import beamtrace, engine, scene
    z = np.load(f"tests/golden/{name}.npz")
    b = load_case(name)
    args = z["scene_args"]
    sc = (scene.make_ground_plane(float(args[0])) if str(z["scene_kind"]) == "plane" else
          scene.make_city(int(args[0]), int(args[1]), float(args[2]), float(args[3]),
                          float(args[4])))
    src = beamtrace.SourceSpec(position=z["src"], frequencies=tuple(z["freqs"]),
                               beam_param_im=float(z["im_b"]))
    grid = beamtrace.LaunchGrid(0.0, 180.0, 0.0, 360.0, int(z["n_theta"]), int(z["n_phi"]))
    cfg = beamtrace.TraceConfig(int(z["n_steps"]), float(z["dt"]), int(z["r_max"]))
    launch = beamtrace.launch_directions(grid)
    dev = torch.device("cuda", 0)
    out = engine.trace_device_rows(engine.DeviceScene.from_scene(sc, dev), src, launch, cfg,
                                   float(z["c"]), 0, len(launch), dev)
    torch.cuda.synchronize()
    assert np.array_equal(out["n_segs"].cpu().numpy(), b["n_segs"])
    assert np.array_equal(out["n_refls"].cpu().numpy(), z["n_refls"])
    for f in ("seg_origin", "seg_dir", "seg_e1", "seg_e2", "seg_len", "seg_s0", "seg_refl"):
        got = out[f].cpu().numpy()
        assert np.array_equal(got.view(np.uint64), b[f].view(np.uint64)), f


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_device_path_equals_host_path(precision):
    """Host-buffer ABI (pageable numpy, streamed beam groups) == device ABI, bit for bit."""
    import torch

    from paper_2501_13382_b200 import kernels
    b = load_case("city_street")
    acc_h, ev_h = run(b, precision)
    dev = torch.device("cuda", 0)
    t = lambda a, dt=torch.float64: torch.as_tensor(np.ascontiguousarray(a)).to(dev, dt)  # noqa
    obs = b["obs"]
    acc = torch.zeros((obs.shape[0], 1), dtype=torch.complex128, device=dev)
    ev = torch.zeros(obs.shape[0], dtype=torch.int64, device=dev)
    kernels.gbs_accumulate(t(b["seg_origin"]), t(b["seg_dir"]), t(b["seg_e1"]), t(b["seg_e2"]),
                           t(b["seg_len"]), t(b["seg_s0"]), t(b["seg_refl"]),
                           t(b["n_segs"], torch.int32), b["max_seg"], t(b["weights"]), t(obs),
                           b["omegas"], float(b["c"]), -float(b["beam_param_im"]), 1.0, True,
                           acc, ev, 0, obs.shape[0], 0, b["n_segs"].shape[0],
                           precision=precision)
    torch.cuda.synchronize()
    assert np.array_equal(acc.cpu().numpy(), acc_h)
    assert np.array_equal(ev.cpu().numpy(), ev_h)


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_memory_budget_grouping_bitexact(precision):
    """A device budget far below the bundle: the host ABI streams many beam groups
    (fp32: groups of whole beam ranges, fp64: padded chunks) through pinned staging and
    the device ABI sums in many groups; the bits equal the one-group call's."""
    import torch

    from paper_2501_13382_b200 import _lib, engine, kernels
    b = load_case("city_corner_f5")
    obs = np.ascontiguousarray(b["obs"][:3000])
    nb = b["n_segs"].shape[0]
    ref, rev = run(b, precision, obs, [(0, obs.shape[0], 0, nb)])
    dev = torch.device("cuda", 0)
    db = engine.DeviceBundle.from_host(_pb(b), dev)
    od = torch.from_numpy(obs).to(dev)
    try:
        _lib.set_memory_budget(0, 1 << 20)  # 1 MiB: dozens of groups
        got, gev = run(b, precision, obs, [(0, obs.shape[0], 0, nb)])
        acc = torch.zeros((obs.shape[0], 5), dtype=torch.complex128, device=dev)
        ev = torch.zeros(obs.shape[0], dtype=torch.int64, device=dev)
        engine.accumulate(db, od, b["omegas"], -float(b["beam_param_im"]), True, acc, ev,
                          precision=precision)
        torch.cuda.synchronize()
    finally:
        _lib.set_memory_budget(0, 0)
    assert np.array_equal(got, ref) and np.array_equal(gev, rev)
    assert np.array_equal(acc.cpu().numpy(), ref) and np.array_equal(ev.cpu().numpy(), rev)
    assert rel_l2(ref, b["acc"][:3000]) <= (FP64_TOL if precision == "fp64" else FP32_L2)


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_many_frequencies(precision, threads):
    """F = 21 (1/3-octave bands 100 Hz - 10 kHz): summed in groups of <= 8 frequencies,
    against the oracle (kernels.py:362,380 loop over any nf)."""
    from paper_2501_13382_b200 import kernels
    b = load_case("city_street")
    obs = np.ascontiguousarray(b["obs"][::3])
    om = 2 * np.pi * 100.0 * 10 ** (np.arange(21) / 10.0)
    args = gbs_args(b, obs)
    args[11] = om
    nb = b["n_segs"].shape[0]
    ref = np.zeros((obs.shape[0], 21), np.complex128)
    rev = np.zeros(obs.shape[0], np.int64)
    oracle.gbs_accumulate(*args, ref, rev, 0, obs.shape[0], 0, nb, threads=threads)
    acc = np.zeros_like(ref)
    ev = np.zeros_like(rev)
    kernels.gbs_accumulate(*args, acc, ev, 0, obs.shape[0], 0, nb, precision=precision)
    if precision == "fp64":
        assert rel_l2(acc, ref) <= FP64_TOL and np.array_equal(ev, rev)
    else:
        for f in range(21):
            assert rel_l2(acc[:, f], ref[:, f]) <= FP32_L2, f
        assert tl_db(acc, ref, floor_db=-60.0) <= FP32_TL_DB
        assert abs(int(ev.sum()) - int(rev.sum())) <= 1e-4 * int(rev.sum()) + 10


def test_device_call_returns_before_the_kernels_end():
    """The device ABI never waits on the GPU: a config-3-sized call returns while its
    work is still queued on the caller's stream (no host syncs inside the call)."""
    import time

    import torch

    from paper_2501_13382_b200 import engine
    b = load_case("city_street")
    dev = torch.device("cuda", 0)
    db = engine.DeviceBundle.from_host(_pb(b), dev, with_frame=False)
    x = np.arange(600) * 0.25 - 75.0
    X, Y = np.meshgrid(x, x, indexing="xy")
    obs = torch.from_numpy(np.stack([X.ravel(), Y.ravel(), np.full(X.size, 1.8)], 1)).to(dev)
    acc = torch.zeros((obs.shape[0], 1), dtype=torch.complex128, device=dev)
    ev = torch.zeros(obs.shape[0], dtype=torch.int64, device=dev)
    s = torch.cuda.Stream(dev)
    for _ in range(3):  # warm-up: grow-only workspaces and both statistics buffers
        engine.accumulate(db, obs, b["omegas"], 10.0, True, acc, ev, stream=s)
    torch.cuda.synchronize()
    blocker = torch.cuda.Event()
    with torch.cuda.stream(s):
        torch.cuda._sleep(200_000_000)  # keep the stream busy (~0.1 s)
        t0 = time.perf_counter()
        engine.accumulate(db, obs, b["omegas"], 10.0, True, acc, ev, stream=s)
        host_s = time.perf_counter() - t0
        blocker.record(s)
    assert not blocker.query()  # the call's kernels have not run yet
    torch.cuda.synchronize()
    assert host_s < 0.05


def test_default_stream_call_is_ordered_and_async():
    """On torch's default stream (handle 0, passed as cudaStreamLegacy) a call is fenced in
    and out of that stream: it returns while earlier default-stream work still runs, sees
    that work's results (acc filled by a torch kernel queued behind a sleep), and later
    default-stream work sees its result; repeated calls (graph replay) keep the bits."""
    import time

    import torch

    from paper_2501_13382_b200 import engine
    b = load_case("city_street")
    dev = torch.device("cuda", 0)
    db = engine.DeviceBundle.from_host(_pb(b), dev, with_frame=False)
    obs = torch.from_numpy(b["obs"][:4096].copy()).to(dev)
    acc = torch.zeros((obs.shape[0], 1), dtype=torch.complex128, device=dev)
    ev = torch.zeros(obs.shape[0], dtype=torch.int64, device=dev)
    assert torch.cuda.current_stream(dev).cuda_stream == 0
    acc.fill_(1.0)
    torch.cuda.synchronize()
    engine.accumulate(db, obs, b["omegas"], 10.0, True, acc, ev)
    torch.cuda.synchronize()
    ref = acc.cpu().numpy().copy()  # acc = 1 + the field, summed onto the 1
    for _ in range(4):  # eager, capture, replays
        torch.cuda._sleep(100_000_000)  # ~50 ms of default-stream work in front
        acc.fill_(1.0)                  # ... then the field the call must continue
        ev.zero_()
        t0 = time.perf_counter()
        engine.accumulate(db, obs, b["omegas"], 10.0, True, acc, ev)
        host_s = time.perf_counter() - t0
        out = acc.clone()               # default-stream work after the call
        torch.cuda.synchronize()
        assert host_s < 0.03
        assert np.array_equal(out.cpu().numpy(), ref)


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_chunked_and_ranged_calls(precision):
    """Beam chunks continue acc in place; rows outside [obs_lo, obs_hi) untouched."""
    b = load_case("city_corner_f5")
    obs = b["obs"][:1500]
    nb = b["n_segs"].shape[0]
    one, ev1 = run(b, precision, obs, [(0, 1500, 0, nb)])
    many, evm = run(b, precision, obs, [(0, 1500, 0, 700), (0, 1500, 700, 701),
                                        (0, 1500, 701, nb)])
    if precision == "fp64":
        assert np.array_equal(one, many)
    else:
        assert rel_l2(many, one) <= 1e-6
    assert np.array_equal(ev1, evm) or precision == "fp32"
    part, evp = run(b, precision, obs, [(100, 900, 0, nb)])
    assert not part[:100].any() and not part[900:].any()
    assert not evp[:100].any() and not evp[900:].any()
    assert rel_l2(part[100:900], one[100:900]) <= (0 if precision == "fp64" else 1e-5)


def test_edge_cases():
    from paper_2501_13382_b200 import kernels
    b = load_case("city_street")
    obs = b["obs"][:300]
    nb = b["n_segs"].shape[0]
    # empty ranges are no-ops
    acc = np.full((300, 1), 1 + 2j)
    ev = np.full(300, 5, np.int64)
    kernels.gbs_accumulate(*gbs_args(b, obs), acc, ev, 10, 10, 0, nb)
    kernels.gbs_accumulate(*gbs_args(b, obs), acc, ev, 0, 300, 7, 7)
    assert (acc == 1 + 2j).all() and (ev == 5).all()
    # beams with n_segs == 0 contribute nothing (kernels.py:369-371)
    a2 = list(gbs_args(b, obs))
    ns = b["n_segs"].copy()
    ns[::3] = 0
    a2[7] = ns
    for prec in ("fp64", "fp32"):
        acc = np.zeros((300, 1), np.complex128)
        ev = np.zeros(300, np.int64)
        kernels.gbs_accumulate(*a2, acc, ev, 0, 300, 0, nb, precision=prec)
        ref = np.zeros_like(acc)
        rev = np.zeros_like(ev)
        oracle.gbs_accumulate(*a2, ref, rev, 0, 300, 0, nb)
        assert rel_l2(acc, ref) <= (FP64_TOL if prec == "fp64" else FP32_L2)
    # bad arguments raise like the reference's callers would
    with pytest.raises(ValueError):
        kernels.gbs_accumulate(*gbs_args(b, obs), np.zeros((300, 1), np.complex128),
                               np.zeros(300, np.int64), 0, 301, 0, nb)
    with pytest.raises(TypeError):
        kernels.gbs_accumulate(*gbs_args(b, obs), np.zeros((300, 1), np.complex64),
                               np.zeros(300, np.int64), 0, 300, 0, nb)


def test_sharded_equals_unsharded_bitexact():
    """Receiver-tile partition (shard.py) gives identical bits for 1, 2, 3 and 8 ranks."""
    import torch

    from paper_2501_13382_b200 import engine, shard
    b = load_case("city_corner_f5")
    dev = torch.device("cuda", 0)
    bundle = engine.DeviceBundle.from_host(_pb(b), dev)
    obs = torch.from_numpy(b["obs"]).to(dev)
    order = shard.tile_order(obs)
    n = obs.shape[0]
    full = {}
    for world in (1, 2, 3, 8):
        acc_full = torch.zeros((n, 5), dtype=torch.complex128, device=dev)
        for r in range(world):
            idx = shard.rank_indices(order, r, world)
            o = obs.index_select(0, idx).contiguous()
            acc = torch.zeros((o.shape[0], 5), dtype=torch.complex128, device=dev)
            ev = torch.zeros(o.shape[0], dtype=torch.int64, device=dev)
            engine.accumulate(bundle, o, b["omegas"], -float(b["beam_param_im"]), True, acc, ev,
                              presorted=True)
            acc_full[idx] = acc
        torch.cuda.synchronize()
        full[world] = acc_full.cpu().numpy()
    for w in (2, 3, 8):
        assert np.array_equal(full[w], full[1])
    assert rel_l2(full[1], b["acc"]) <= FP32_L2


def _pb(b):
    from paper_2501_13382_b200.beamtrace import PathBundle
    return PathBundle(seg_origin=b["seg_origin"], seg_dir=b["seg_dir"], seg_e1=b["seg_e1"],
                      seg_e2=b["seg_e2"], seg_len=b["seg_len"], seg_s0=b["seg_s0"],
                      seg_refl=b["seg_refl"], n_segs=b["n_segs"], n_refls=b["n_refls"],
                      max_seg=int(b["max_seg"]), weights=b["weights"], gamma1=b["gamma1"],
                      gamma2=b["gamma2"], c=float(b["c"]),
                      beam_param_im=float(b["beam_param_im"]),
                      amplitude_phi=float(b["amplitude_phi"]))


def test_async_calls_on_two_streams():
    """Asynchronous device calls on different caller streams share the engine's
    workspaces; each call is ordered after the previous one, so results equal the
    synchronous ones bit for bit."""
    import torch

    from paper_2501_13382_b200 import engine
    b = load_case("city_street")
    dev = torch.device("cuda", 0)
    db = engine.DeviceBundle.from_host(_pb(b), dev, with_frame=False)
    obs = torch.from_numpy(b["obs"]).to(dev)
    parts = [obs[0::2].contiguous(), obs[1::2].contiguous().flip(0).contiguous()]
    want = []
    for o in parts:
        acc = torch.zeros((o.shape[0], 1), dtype=torch.complex128, device=dev)
        ev = torch.zeros(o.shape[0], dtype=torch.int64, device=dev)
        engine.accumulate(db, o, b["omegas"], 10.0, True, acc, ev, precision="fp32")
        torch.cuda.synchronize()
        want.append((acc.clone(), ev.clone()))
    streams = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]
    got = []
    for rep in range(3):
        for o, s in zip(parts, streams):
            acc = torch.zeros((o.shape[0], 1), dtype=torch.complex128, device=dev)
            ev = torch.zeros(o.shape[0], dtype=torch.int64, device=dev)
            s.wait_stream(torch.cuda.current_stream(dev))
            with torch.cuda.stream(s):
                engine.accumulate(db, o, b["omegas"], 10.0, True, acc, ev, precision="fp32",
                                  stream=s)
            got.append((acc, ev))
    torch.cuda.synchronize()
    for i, (acc, ev) in enumerate(got):
        assert torch.equal(acc, want[i % 2][0]) and torch.equal(ev, want[i % 2][1])


def test_run_pipeline_city_vs_oracle():
    """run_pipeline (GPU trace + GPU sum, uncalibrated) vs the oracle on the same bundle."""
    from paper_2501_13382_b200 import (Atmosphere, ExecPlan, LaunchGrid, ObserverSet,
                                       SourceSpec, TraceConfig, make_city, parallel)
    z = np.load("tests/golden/city_street.npz")
    b = load_case("city_street")
    sc = make_city(5, 10, 40.0, 20.0, 300.0)
    src = SourceSpec(position=z["src"], frequencies=(125.0,), beam_param_im=-10.0)
    res, t = parallel.run_pipeline(sc, src, LaunchGrid(n_theta=32, n_phi=64),
                                   TraceConfig(5000, 1e-4, 8), ObserverSet(b["obs"]),
                                   ExecPlan(memory_budget=700 * 1080, per_ray_bytes=1080),
                                   Atmosphere(20.0), calibration=1.0)
    assert rel_l2(res.pressure, b["acc"]) <= FP32_L2
    assert tl_db(res.pressure, b["acc"], -60.0) <= FP32_TL_DB
    assert t.gbs_seconds > 0 and t.rt_seconds > 0
    assert abs(t.gbs_evaluations - int(b["evals"].sum())) <= 1e-4 * b["evals"].sum() + 10


def test_calibrate_phi_vs_reference():
    from paper_2501_13382_b200 import Atmosphere, SourceSpec, gbs
    z = np.load("tests/golden/calibration_origin.npz")
    b = oracle.load_bundle("tests/golden/calibration_origin.npz")
    pb = _pb(dict(b, gamma1=np.zeros(len(b["n_segs"])), gamma2=np.zeros(len(b["n_segs"])),
                  n_refls=b["n_refls"]))
    src = SourceSpec(position=np.zeros(3), frequencies=(500.0,), beam_param_im=-12.0)
    for prec, tol in (("fp64", 1e-12), ("fp32", 1e-5)):
        scale = gbs.calibrate_phi(pb, Atmosphere(20.0), src, precision=prec)
        assert abs(scale / float(z["scale"]) - 1) <= tol
        p = gbs.sum_at_observer(z["probe"], pb, src.omegas[0], Atmosphere(20.0), src,
                                precision=prec)
        assert abs(p - complex(z["probe_p"])) <= tol * abs(complex(z["probe_p"]))


@pytest.mark.parametrize("name,dense", [("city_street", False), ("city_street", True),
                                        ("city_corner_f5", True), ("cfg1_open_plane", True),
                                        ("city_street_nocut", True)])
def test_worklist_bitexact_vs_oracle(name, dense):
    """Device work list (tile, beam) candidates == the C restatement, bit for bit."""
    import ctypes

    from paper_2501_13382_b200 import _lib
    b = load_case(name)
    obs = b["obs"]
    if dense:  # config-3 receiver spacing (0.25 m): small tiles, non-trivial candidate sets
        x = np.arange(160) * 0.25 - 20.0
        X, Y = np.meshgrid(x, x, indexing="xy")
        obs = np.stack([X.ravel(), Y.ravel(), np.full(X.size, 1.8)], axis=1)
    n = obs.shape[0]
    nb = b["n_segs"].shape[0]
    T = int(_lib.load().bf_tile_size())
    nt = -(-n // T)
    perm = np.zeros(n, np.int32)
    centre = np.zeros((nt, 4))
    box = np.zeros((nt, 4))
    bits = np.zeros((nt, -(-nb // 32)), np.uint32)
    tbits = np.zeros_like(bits)
    got = ctypes.c_int64(0)
    keep = []  # the arrays must outlive the call

    def p(a):
        a = np.ascontiguousarray(a)
        keep.append(a)
        return ctypes.c_void_p(a.ctypes.data)

    use_cut = bool(b["use_cutoff"])
    _lib.check(_lib.load().bf_worklist(
        p(b["seg_origin"]), p(b["seg_dir"]), p(b["seg_len"]), p(b["seg_s0"]),
        p(b["n_segs"].astype(np.int32)), nb, int(b["max_seg"]), p(obs), n, p(b["omegas"]),
        b["omegas"].shape[0], float(b["c"]), -float(b["beam_param_im"]), int(use_cut),
        ctypes.c_void_p(perm.ctypes.data), ctypes.c_void_p(centre.ctypes.data),
        ctypes.c_void_p(box.ctypes.data),
        ctypes.c_void_p(bits.ctypes.data), ctypes.c_void_p(tbits.ctypes.data), nt,
        ctypes.byref(got), 0))
    assert got.value == nt
    assert np.array_equal(np.sort(perm), np.arange(n))
    ref = oracle.worklist(b["seg_origin"], b["seg_dir"], b["seg_len"], b["seg_s0"],
                          b["n_segs"], b["max_seg"], centre, float(b["c"]),
                          -float(b["beam_param_im"]), b["omegas"].min(), use_cut)
    assert np.array_equal(bits, ref)
    tref = oracle.worklist(b["seg_origin"], b["seg_dir"], b["seg_len"], b["seg_s0"],
                           b["n_segs"], b["max_seg"], centre, float(b["c"]),
                           -float(b["beam_param_im"]), b["omegas"].min(), use_cut, tight=True,
                           box=box)
    # the boxes are the tiles' coordinate ranges about their centres
    assert np.all(box[:, :3] >= 0) and np.all(box[:, :3] <= box[:, 3:4] * (1 + 1e-6) + 1e-9)
    assert np.array_equal(tbits, tref)
    assert not (tbits & ~bits).any()  # tight list is a subset of the a9 list
    # the tile radius bounds every member's distance from the centre (fp64, no rounding
    # below it: the cut tests rely on it)
    so = obs[perm]
    for t in range(nt):
        d = np.sqrt(((so[t * T:(t + 1) * T] - centre[t, :3]) ** 2).sum(axis=1))
        assert d.max() <= centre[t, 3], (t, d.max(), centre[t, 3])
    if dense:
        assert 0 < np.unpackbits(bits.view(np.uint8)).mean() < 1


@pytest.mark.parametrize("freqs,src,corner,im_b", [
    ((125.0,), (20.0, 0.0, 2.0), (-10.0, -20.0), -10.0),
    ((63.0, 250.0, 1000.0), (0.0, 20.0, 2.0), (-30.0, 5.0), -10.0),
    ((50.0, 63.0, 80.0, 100.0, 125.0, 160.0, 200.0, 250.0), (20.0, 0.0, 2.0), (10.0, -5.0),
     -10.0),
    # the paper's beam parameter: the cutoff never fires, every non-behind pair evaluated
    ((125.0,), (20.0, 0.0, 2.0), (-10.0, -20.0), -45874.0),
    # frequencies not in ascending order (no early exit of the frequency loop)
    ((500.0, 63.0, 250.0, 125.0), (0.0, 20.0, 2.0), (-30.0, 5.0), -10.0)])
def test_fp32_dense_city_vs_oracle(freqs, src, corner, im_b, threads):
    """Config-3 receiver density (0.25 m) around street corners of the city scene: every
    fp32 path (single survivor, corner wedge, several candidates with junction and
    general fp64 re-decisions, behind plane) against the C oracle on the same traced
    bundle (device tracer, bit-exact with the reference tracer)."""
    import torch

    from paper_2501_13382_b200 import _lib, engine, kernels
    from paper_2501_13382_b200.beamtrace import (Atmosphere, LaunchGrid, SourceSpec,
                                                 TraceConfig, launch_directions)
    from paper_2501_13382_b200.scene import make_city
    dev = torch.device("cuda", 0)
    sc = make_city(5, 10, 40.0, 20.0, 300.0)
    source = SourceSpec(position=np.array(src), frequencies=freqs, beam_param_im=im_b)
    launch = launch_directions(LaunchGrid(0.0, 180.0, 0.0, 360.0, 60, 120))
    cfg = TraceConfig(5000, 1e-4, 8)
    c = Atmosphere(20.0).sound_speed
    tr = engine.trace_device_rows(engine.DeviceScene.from_scene(sc, dev), source, launch, cfg,
                                  c, 0, len(launch), dev)
    hb = tr["bundle"].to_host()
    x = corner[0] + np.arange(96) * 0.25
    y = corner[1] + np.arange(96) * 0.25
    X, Y = np.meshgrid(x, y, indexing="xy")
    obs = np.ascontiguousarray(np.stack([X.ravel(), Y.ravel(), np.full(X.size, 1.8)], axis=1))
    om = source.omegas
    args = [hb.seg_origin, hb.seg_dir, hb.seg_e1, hb.seg_e2, hb.seg_len, hb.seg_s0,
            hb.seg_refl, hb.n_segs, hb.max_seg, hb.weights, obs, om, float(c),
            -float(source.beam_param_im), float(source.amplitude_phi), True]
    nb = hb.n_segs.shape[0]
    ref = np.zeros((obs.shape[0], om.shape[0]), np.complex128)
    rev = np.zeros(obs.shape[0], np.int64)
    oracle.gbs_accumulate(*args, ref, rev, 0, obs.shape[0], 0, nb, threads=threads)
    acc = np.zeros_like(ref)
    ev = np.zeros_like(rev)
    kernels.gbs_accumulate(*args, acc, ev, 0, obs.shape[0], 0, nb, precision="fp32")
    st = _lib.last_stats()
    assert rel_l2(acc, ref) <= FP32_L2
    assert tl_db(acc, ref, floor_db=-60.0) <= FP32_TL_DB
    assert tl_db(acc, ref) <= FP32_TL_ALL_DB
    assert abs(int(ev.sum()) - int(rev.sum())) <= 1e-4 * int(rev.sum()) + 10
    # the scene exercises the exact-decision paths
    assert st["patch_beams"]["wedge"] > 0 and st["patch_beams"]["multi"] > 0
    assert st["tie_pairs"] > 0


def test_max_seg_limit():
    """The fp32 path packs survivor masks with two flag bits: max_seg <= 30."""
    from paper_2501_13382_b200 import kernels
    b = load_case("cfg1_open_plane")
    nb, S = b["n_segs"].shape[0], 31
    pad = lambda a, w: np.zeros((nb * S,) + ((w,) if w else ()))  # noqa: E731
    args = [pad(0, 3), pad(0, 3), pad(0, 3), pad(0, 3), pad(0, 0), pad(0, 0), pad(0, 0),
            np.ones(nb, np.int32), S, b["weights"], b["obs"][:4], b["omegas"], float(b["c"]),
            -float(b["beam_param_im"]), 1.0, True]
    acc = np.zeros((4, 1), np.complex128)
    ev = np.zeros(4, np.int64)
    with pytest.raises(ValueError):
        kernels.gbs_accumulate(*args, acc, ev, 0, 4, 0, nb, precision="fp32")


@pytest.mark.parametrize("kind", ["one", "coincident", "vertical", "on_source"])
def test_fp32_degenerate_receiver_sets(kind):
    """Patch geometry corner cases of the fp32 path (zero-extent boxes, a lone receiver,
    non-planar patches, receivers at the source where segment 0's launch plane, ties and
    q = 0 meet) against the oracle."""
    from paper_2501_13382_b200 import kernels
    b = load_case("city_street")
    src = np.asarray(b["seg_origin"][0], float)  # segment 0 of beam 0 starts at the source
    if kind == "one":
        obs = np.array([[3.0, -4.0, 1.8]])
    elif kind == "coincident":
        obs = np.tile([[5.0, 1.0, 1.8]], (130, 1))
    elif kind == "vertical":
        obs = np.stack([np.full(200, 12.0), np.full(200, 3.0), np.linspace(0.1, 30.0, 200)], 1)
    else:
        obs = src[None, :] + np.linspace(-1e-3, 1e-3, 64)[:, None] * np.array([1.0, 0.5, 0.25])
    obs = np.ascontiguousarray(obs)
    nb = b["n_segs"].shape[0]
    acc = np.zeros((obs.shape[0], 1), np.complex128)
    ev = np.zeros(obs.shape[0], np.int64)
    kernels.gbs_accumulate(*gbs_args(b, obs), acc, ev, 0, obs.shape[0], 0, nb, precision="fp32")
    ref = np.zeros_like(acc)
    rev = np.zeros_like(ev)
    oracle.gbs_accumulate(*gbs_args(b, obs), ref, rev, 0, obs.shape[0], 0, nb)
    assert np.all(np.isfinite(acc))
    assert rel_l2(acc, ref) <= FP32_L2
    assert abs(int(ev.sum()) - int(rev.sum())) <= 1e-4 * int(rev.sum()) + 10


def test_run_snapshots_energy_mean():
    """run_snapshots == one run_pipeline per source; energy-mean SPL of the fields."""
    from paper_2501_13382_b200 import (Atmosphere, ExecPlan, LaunchGrid, ObserverSet,
                                       SourceSpec, TraceConfig, make_city, parallel)
    from paper_2501_13382_b200.gbs import P_REF
    sc = make_city(5, 10, 40.0, 20.0, 300.0)
    srcs = [SourceSpec(position=np.array([20.0 + 5 * k, 0.0, 2.0]), frequencies=(125.0,),
                       beam_param_im=-10.0) for k in range(3)]
    x = np.arange(40) * 0.5 - 10.0
    X, Y = np.meshgrid(x, x, indexing="xy")
    pts = np.stack([X.ravel(), Y.ravel(), np.full(X.size, 1.8)], 1)
    args = (LaunchGrid(n_theta=32, n_phi=64), TraceConfig(5000, 1e-4, 8), ObserverSet(pts),
            ExecPlan(), Atmosphere(20.0))
    fields, spl_mean, tims = parallel.run_snapshots(sc, srcs, *args, calibration=1.0)
    assert len(fields) == 3 and len(tims) == 3
    for src, f in zip(srcs, fields):
        res, _ = parallel.run_pipeline(sc, src, *args, calibration=1.0)
        assert np.array_equal(res.pressure, f.pressure)
    e = sum(np.abs(f.pressure) ** 2 for f in fields) / 3
    assert np.allclose(spl_mean, 10 * np.log10(e / P_REF ** 2), equal_nan=True)


@pytest.mark.parametrize("seed", range(8))
def test_fp32_random_city_vs_oracle(seed, threads):
    """Seeded random configurations (city layout, source in a street, frequency set,
    beam parameter, cutoff on/off, receivers: a 0.25 m grid patch plus scattered points
    at random heights, some inside buildings), fp32 path vs the C oracle on the same
    device-traced bundle.  Ragged receiver counts exercise partial tiles and patches."""
    import torch

    from paper_2501_13382_b200 import engine, kernels
    from paper_2501_13382_b200.beamtrace import (Atmosphere, LaunchGrid, SourceSpec,
                                                 TraceConfig, launch_directions)
    from paper_2501_13382_b200.scene import make_city
    rng = np.random.default_rng(1000 + seed)
    dev = torch.device("cuda", 0)
    nx, ny = int(rng.integers(2, 6)), int(rng.integers(2, 8))
    sc = make_city(nx, ny, 40.0, 20.0, 300.0)
    # a street along y between building columns (buildings span +-10 m around centres)
    x_streets = -(nx - 1) * 20.0 + 20.0 + 40.0 * np.arange(nx - 1)
    src = np.array([rng.choice(x_streets) + rng.uniform(-4, 4), rng.uniform(-60, 60),
                    rng.uniform(1.0, 12.0)])
    nf = int(rng.integers(1, 4))
    freqs = tuple(float(f) for f in np.sort(rng.choice([63.0, 125.0, 250.0, 500.0], nf,
                                                       replace=False)))
    im_b = float(rng.choice([-5.0, -10.0, -25.0, -45874.0]))
    use_cutoff = bool(rng.integers(0, 4) > 0)
    source = SourceSpec(position=src, frequencies=freqs, beam_param_im=im_b)
    launch = launch_directions(LaunchGrid(0.0, 180.0, 0.0, 360.0, int(rng.integers(30, 70)),
                                          int(rng.integers(60, 140))))
    cfg = TraceConfig(5000, 1e-4, int(rng.integers(2, 9)))
    c = Atmosphere(float(rng.uniform(0, 30))).sound_speed
    tr = engine.trace_device_rows(engine.DeviceScene.from_scene(sc, dev), source, launch, cfg,
                                  c, 0, len(launch), dev)
    hb = tr["bundle"].to_host()
    n1, n2 = int(rng.integers(20, 70)), int(rng.integers(20, 70))
    x0 = src[0] + rng.uniform(-40, 20)
    y0 = src[1] + rng.uniform(-40, 20)
    X, Y = np.meshgrid(x0 + 0.25 * np.arange(n1), y0 + 0.25 * np.arange(n2), indexing="xy")
    grid = np.stack([X.ravel(), Y.ravel(), np.full(X.size, rng.uniform(0.5, 3.0))], axis=1)
    m = int(rng.integers(100, 3000))
    scat = np.stack([src[0] + rng.uniform(-80, 80, m), src[1] + rng.uniform(-80, 80, m),
                     rng.uniform(0.2, 15.0, m)], axis=1)
    obs = np.ascontiguousarray(np.concatenate([grid, scat]))
    om = source.omegas
    args = [hb.seg_origin, hb.seg_dir, hb.seg_e1, hb.seg_e2, hb.seg_len, hb.seg_s0,
            hb.seg_refl, hb.n_segs, hb.max_seg, hb.weights, obs, om, float(c),
            -float(source.beam_param_im), float(source.amplitude_phi), use_cutoff]
    nb = hb.n_segs.shape[0]
    ref = np.zeros((obs.shape[0], om.shape[0]), np.complex128)
    rev = np.zeros(obs.shape[0], np.int64)
    oracle.gbs_accumulate(*args, ref, rev, 0, obs.shape[0], 0, nb, threads=threads)
    acc = np.zeros_like(ref)
    ev = np.zeros_like(rev)
    kernels.gbs_accumulate(*args, acc, ev, 0, obs.shape[0], 0, nb, precision="fp32")
    assert rel_l2(acc, ref) <= FP32_L2
    assert tl_db(acc, ref, floor_db=-60.0) <= FP32_TL_DB
    assert tl_db(acc, ref) <= FP32_TL_ALL_DB
    assert abs(int(ev.sum()) - int(rev.sum())) <= 1e-4 * int(rev.sum()) + 10


@pytest.mark.parametrize("n1,n2", [(100, 37), (1000, 40), (333, 333), (37, 100)])
def test_tile_order_compact_patches(n1, n2):
    """The receiver order (bf_tile_order_dev) has no jumps on rectangular grids, so every
    128-receiver patch is a compact blob (0.25 m grid: radius <= 4 m; Morton order and an
    isotropic single Hilbert square left 12-60 m patches across jumps)."""
    import torch

    from paper_2501_13382_b200 import shard
    X, Y = np.meshgrid(np.arange(n1) * 0.25 - 7.0, np.arange(n2) * 0.25 + 3.0, indexing="xy")
    P = np.stack([X.ravel(), Y.ravel(), np.full(X.size, 1.5)], axis=1)
    order = shard.tile_order(torch.from_numpy(P).to("cuda:0")).cpu().numpy()
    assert np.array_equal(np.sort(order), np.arange(P.shape[0]))
    Q = P[order]
    for p in range(Q.shape[0] // 128):
        B = Q[128 * p:128 * (p + 1)]
        c = 0.5 * (B.min(0) + B.max(0))
        assert np.sqrt(((B - c) ** 2).sum(1).max()) <= 4.0


@pytest.mark.parametrize("src", [(0.0, 20.0, 2.0), (-37.0, 3.0, 25.0), (150.0, -260.0, 1.0)])
def test_tracer_cluster_culling_equals_exhaustive(src):
    """The tracer's triangle-cluster culling returns the same bits as testing every
    triangle (config-4 city: 500 buildings, 5002 triangles, up to 8 reflections)."""
    import torch

    from paper_2501_13382_b200 import engine
    from paper_2501_13382_b200.beamtrace import (Atmosphere, LaunchGrid, SourceSpec,
                                                 TraceConfig, launch_directions)
    from paper_2501_13382_b200.scene import make_city
    dev = torch.device("cuda", 0)
    sc = make_city(20, 25, 40.0, 20.0, 600.0)
    source = SourceSpec(position=np.array(src), frequencies=(125.0,), beam_param_im=-10.0)
    launch = launch_directions(LaunchGrid(0.0, 180.0, 0.0, 360.0, 90, 180))
    cfg = TraceConfig(5000, 1e-4, 8)
    c = Atmosphere(20.0).sound_speed
    ds = engine.DeviceScene.from_scene(sc, dev)
    out = {}
    for mode in (False, True):
        out[mode] = engine.trace_device_rows(ds, source, launch, cfg, c, 0, len(launch), dev,
                                             exhaustive=mode)
        torch.cuda.synchronize()
    a, b = out[False]["bundle"], out[True]["bundle"]
    for name in ("seg_origin", "seg_dir", "seg_e1", "seg_e2", "seg_len", "seg_s0", "seg_refl",
                 "n_segs", "n_refls"):
        assert torch.equal(getattr(a, name), getattr(b, name)), name
    assert int(a.n_refls.max()) >= 2  # the rays do bounce between buildings


@pytest.mark.parametrize("case", ["city_street", "city_corner_f5"])
def test_repeated_small_calls_replay_a_graph_bitexact(case):
    """Identical small device calls: the first runs eagerly, the second is captured into a
    CUDA graph, later ones replay it (engine.cu run_fp32_graph).  The sequence must equal,
    bit for bit, the same calls made with a changing memory budget (a different key every
    call, so always eager; the budget never changes a one-group call's bits), statistics
    included; a call that reallocates the workspaces in between invalidates the graph."""
    import torch

    from paper_2501_13382_b200 import _lib, kernels
    b = load_case(case)
    dev = torch.device("cuda", 0)
    t = lambda a, dt=torch.float64: torch.as_tensor(np.ascontiguousarray(a)).to(dev, dt)  # noqa
    args = [t(b["seg_origin"]), t(b["seg_dir"]), t(b["seg_e1"]), t(b["seg_e2"]),
            t(b["seg_len"]), t(b["seg_s0"]), t(b["seg_refl"]), t(b["n_segs"], torch.int32),
            b["max_seg"], t(b["weights"]), t(b["obs"]), b["omegas"], float(b["c"]),
            -float(b["beam_param_im"]), 1.0, True]
    n_obs, nb = b["obs"].shape[0], b["n_segs"].shape[0]

    def sequence(budgets, big_after=None):
        nf = b["omegas"].shape[0]
        acc = torch.zeros((n_obs, nf), dtype=torch.complex128, device=dev)
        ev = torch.zeros(n_obs, dtype=torch.int64, device=dev)
        out, evs = [], []
        for i, bud in enumerate(budgets):
            _lib.set_memory_budget(0, bud)
            kernels.gbs_accumulate(*args, acc, ev, 0, n_obs, 0, nb, precision="fp32")
            out.append(acc.cpu().numpy().copy())
            st = _lib.last_stats()
            evs.append((st["tie_pairs"], st["nonbehind_pairs"], st["tight_pairs"],
                        tuple(st["patch_beams"].values())))
            if big_after == i:  # a larger call grows the workspaces (new generation)
                big = torch.cat([args[10]] * 4)
                a2 = torch.zeros((big.shape[0], nf), dtype=torch.complex128, device=dev)
                e2 = torch.zeros(big.shape[0], dtype=torch.int64, device=dev)
                kernels.gbs_accumulate(*args[:10], big, *args[11:], a2, e2, 0, big.shape[0],
                                       0, nb, precision="fp32")
        _lib.set_memory_budget(0, 0)
        return out, evs

    n0 = _lib.launch_count()
    ref, ref_st = sequence([(1 << 30) + i for i in range(5)])  # always eager
    n_eager = _lib.launch_count() - n0
    n0 = _lib.launch_count()
    got, got_st = sequence([1 << 30] * 5)                      # eager, capture, 3 replays
    assert _lib.launch_count() - n0 == n_eager  # replays count the graph's kernels
    for r, g in zip(ref, got):
        assert np.array_equal(r, g)
    assert ref_st == got_st
    got2, _ = sequence([1 << 30] * 5, big_after=2)             # graph invalidated midway
    for r, g in zip(ref, got2):
        assert np.array_equal(r, g)


@pytest.mark.gpu
def test_kernel_timing_switch_changes_no_bits():
    """bf_set_kernel_timing: kernel_ms is 0 while off (the default: no event nodes in a small
    call) and positive while on; the results, statistics and graph replays are identical
    either way (the switch is part of the graph key)."""
    import torch

    from paper_2501_13382_b200 import _lib, kernels
    b = load_case("city_street")
    dev = torch.device("cuda", 0)
    t = lambda a, dt=torch.float64: torch.as_tensor(np.ascontiguousarray(a)).to(dev, dt)  # noqa
    args = [t(b["seg_origin"]), t(b["seg_dir"]), t(b["seg_e1"]), t(b["seg_e2"]),
            t(b["seg_len"]), t(b["seg_s0"]), t(b["seg_refl"]), t(b["n_segs"], torch.int32),
            b["max_seg"], t(b["weights"]), t(b["obs"]), b["omegas"], float(b["c"]),
            -float(b["beam_param_im"]), 1.0, True]
    n_obs, nb, nf = b["obs"].shape[0], b["n_segs"].shape[0], b["omegas"].shape[0]
    runs = {}
    try:
        for on in (False, True, False, True):
            _lib.set_kernel_timing(on)
            res = []
            for _ in range(4):  # eager, capture, replays
                acc = torch.zeros((n_obs, nf), dtype=torch.complex128, device=dev)
                ev = torch.zeros(n_obs, dtype=torch.int64, device=dev)
                kernels.gbs_accumulate(*args, acc, ev, 0, n_obs, 0, nb, precision="fp32")
                st = _lib.last_stats()
                res.append((acc.cpu().numpy(), ev.cpu().numpy(), st["tie_pairs"],
                            st["nonbehind_pairs"]))
                assert (st["kernel_ms"] > 0) == on
            runs.setdefault(on, []).append(res)
    finally:
        _lib.set_kernel_timing(False)
    ref = runs[False][0][0]
    for on in (False, True):
        for res in runs[on]:
            for r in res:
                assert np.array_equal(r[0], ref[0]) and np.array_equal(r[1], ref[1])
                assert r[2:] == ref[2:]

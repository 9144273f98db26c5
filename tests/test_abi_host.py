"""CPU-side checks: the C ABI library loads and exports every declared symbol,
and the host-side mirror of the reference API behaves like the reference."""
import ctypes
import re

import numpy as np
import pytest

from conftest import GOLDEN, ROOT, load_case
from paper_2501_13382_b200 import _lib, beamtrace, gbs, parallel, scene, shard
from paper_2501_13382_b200.errors import BudgetError

HEADER = ROOT / "include" / "bf_gbs.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w]+\s*\*?\s*(bf_\w+)\s*\(", text, re.M)))


def test_header_declares_and_lib_exports_everything():
    syms = declared_symbols()
    assert "bf_gbs_accumulate" in syms and "bf_gbs_accumulate_dev" in syms
    assert set(syms) == set(_lib.EXPORTS)
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    for s in syms:
        assert hasattr(lib, s), s


def test_version_and_no_device_fails_loudly():
    lib = _lib.load()
    assert b"sm_100a" in lib.bf_version()
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    b = load_case("open_paper_imb")
    from paper_2501_13382_b200 import kernels
    acc = np.zeros((4, 1), np.complex128)
    ev = np.zeros(4, np.int64)
    with pytest.raises(RuntimeError, match="no CUDA device"):
        kernels.gbs_accumulate(b["seg_origin"], b["seg_dir"], b["seg_e1"], b["seg_e2"],
                               b["seg_len"], b["seg_s0"], b["seg_refl"], b["n_segs"],
                               b["max_seg"], b["weights"], b["obs"][:4], b["omegas"], 343.0,
                               10.0, 1.0, True, acc, ev, 0, 4, 0, 10)


def test_plan_chunks_matches_reference_semantics():
    # 16384 rays under the paper budget -> [11364, 5020]
    per_ray = 2520
    budget = 11364 * per_ray + 100
    assert parallel.plan_chunks(16384, budget, per_ray).chunk_sizes == (11364, 5020)
    assert parallel.plan_chunks(10, 100, 10).chunk_sizes == (10,)
    assert parallel.plan_chunks(7, 30, 10).chunk_sizes == (3, 3, 1)
    with pytest.raises(BudgetError):
        parallel.plan_chunks(10, 5, 10)
    with pytest.raises(ValueError):
        parallel.plan_chunks(0, 5, 10)
    with pytest.raises(ValueError):
        parallel.plan_chunks(5, 5, 0)


def test_exec_plan_validation():
    with pytest.raises(ValueError):
        parallel.ExecPlan(mode="bogus")
    with pytest.raises(ValueError):
        parallel.ExecPlan(workers=0)
    with pytest.raises(ValueError):
        parallel.ExecPlan(memory_budget=10, per_ray_bytes=20)


@pytest.mark.parametrize("name", ["cfg1_open_plane", "city_street", "city_corner_f5"])
def test_launch_directions_bitexact(name):
    z = np.load(GOLDEN / f"{name}.npz")
    ls = beamtrace.launch_directions(beamtrace.LaunchGrid(0.0, 180.0, 0.0, 360.0,
                                                          int(z["n_theta"]), int(z["n_phi"])))
    for mine, ref in ((ls.directions, z["launch_dirs"]), (ls.e1, z["launch_e1"]),
                      (ls.e2, z["launch_e2"]), (ls.weights, z["launch_weights"])):
        assert np.array_equal(mine.view(np.uint64), np.asarray(ref).view(np.uint64))


@pytest.mark.parametrize("name", ["cfg1_open_plane", "city_street", "city_corner_f5"])
def test_scene_generators_bitexact(name):
    z = np.load(GOLDEN / f"{name}.npz")
    args = z["scene_args"]
    if str(z["scene_kind"]) == "plane":
        sc = scene.make_ground_plane(float(args[0]))
    else:
        sc = scene.make_city(int(args[0]), int(args[1]), float(args[2]), float(args[3]),
                             float(args[4]))
    for mine, ref in ((sc.v0, z["scene_v0"]), (sc.v1, z["scene_v1"]), (sc.v2, z["scene_v2"])):
        assert np.array_equal(mine, ref)


def test_observer_set_and_spl():
    with pytest.raises(ValueError):
        gbs.ObserverSet(np.zeros((0, 3)))
    with pytest.raises(ValueError):
        gbs.ObserverSet(np.array([[0.0, np.nan, 0.0]]))
    o = gbs.ObserverSet([1.0, 2.0, 3.0])
    assert o.points.shape == (1, 3) and o.count == 1
    assert gbs.spl(2e-5) == 0.0
    assert gbs.spl(0.0) == -np.inf
    p = np.array([[2e-4 + 0j], [0j]])
    s = gbs.spl(p)
    assert s[0, 0] == pytest.approx(20.0) and s[1, 0] == -np.inf


def test_bundle_from_paths_layout():
    b = load_case("city_street")
    pb = beamtrace.PathBundle(
        seg_origin=b["seg_origin"], seg_dir=b["seg_dir"], seg_e1=b["seg_e1"],
        seg_e2=b["seg_e2"], seg_len=b["seg_len"], seg_s0=b["seg_s0"], seg_refl=b["seg_refl"],
        n_segs=b["n_segs"], n_refls=b["n_refls"], max_seg=int(b["max_seg"]),
        weights=b["weights"], gamma1=b["gamma1"], gamma2=b["gamma2"], c=float(b["c"]),
        beam_param_im=float(b["beam_param_im"]), amplitude_phi=float(b["amplitude_phi"]))
    paths = [pb.path(i) for i in range(50)]
    rb = gbs.bundle_from_paths(paths)
    S = rb.max_seg
    assert S == max(len(p.segments) for p in paths)
    for i in range(50):
        n = int(rb.n_segs[i])
        assert n == int(pb.n_segs[i])
        src = slice(i * pb.max_seg, i * pb.max_seg + n)
        dst = slice(i * S, i * S + n)
        for f in ("seg_origin", "seg_dir", "seg_e1", "seg_e2", "seg_len", "seg_s0", "seg_refl"):
            assert np.array_equal(getattr(rb, f)[dst], getattr(pb, f)[src])
    with pytest.raises(ValueError):
        gbs.bundle_from_paths([])


def test_calibration_probes_order():
    p = gbs.calibration_probes(10.0)
    assert p.shape == (26, 3)
    assert np.allclose(np.linalg.norm(p, axis=1), 10.0)
    assert np.allclose(p[0], 10.0 * np.array([-1, -1, -1]) / np.sqrt(3))


@pytest.mark.parametrize("n,world", [(1000, 1), (1000, 2), (1000, 3), (256, 4), (5, 2),
                                     (1_000_003, 8)])
def test_rank_tiles_partition(n, world):
    parts = [shard.rank_tiles(n, r, world, tile=256) for r in range(world)]
    allp = np.concatenate(parts)
    assert np.array_equal(np.sort(allp), np.arange(n))
    for r, p in enumerate(parts):  # whole tiles, dealt round-robin
        if p.size:
            assert set(np.unique(p // 256) % world) == {r}


def test_field_csv_bytes_match_python_format(tmp_path):
    """bf_write_field_csv == the reference's row loop (harness.py:197-208): '%.17g'
    numbers incl. -inf SPL of null pressure, -0, tiny/huge magnitudes."""
    from paper_2501_13382_b200 import harness
    from paper_2501_13382_b200.gbs import FieldResult
    rng = np.random.default_rng(7)
    n, freqs = 40000, np.array([63.0, 125.0, 1000.0])
    pts = rng.normal(size=(n, 3)) * 100.0
    pts[0] = [-0.0, 1e-300, 1e300]
    p = (rng.normal(size=(n, 3)) + 1j * rng.normal(size=(n, 3))) * 10.0 ** rng.integers(-12, 3, (n, 3))
    p[5, 1] = 0.0
    field = FieldResult.from_pressure(p, 1.0)
    path = tmp_path / "field.csv"
    harness.write_field_csv(path, pts, freqs, field, threads=4)
    g = harness._g
    rows = [harness.FIELD_CSV_HEADER]
    for oi in range(n):
        x, y, z = pts[oi]
        for fi, f in enumerate(freqs):
            q = field.pressure[oi, fi]
            rows.append(f"{g(x)},{g(y)},{g(z)},{g(f)},{g(q.real)},{g(q.imag)},"
                        f"{g(field.spl[oi, fi])}")
    assert path.read_text() == "\n".join(rows) + "\n"
    with pytest.raises(OSError):
        harness.write_field_csv(tmp_path / "missing" / "x.csv", pts, freqs, field)


def test_heatmap(tmp_path):
    from paper_2501_13382_b200 import harness
    from PIL import Image

    class Grid:
        n1, n2 = 5, 3
    v = np.arange(15, dtype=float)
    v[4] = -np.inf
    meta = harness.emit_heatmap(v, Grid, tmp_path / "h.png")
    img = np.asarray(Image.open(tmp_path / "h.png"))
    assert img.shape == (3, 5) and img[0, 4] == 0 and img.max() == 255
    assert meta["null_points"] == 1 and meta["spl_min_db"] == 0.0 and meta["spl_max_db"] == 14.0
    assert (tmp_path / "h.png.txt").read_text().startswith("width=5\nheight=3\n")

"""The C oracle (oracle/gbs_oracle.c) pinned against the reference's own outputs.

tests/golden/*.npz were produced by executing the reference beamfield package
(tests/golden/make_golden.py); the oracle must reproduce them BIT-EXACTLY.
"""
import numpy as np
import pytest

import oracle
from conftest import CASES, gbs_args, load_case


@pytest.mark.parametrize("name", CASES)
def test_oracle_bitexact_vs_reference(name):
    b = load_case(name)
    obs = b["obs"]
    acc = np.zeros((obs.shape[0], b["omegas"].shape[0]), np.complex128)
    ev = np.zeros(obs.shape[0], np.int64)
    for olo, ohi, blo, bhi in b["calls"]:
        oracle.gbs_accumulate(*gbs_args(b), acc, ev, olo, ohi, blo, bhi, threads=4)
    assert np.array_equal(acc.view(np.uint64), b["acc"].view(np.uint64))
    assert np.array_equal(ev, b["evals"])


@pytest.mark.parametrize("name", ["cfg1_open_plane", "city_street", "city_corner_f5"])
def test_oracle_nearest_bitexact(name):
    b = load_case(name)
    obs = b["obs"]
    S = b["max_seg"]
    for j in range(0, b["ns_obs"].shape[0], 7):
        oi, bi = int(b["ns_obs"][j]), int(b["ns_beam"][j])
        ns = int(b["n_segs"][bi])
        if ns == 0:
            continue
        k, s, q1, q2, refl, behind = oracle.nearest_on_segments(
            b["seg_origin"], b["seg_dir"], b["seg_e1"], b["seg_e2"], b["seg_len"], b["seg_s0"],
            b["seg_refl"], bi * S, ns, *obs[oi])
        assert k == b["ns_k"][j]
        assert (s, q1, q2, refl) == (b["ns_s"][j], b["ns_q1"][j], b["ns_q2"][j], b["ns_refl"][j])
        assert behind == bool(b["ns_behind"][j])


def test_oracle_thread_count_invariance():
    b = load_case("city_street")
    obs = b["obs"][:700]
    res = []
    for t in (1, 3, 8):
        acc = np.zeros((obs.shape[0], 1), np.complex128)
        ev = np.zeros(obs.shape[0], np.int64)
        oracle.gbs_accumulate(*gbs_args(b, obs), acc, ev, 0, obs.shape[0], 0,
                              b["n_segs"].shape[0], threads=t)
        res.append(acc.copy())
    assert all(np.array_equal(r.view(np.uint64), res[0].view(np.uint64)) for r in res)


def test_oracle_chunked_beams_compose():
    """In-place continuation (kernels.py:358-359): beam chunks reproduce one call."""
    b = load_case("cfg1_open_plane")
    obs = b["obs"][::37]
    nb = b["n_segs"].shape[0]
    one = np.zeros((obs.shape[0], 1), np.complex128)
    ev1 = np.zeros(obs.shape[0], np.int64)
    oracle.gbs_accumulate(*gbs_args(b, obs), one, ev1, 0, obs.shape[0], 0, nb)
    two = np.zeros_like(one)
    ev2 = np.zeros_like(ev1)
    for lo, hi in ((0, 333), (333, 1500), (1500, nb)):
        oracle.gbs_accumulate(*gbs_args(b, obs), two, ev2, 0, obs.shape[0], lo, hi)
    assert np.array_equal(one.view(np.uint64), two.view(np.uint64))
    assert np.array_equal(ev1, ev2)


@pytest.mark.parametrize("name", ["cfg1_open_plane", "city_street", "city_corner_f5",
                                  "open_paper_imb"])
def test_oracle_tracer_bitexact_vs_reference(name):
    """C tracer restatement == reference trace_into bundles (exhaustive nearest hit vs BVH)."""
    z = np.load(f"tests/golden/{name}.npz")
    b = load_case(name)
    v0, v1, v2 = z["scene_v0"], z["scene_v1"], z["scene_v2"]
    allv = np.concatenate([v0, v1, v2])
    bounds = np.stack([allv.min(axis=0), allv.max(axis=0)])
    c = float(z["c"])
    out = oracle.trace(v0, v1, v2, np.ones(v0.shape[0]), bounds,
                       float(np.linalg.norm(bounds[1] - bounds[0])), z["src"], z["launch_dirs"],
                       z["launch_e1"], z["launch_e2"], int(z["n_steps"]) * float(z["dt"]) * c,
                       int(z["r_max"]), threads=4)
    assert np.array_equal(out["n_segs"], b["n_segs"])
    assert np.array_equal(out["n_refls"], z["n_refls"])
    for f in ("seg_origin", "seg_dir", "seg_e1", "seg_e2", "seg_len", "seg_s0", "seg_refl"):
        assert np.array_equal(out[f].view(np.uint64), b[f].view(np.uint64)), f


@pytest.mark.parametrize("tight", [False, True])
@pytest.mark.parametrize("name", ["city_street", "city_corner_f5", "cfg1_open_plane"])
def test_worklist_is_sound(name, tight):
    """Culled (tile, beam) pairs are pairs the reference skips: no receiver of a culled
    tile gets an evaluation from that beam (kernels.py:375,384-385)."""
    b = load_case(name)
    n1 = int(b["grid_n"][0])
    obs = b["obs"][: n1 * 32]
    # spatially compact 4x4 receiver blocks of the row-major grid
    tiles = [np.array([(j0 + dj) * n1 + i0 + di for dj in range(4) for di in range(4)])
             for j0 in range(0, 32, 4) for i0 in range(0, n1, 4)]
    centre, box = [], []
    for t in tiles:
        p = obs[t]
        c = 0.5 * (p.min(0) + p.max(0))
        rt = np.linalg.norm(p - c, axis=1).max()
        centre.append([*c, rt])
        box.append([*(0.5 * (p.max(0) - p.min(0))), rt])
    centre = np.array(centre)
    om = b["omegas"]
    bits = oracle.worklist(b["seg_origin"], b["seg_dir"], b["seg_len"], b["seg_s0"],
                           b["n_segs"], b["max_seg"], centre, float(b["c"]),
                           -float(b["beam_param_im"]), om.min(), True, tight=tight,
                           box=np.array(box))
    nb = b["n_segs"].shape[0]
    cand = np.unpackbits(bits.view(np.uint8), bitorder="little").reshape(len(tiles), -1)[:, :nb]
    assert 0 < cand.mean() < 1
    for bi in range(0, nb, 3):
        ev = np.zeros(obs.shape[0], np.int64)
        acc = np.zeros((obs.shape[0], om.shape[0]), np.complex128)
        oracle.gbs_accumulate(*gbs_args(b, obs), acc, ev, 0, obs.shape[0], bi, bi + 1)
        for ti, t in enumerate(tiles):
            if not cand[ti, bi]:
                assert not ev[t].any() and not acc[t].any()

import os
import pathlib
import sys

import numpy as np
import pytest

ROOT = pathlib.Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

CASES = ["cfg1_open_plane", "cfg1_chunked", "city_street", "city_street_nocut",
         "city_corner_f5", "open_paper_imb"]


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        have_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        have_gpu = False
    if have_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


def load_case(name):
    import oracle
    return oracle.load_bundle(GOLDEN / f"{name}.npz")


def gbs_args(b, obs=None):
    obs = b["obs"] if obs is None else obs
    return [b["seg_origin"], b["seg_dir"], b["seg_e1"], b["seg_e2"], b["seg_len"], b["seg_s0"],
            b["seg_refl"], b["n_segs"], b["max_seg"], b["weights"], obs, b["omegas"],
            float(b["c"]), -float(b["beam_param_im"]), float(b["amplitude_phi"]),
            bool(b["use_cutoff"]) if "use_cutoff" in b else True]


def tl_db(acc, ref, floor_db=None):
    """max |20 log10 |acc|/|ref||, optionally over receivers within floor_db of the max."""
    a = np.abs(acc)
    r = np.abs(ref)
    m = r > 0
    if floor_db is not None:
        m &= 20 * np.log10(np.maximum(r, 1e-300) / r.max()) > floor_db
    return float(np.max(np.abs(20 * np.log10(a[m] / r[m])))) if m.any() else 0.0


def rel_l2(acc, ref):
    return float(np.linalg.norm(acc - ref) / np.linalg.norm(ref))


@pytest.fixture(scope="session")
def threads():
    return len(os.sched_getaffinity(0))

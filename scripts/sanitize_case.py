#!/usr/bin/env python3
# Small fp32 + fp64 calls for compute-sanitizer: config 1 (golden) and a city corner subset.
import sys, numpy as np
import os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, 'tests'))
from conftest import load_case, gbs_args
from paper_2501_13382_b200 import kernels
for name, n in (("cfg1_open_plane", 4096), ("city_corner_f5", 3000)):
    b = load_case(name)
    obs = np.ascontiguousarray(b["obs"][:n])
    nb = b["n_segs"].shape[0]
    for prec in ("fp32", "fp64"):
        acc = np.zeros((obs.shape[0], b["omegas"].shape[0]), np.complex128)
        ev = np.zeros(obs.shape[0], np.int64)
        kernels.gbs_accumulate(*gbs_args(b, obs), acc, ev, 0, obs.shape[0], 0, nb, precision=prec)
        print(name, prec, float(np.abs(acc).sum()), int(ev.sum()), flush=True)
# wide patches (scattered receivers), no cutoff (TINY kernels), grouped host streaming
from paper_2501_13382_b200 import _lib
b = load_case("city_street")
rng = np.random.default_rng(4)
obs = np.ascontiguousarray(np.stack([rng.uniform(-80, 80, 2500), rng.uniform(-80, 80, 2500), rng.uniform(0, 20, 2500)], 1))
nb = b["n_segs"].shape[0]
for cut in (True, False):
    a = gbs_args(b, obs); a[-1] = cut
    acc = np.zeros((obs.shape[0], 1), np.complex128); ev = np.zeros(obs.shape[0], np.int64)
    kernels.gbs_accumulate(*a, acc, ev, 0, obs.shape[0], 0, nb, precision="fp32")
    print("scattered cut", cut, float(np.abs(acc).sum()), int(ev.sum()), _lib.last_stats()["n_tiles"], flush=True)
_lib.set_memory_budget(0, 1 << 20)
acc = np.zeros((obs.shape[0], 1), np.complex128); ev = np.zeros(obs.shape[0], np.int64)
kernels.gbs_accumulate(*gbs_args(b, obs), acc, ev, 0, obs.shape[0], 0, nb, precision="fp32")
print("budget 1 MiB", float(np.abs(acc).sum()), int(ev.sum()), flush=True)
_lib.set_memory_budget(0, 0)
# device ABI on torch's default stream (fenced onto the engine stream), repeated identical
# calls: eager, captured, replayed graph; statistics read back on the side stream
import torch
from paper_2501_13382_b200 import engine
from paper_2501_13382_b200.beamtrace import PathBundle
b = load_case("cfg1_open_plane")
pb = PathBundle(seg_origin=b["seg_origin"], seg_dir=b["seg_dir"], seg_e1=b["seg_e1"],
                seg_e2=b["seg_e2"], seg_len=b["seg_len"], seg_s0=b["seg_s0"],
                seg_refl=b["seg_refl"], n_segs=b["n_segs"], n_refls=b["n_refls"],
                max_seg=int(b["max_seg"]), weights=b["weights"], gamma1=b["gamma1"],
                gamma2=b["gamma2"], c=float(b["c"]), beam_param_im=float(b["beam_param_im"]),
                amplitude_phi=float(b["amplitude_phi"]))
dev = torch.device("cuda", 0)
db = engine.DeviceBundle.from_host(pb, dev, with_frame=False)
od = torch.from_numpy(np.ascontiguousarray(b["obs"][:4096])).to(dev)
acc = torch.zeros((od.shape[0], 1), dtype=torch.complex128, device=dev)
ev = torch.zeros(od.shape[0], dtype=torch.int64, device=dev)
for i in range(4):
    acc.zero_()
    ev.zero_()
    engine.accumulate(db, od, b["omegas"], -float(b["beam_param_im"]), True, acc, ev)
    st = _lib.last_stats()
    print("device call", i, float(acc.abs().sum()), int(ev.sum()), st["n_tiles"], flush=True)

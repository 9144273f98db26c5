"""GPU timeline of one host-buffer (e2e) call on pageable numpy inputs (bench's e2e leg):
kernels and copies with the idle gap before each, from CUPTI records (torch.profiler).
    python scripts/e2e_timeline.py [cfg3]"""
import json
import os
import sys
import tempfile

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2501_13382_b200 import engine, kernels  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
sc, src, launch, tcfg, c, obs = bench.make_inputs(dict(bench.CONFIGS[name]))
dev = torch.device("cuda", 0)
b = engine.trace_device_rows(engine.DeviceScene.from_scene(sc, dev), src, launch, tcfg, c, 0,
                             len(launch), dev)["bundle"]
torch.cuda.synchronize()
om = src.omegas
nb = b.n_segs.shape[0]
hb = {k: getattr(b, k).cpu().numpy().copy() for k in engine.SEG_FIELDS + ("n_segs", "weights")}
acc = np.zeros((obs.shape[0], len(om)), np.complex128)
ev = np.zeros(obs.shape[0], np.int64)


def call():
    kernels.gbs_accumulate(hb["seg_origin"], hb["seg_dir"], hb["seg_e1"], hb["seg_e2"],
                           hb["seg_len"], hb["seg_s0"], hb["seg_refl"], hb["n_segs"], b.max_seg,
                           hb["weights"], obs, om, c, -src.beam_param_im, src.amplitude_phi,
                           True, acc, ev, 0, obs.shape[0], 0, nb, precision="fp32")


for _ in range(2):
    call()
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    call()
    torch.cuda.synchronize()
path = os.path.join(tempfile.mkdtemp(), "t.json")
prof.export_chrome_trace(path)
evs = [e for e in json.load(open(path))["traceEvents"]
       if e.get("cat") in ("kernel", "gpu_memset", "gpu_memcpy")]
evs.sort(key=lambda e: e["ts"])
t0 = evs[0]["ts"]
end_prev = t0
print(f"{name}: one pageable host-buffer call's GPU timeline (ms; gap = idle before)")
for e in evs:
    gap = e["ts"] - end_prev
    if e["dur"] > 50 or gap > 50:
        print(f"{(e['ts'] - t0) / 1e3:9.3f} {e['dur'] / 1e3:8.3f} gap {gap / 1e3:7.3f}  "
              f"{e['name'][:70]}")
    end_prev = max(end_prev, e["ts"] + e["dur"])
busy = sum(e["dur"] for e in evs if e.get("cat") == "kernel" and "gbs_fp32_kernel" in e["name"])
print(f"span {(end_prev - t0) / 1e3:.3f} ms, summation kernels {busy / 1e3:.3f} ms")

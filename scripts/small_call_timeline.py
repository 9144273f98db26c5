"""GPU timeline of one small device call (bench's config-1 step, graph replay) from CUPTI
kernel records (torch.profiler): each kernel's start offset, duration and the idle gap
before it.   python scripts/small_call_timeline.py [cfg1]"""
import json
import os
import sys
import tempfile

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2501_13382_b200 import engine, shard  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
sc, src, launch, tcfg, c, obs_np = bench.make_inputs(dict(bench.CONFIGS[name]))
dev = torch.device("cuda", 0)
tr = engine.trace_device_rows(engine.DeviceScene.from_scene(sc, dev), src, launch, tcfg, c, 0,
                              len(launch), dev)
bundle = tr["bundle"]
obs_all = torch.from_numpy(obs_np).to(dev)
obs = obs_all.index_select(0, shard.tile_order(obs_all)).contiguous()
nf = src.omegas.shape[0]
acc = torch.zeros((obs.shape[0], nf), dtype=torch.complex128, device=dev)
ev = torch.zeros(obs.shape[0], dtype=torch.int64, device=dev)
busy = torch.zeros(64 * 1024 * 1024, dtype=torch.float32, device=dev)


def call():
    engine.accumulate(bundle, obs, src.omegas, -src.beam_param_im, True, acc, ev,
                      precision="fp32", presorted=True)


for _ in range(5):
    call()
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        for _ in range(20):
            busy.add_(1.0)  # the host gets ahead: the calls' own GPU timeline
        call()
    torch.cuda.synchronize()
path = os.path.join(tempfile.mkdtemp(), "t.json")
prof.export_chrome_trace(path)
evs = [e for e in json.load(open(path))["traceEvents"]
       if e.get("cat") in ("kernel", "gpu_memset", "gpu_memcpy")]
evs.sort(key=lambda e: e["ts"])
# the last call: everything after the last busy add
last_add = max(i for i, e in enumerate(evs) if "CUDAFunctorOnSelf_add" in e["name"])
call_evs = evs[last_add + 1:]
t0 = evs[last_add]["ts"] + evs[last_add]["dur"]
end_prev = t0
print(f"{name}: one call's GPU timeline (us; gap = idle since the previous record ended)")
for e in call_evs:
    gap = e["ts"] - end_prev
    print(f"{e['ts'] - t0:8.1f} {e['dur']:7.1f} gap {gap:6.1f}  {e['name'][:80]}")
    end_prev = max(end_prev, e["ts"] + e["dur"])
print(f"total {end_prev - t0:.1f} us, kernels {sum(e['dur'] for e in call_evs):.1f} us")

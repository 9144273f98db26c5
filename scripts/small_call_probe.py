"""Host vs device time of one small device call (bench's config-1 step):
    python scripts/small_call_probe.py [cfg1]
host  = wall time of the call while the GPU is still busy with earlier work (submission
        cost only: Python wrapper, C-ABI, graph launch);
gpu   = CUDA-event time of the call's work with the host ahead of the GPU;
step  = bench.py's step as timed there (flush, events, call, sync)."""
import sys
import time

import numpy as np
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
stream = torch.cuda.current_stream(dev)
busy = torch.zeros(64 * 1024 * 1024, dtype=torch.float32, device=dev)


def call():
    acc.zero_()
    ev.zero_()
    engine.accumulate(bundle, obs, src.omegas, -src.beam_param_im, True, acc, ev,
                      precision="fp32", stream=stream, presorted=True)


for _ in range(5):
    call()
torch.cuda.synchronize()

# host submission cost: queue ~3 ms of GPU work first, then time the calls' submission
host = []
for _ in range(50):
    for _ in range(40):
        busy.add_(1.0)
    t0 = time.perf_counter()
    call()
    host.append(1e3 * (time.perf_counter() - t0))
    torch.cuda.synchronize()

# device time with the host ahead
gpu = []
for _ in range(50):
    for _ in range(40):
        busy.add_(1.0)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    call()
    e1.record(stream)
    e1.synchronize()
    gpu.append(e0.elapsed_time(e1))

# pieces: the two zero_ alone, and back-to-back calls (throughput)
z = []
for _ in range(50):
    for _ in range(40):
        busy.add_(1.0)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    acc.zero_()
    ev.zero_()
    e1.record(stream)
    e1.synchronize()
    z.append(e0.elapsed_time(e1))
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(200):
    call()
torch.cuda.synchronize()
b2b = 1e3 * (time.perf_counter() - t0) / 200

print(f"{name}: host submit {np.median(host):.3f} ms, gpu {np.median(gpu):.3f} ms "
      f"(zero_ x2 {np.median(z):.3f}), back-to-back {b2b:.3f} ms/call")

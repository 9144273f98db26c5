"""Per-unit cycle distribution of one fp32 call (run with the BF_UNIT_TIMES=1 library variant,
scripts/build_variants.sh, and BF_UNIT_TIMES_OUT set):
    BF_UNIT_TIMES_OUT=gpurun_out/u.bin BF_GBS_LIB=.../libbf_gbs_-BF_UNIT_TIMES-1.so python scripts/unit_times.py cfg1"""
import os
import sys, numpy as np, torch
sys.path.insert(0, ".")
import bench
from paper_2501_13382_b200 import engine, shard
sc, src, launch, tcfg, c, obs_np = bench.make_inputs(dict(bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg1"]))
dev = torch.device("cuda", 0)
tr = engine.trace_device_rows(engine.DeviceScene.from_scene(sc, dev), src, launch, tcfg, c, 0, len(launch), dev)
b = tr["bundle"]
oa = torch.from_numpy(obs_np).to(dev)
obs = oa.index_select(0, shard.tile_order(oa)).contiguous()
acc = torch.zeros((obs.shape[0], 1), dtype=torch.complex128, device=dev)
ev = torch.zeros(obs.shape[0], dtype=torch.int64, device=dev)
engine.accumulate(b, obs, src.omegas, -src.beam_param_im, True, acc, ev, precision="fp32", presorted=True)
torch.cuda.synchronize()
raw = np.fromfile(os.environ.get("BF_UNIT_TIMES_OUT", "gpurun_out/unit_cycles.bin"), dtype=np.int64)
npat, nr, ppt = raw[:3]; cyc = raw[3:].astype(float)
print("units", cyc.size, "patches", npat, "ranges", nr, "sum cyc %.3e" % cyc.sum(), "mean %.0f max %.0f p50 %.0f p99 %.0f" % (cyc.mean(), cyc.max(), np.median(cyc), np.percentile(cyc, 99)))
print("sum/2368 warps = %.1f us at 1.9 GHz; max unit %.1f us" % (cyc.sum()/2368/1.9e3, cyc.max()/1.9e3))

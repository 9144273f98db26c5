"""Where the host-buffer (e2e) call spends its time on a bench config: device-path step vs
bf_gbs_accumulate on pageable / pinned numpy inputs, and the pieces around it.
    python scripts/e2e_probe.py [cfg3]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2501_13382_b200 import engine, kernels  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
cfg = dict(bench.CONFIGS[name])
sc, src, launch, tcfg, c, obs = bench.make_inputs(cfg)
dev = torch.device("cuda", 0)
tr = engine.trace_device_rows(engine.DeviceScene.from_scene(sc, dev), src, launch, tcfg, c,
                              0, len(launch), dev)
b = tr["bundle"]
torch.cuda.synchronize()
om = np.array([2 * np.pi * f for f in src.frequencies])
wb = -float(src.beam_param_im)
nb = b.n_segs.shape[0]
od = torch.from_numpy(obs).to(dev)
acc = torch.zeros((obs.shape[0], len(om)), dtype=torch.complex128, device=dev)
ev = torch.zeros(obs.shape[0], dtype=torch.int64, device=dev)


def dev_step():
    kernels.gbs_accumulate(b.seg_origin, b.seg_dir, b.seg_e1, b.seg_e2, b.seg_len, b.seg_s0,
                           b.seg_refl, b.n_segs, b.max_seg, b.weights, od, om, c, wb,
                           src.amplitude_phi, True, acc, ev, 0, obs.shape[0], 0, nb, precision="fp32")
    torch.cuda.synchronize()


hb = {k: getattr(b, k).cpu().numpy().copy() for k in engine.SEG_FIELDS + ("n_segs", "weights")}
obs_h = obs.copy()
acc_h = np.zeros((obs.shape[0], len(om)), np.complex128)
ev_h = np.zeros(obs.shape[0], np.int64)


def host_step(hb, obs_h, acc_h, ev_h):
    kernels.gbs_accumulate(hb["seg_origin"], hb["seg_dir"], hb["seg_e1"], hb["seg_e2"],
                           hb["seg_len"], hb["seg_s0"], hb["seg_refl"], hb["n_segs"], b.max_seg,
                           hb["weights"], obs_h, om, c, wb, src.amplitude_phi, True, acc_h,
                           ev_h, 0, obs.shape[0], 0, nb, precision="fp32")


def t(fn, n=3):
    fn()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return 1e3 * min(ts)


print(f"{name}: device step {t(dev_step):.2f} ms")
print(f"host step pageable {t(lambda: host_step(hb, obs_h, acc_h, ev_h)):.2f} ms")
pin = {k: torch.from_numpy(v).pin_memory().numpy() for k, v in hb.items()}
obs_p = torch.from_numpy(obs_h).pin_memory().numpy()
acc_p = torch.from_numpy(acc_h).pin_memory().numpy()
ev_p = torch.from_numpy(ev_h).pin_memory().numpy()
print(f"host step pinned   {t(lambda: host_step(pin, obs_p, acc_p, ev_p)):.2f} ms")
print(f"zero acc+evals (numpy) {t(lambda: (acc_h.fill(0), ev_h.fill(0))):.2f} ms")

# raw staging speeds on this host: pageable -> pinned memcpy, pinned H2D / D2H, driver pageable
big = np.random.default_rng(0).random(3 * 10**6)  # 24 MB
pin_t = torch.empty(big.shape, dtype=torch.float64).pin_memory()
pin_n = pin_t.numpy()
dev_t = torch.empty(big.shape, dtype=torch.float64, device=dev)
print(f"np.copyto 24 MB pageable->pinned {t(lambda: np.copyto(pin_n, big)):.2f} ms")
print(f"H2D 24 MB pinned {t(lambda: (dev_t.copy_(pin_t, non_blocking=True), torch.cuda.synchronize())):.2f} ms")
print(f"D2H 24 MB pinned {t(lambda: (pin_t.copy_(dev_t, non_blocking=True), torch.cuda.synchronize())):.2f} ms")
pg = torch.from_numpy(big)
print(f"H2D 24 MB pageable (driver) {t(lambda: (dev_t.copy_(pg), torch.cuda.synchronize())):.2f} ms")
print(f"D2H 24 MB pageable (driver) {t(lambda: pg.copy_(dev_t)):.2f} ms")
for i in range(5):
    print(f"host step pageable again {t(lambda: host_step(hb, obs_h, acc_h, ev_h), 1):.2f} ms")

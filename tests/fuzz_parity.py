"""Broad randomized parity fuzz of the fp32 path against the C oracle (GPU; test
infrastructure, not collected by pytest):

    python tests/fuzz_parity.py FIRST_SEED LAST_SEED          (fp32 mode)
    FUZZ_PREC=fp64 python tests/fuzz_parity.py FIRST LAST     (fp64 mode: rel <= 1e-12,
                                                              evaluation counts bit-exact)

Per seed: ground plane or city, source anywhere in a street (0.3-40 m high), 1-8
frequencies in 40-2000 Hz, beam parameter -1.5 .. -50000 (log-uniform), cutoff on/off,
0-8 reflections, a receiver grid (0.05-3 m spacing, 0-5 m high) plus up to 1500
scattered receivers (up to 300 m away, 0-30 m high) plus one AT the source.  Gates as
tests/test_gbs_gpu.py (relL2 <= 1e-4, dTL <= 0.01 dB within 60 dB of the maximum,
evaluation counts).  "ZERO" lines list receivers whose fp32 result underflowed to 0
(every contribution below ~1e-38 of the maximum; only reachable without the cutoff).
"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy as np, torch
import oracle
from conftest import rel_l2, tl_db
from paper_2501_13382_b200 import engine, kernels
from paper_2501_13382_b200.beamtrace import Atmosphere, LaunchGrid, SourceSpec, TraceConfig, launch_directions
from paper_2501_13382_b200.scene import make_city, make_ground_plane
dev = torch.device("cuda", 0)
PREC = os.environ.get("FUZZ_PREC", "fp32")
fails = []; worst = 0.0; worst_all = 0.0; n_all_over = 0
for seed in range(int(sys.argv[1]), int(sys.argv[2])):
    rng = np.random.default_rng(5000 + seed)
    kind = rng.integers(0, 3)
    if kind == 0:
        sc = make_ground_plane(float(rng.uniform(100, 2000)))
        src = np.array([rng.uniform(-20, 20), rng.uniform(-20, 20), rng.uniform(0.5, 30)])
    else:
        nx, ny = int(rng.integers(2, 7)), int(rng.integers(2, 7))
        sc = make_city(nx, ny, 40.0, 20.0, 300.0)
        xs = -(nx - 1) * 20.0 + 20.0 + 40.0 * np.arange(nx - 1)
        src = np.array([rng.choice(xs) + rng.uniform(-9, 9), rng.uniform(-100, 100), rng.uniform(0.3, 40.0)])
    nf = int(rng.integers(1, 9))
    freqs = tuple(float(f) for f in np.sort(rng.uniform(40, 2000, nf)))
    im_b = float(-np.exp(rng.uniform(np.log(1.5), np.log(50000))))
    use_cutoff = bool(rng.integers(0, 3) > 0)
    source = SourceSpec(position=src, frequencies=freqs, beam_param_im=im_b)
    launch = launch_directions(LaunchGrid(0.0, 180.0, 0.0, 360.0, int(rng.integers(10, 60)), int(rng.integers(20, 120))))
    cfg = TraceConfig(int(rng.integers(500, 6000)), 1e-4, int(rng.integers(1, 9)))
    c = Atmosphere(float(rng.uniform(-10, 40))).sound_speed
    tr = engine.trace_device_rows(engine.DeviceScene.from_scene(sc, dev), source, launch, cfg, c, 0, len(launch), dev)
    hb = tr["bundle"].to_host()
    parts = []
    sp = float(np.exp(rng.uniform(np.log(0.05), np.log(3.0))))
    n1, n2 = int(rng.integers(5, 60)), int(rng.integers(5, 60))
    X, Y = np.meshgrid(src[0] + rng.uniform(-60, 20) + sp * np.arange(n1), src[1] + rng.uniform(-60, 20) + sp * np.arange(n2), indexing="xy")
    parts.append(np.stack([X.ravel(), Y.ravel(), np.full(X.size, rng.uniform(0.0, 5.0))], axis=1))
    m = int(rng.integers(1, 1500))
    R = float(rng.uniform(1, 300))
    parts.append(np.stack([src[0] + rng.uniform(-R, R, m), src[1] + rng.uniform(-R, R, m), rng.uniform(0.0, 30.0, m)], axis=1))
    parts.append(src[None, :].copy())  # a receiver at the source
    obs = np.ascontiguousarray(np.concatenate(parts))
    om = source.omegas
    args = [hb.seg_origin, hb.seg_dir, hb.seg_e1, hb.seg_e2, hb.seg_len, hb.seg_s0, hb.seg_refl, hb.n_segs, hb.max_seg, hb.weights, obs, om, float(c), -float(source.beam_param_im), float(source.amplitude_phi), use_cutoff]
    nb = hb.n_segs.shape[0]
    ref = np.zeros((obs.shape[0], om.shape[0]), np.complex128); rev = np.zeros(obs.shape[0], np.int64)
    oracle.gbs_accumulate(*args, ref, rev, 0, obs.shape[0], 0, nb, threads=16)
    acc = np.zeros_like(ref); ev = np.zeros_like(rev)
    try:
        kernels.gbs_accumulate(*args, acc, ev, 0, obs.shape[0], 0, nb, precision=PREC)
    except Exception as e:
        fails.append((seed, "ERR " + repr(e)[:200])); continue
    if not np.any(ref):
        continue
    z = (np.abs(acc) == 0) & (np.abs(ref) > 0)
    if z.any():
        ii = np.argwhere(z)
        rl = 20 * np.log10(np.abs(ref[z]) / np.abs(ref).max())
        fails.append((seed, "ZERO", int(z.sum()), [tuple(x) for x in ii[:5]], obs.shape[0], [round(float(v), 1) for v in rl[:5]], "evref", [int(rev[i[0]]) for i in ii[:5]], "ev", [int(ev[i[0]]) for i in ii[:5]], "nf", nf, "cut", use_cutoff, "imb", round(im_b, 2)))
    l2 = rel_l2(acc, ref); t60 = tl_db(acc, ref, floor_db=-60.0); tall = tl_db(acc, ref)
    evd = abs(int(ev.sum()) - int(rev.sum()))
    worst = max(worst, t60)
    if np.isfinite(tall):
        worst_all = max(worst_all, tall)
        n_all_over += int(tall > 0.01)
        if tall > 0.01:  # where: the worst receiver's level below the field maximum
            nz = np.abs(ref) > 0
            d = np.full(ref.shape, 0.0)
            d[nz] = np.abs(20 * np.log10(np.abs(acc[nz]) / np.abs(ref[nz])))
            i = np.unravel_index(np.argmax(d), d.shape)
            lvl = 20 * np.log10(np.abs(ref[i]) / np.abs(ref).max())
            print("ALL", seed, "dTL %.4f at %.1f dB below max" % (tall, -lvl), "kind", int(kind),
                  "nf", nf, "cut", use_cutoff, "imb", round(im_b, 2), "sp", round(sp, 3),
                  "n>0.01", int((d > 0.01).sum()), "of", int(nz.sum()), flush=True)
    if PREC == "fp64":
        bad = l2 > 1e-12 or not np.array_equal(ev, rev)
    else:
        bad = l2 > 1e-4 or t60 > 0.01 or evd > 1e-4 * int(rev.sum()) + 10
    if bad:
        fails.append((seed, dict(kind=int(kind), nf=nf, im_b=round(im_b, 2), cut=use_cutoff, sp=round(sp, 3), R=round(R, 1), rmax=cfg.r_max if hasattr(cfg, 'r_max') else None, l2=l2, t60=t60, tall=tall, evd=evd, evsum=int(rev.sum()))))
print("fuzz2", sys.argv[1:], PREC, "failures", len(fails), "worst t60 %.4f" % worst,
      "worst all-receiver dTL %.4f" % worst_all, "seeds with all-receiver dTL > 0.01:", n_all_over)
for f in fails: print(f)

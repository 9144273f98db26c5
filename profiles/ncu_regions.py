#!/usr/bin/env python3
"""Instruction / stall share per region of gbs_fp32.cu in an ncu report, with regions
located by marker text in the report's own embedded source (robust to line shifts).

    python profiles/ncu_regions.py gpurun_out/X.ncu-rep
"""
import csv
import io
import subprocess
import sys

MARKERS = [  # (region name, first line containing this text starts the region)
    ("pick4", "T pick4("), ("consts/helpers", "struct Fp32Consts"),
    ("eval (tiny/freq/pair2)", "void tiny_contribution("), ("clamp2", "float clamp2("),
    ("classify", "float patch_dist("), ("behind_mask", "unsigned behind_mask("),
    ("junction", "struct Junction {"),
    ("exact_pick", "struct ExactPick"), ("exact_pending", "void exact_pending("),
    ("stage", "void stage_rows("), ("unit_head", "void run_unit("),
    ("gather", "// ---- gather the next"), ("rows", "// ---- row capacity"),
    ("workgen", "// ---- work generation"), ("liveloop", "// ---- summation over"),
    ("single", "// ---- single surviving"), ("wedge", "// ---- corner wedge"),
    ("multi", "// ---- several candidate"), ("tail", "// ---- shared tail"),
    ("flush", "// flush fp32 partial"), ("unit_out", "// ---- the unit's partial"),
    ("kernel", "__global__ void __launch_bounds__"), ("prep", "pack_kernel("),
]


def main():
    rep = sys.argv[1]
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    lines = [(int(x[0]), x[1], x) for x in rows[3:] if len(x) > 8 and x[0].isdigit()]
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source",
                          "cuda"], capture_output=True, text=True).stdout
    text = {int(x[0]): x[1] for x in csv.reader(io.StringIO(src)) if x and x[0].isdigit()}
    starts = []
    for name, mark in MARKERS:
        hit = [ln for ln, t in sorted(text.items()) if mark in t]
        if hit:
            starts.append((hit[0], name))
    starts.sort()

    def region(ln):
        cur = "preamble"
        for s, n in starts:
            if ln >= s:
                cur = n
        return cur

    def f(v):
        try:
            return float(v)
        except ValueError:
            return 0.0
    agg = {}
    for ln, _, x in lines:
        r = region(ln)
        a = agg.setdefault(r, [0.0, 0.0, 0.0])
        a[0] += f(x[4])
        a[1] += f(x[7])
        a[2] += f(x[8])
    ts = sum(v[0] for v in agg.values()) or 1
    ti = sum(v[1] for v in agg.values()) or 1
    print(f"{'region':16s} {'stall%':>7s} {'inst%':>7s} {'lanes%':>7s} {'warp-inst':>12s}")
    for r, (s_, i, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{r:16s} {s_ / ts * 100:7.1f} {i / ti * 100:7.1f} "
              f"{(t / i / 32 * 100 if i else 0):7.1f} {i:12.4g}")


if __name__ == "__main__":
    main()

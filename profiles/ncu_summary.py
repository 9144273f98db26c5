#!/usr/bin/env python3
"""Summarise an ncu --set full report of gbs_fp32_kernel: pipes, stalls, and the
stall / instruction share per source line and per kernel region.

    python profiles/ncu_summary.py gpurun_out/X.ncu-rep [--regions] [--top N]
"""
import argparse
import csv
import io
import re
import subprocess

KEYS = ["gpu__time_duration.sum", "launch__registers_per_thread", "launch__grid_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
        "smsp__thread_inst_executed_per_inst_executed.ratio",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "thread_inst_executed_true"]


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def raw(rep):
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    h, u, v = rows[0], rows[1], rows[2]
    out = {}
    for k, unit, x in zip(h, u, v):
        out[k] = (x, unit)
    return out


def fnum(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--top", type=int, default=30)
    ap.add_argument("--regions", default="", help="name:lo-hi,name:lo-hi (source lines)")
    args = ap.parse_args()
    r = raw(args.rep)
    for k in KEYS:
        if k in r:
            print(f"{k:60s} {r[k][0]} {r[k][1]}")
    stalls = sorted(((fnum(v), k) for k, (v, _) in r.items()
                     if re.match(r"smsp__average_warps_issue_stalled_.*_per_issue_active.ratio", k)),
                    reverse=True)
    print("stalls/issue: " + " ".join(
        f"{k.split('stalled_')[1].split('_per')[0]}={v:.2f}" for v, k in stalls if v > 0.02))
    rows = list(csv.reader(io.StringIO(ncu(args.rep, "--page", "source", "--csv",
                                            "--print-source", "cuda,sass"))))
    data = [x for x in rows[3:] if len(x) > 8 and x[0].isdigit()]
    tot = sum(fnum(x[4]) for x in data) or 1.0
    toti = sum(fnum(x[7]) for x in data) or 1.0
    print(f"\nper source line (stall samples {tot:.0f}, warp instructions {toti:.3g})")
    for x in sorted(data, key=lambda x: -fnum(x[4]))[:args.top]:
        print(f"{x[0]:>5} stall {fnum(x[4]) / tot * 100:5.1f}% inst {fnum(x[7]) / toti * 100:5.1f}%"
              f"  {x[1].strip()[:96]}")
    if args.regions:
        print("\nregions")
        for item in args.regions.split(","):
            name, rng = item.split(":")
            lo, hi = map(int, rng.split("-"))
            s = sum(fnum(x[4]) for x in data if lo <= int(x[0]) <= hi)
            i = sum(fnum(x[7]) for x in data if lo <= int(x[0]) <= hi)
            print(f"{name:28s} stall {s / tot * 100:5.1f}%  inst {i / toti * 100:5.1f}%")


if __name__ == "__main__":
    main()

#!/usr/bin/env python3
"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum --csv).

    python profiles/launch_summary.py launches.csv [--title "..."]
"""
import argparse
import collections
import csv


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--title", default="")
    args = ap.parse_args()
    with open(args.csv) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    rows = list(csv.DictReader(lines))
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0]
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}.get(
            r["Metric Unit"], 1e-6)
        tot[name] += float(r["Metric Value"].replace(",", "")) * scale
        cnt[name] += 1
    all_ms = sum(tot.values()) or 1.0
    if args.title:
        print(args.title)
    print("cold-cache, serialised per-launch times; kernel share of the whole run\n")
    for name, ms in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{name[:72]:72s} launches {cnt[name]:4d} total {ms:10.3f} ms  "
              f"mean {ms / cnt[name]:9.3f} ms  share {ms / all_ms * 100:5.1f}%")


if __name__ == "__main__":
    main()

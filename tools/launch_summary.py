"""Summarise an ncu launch list (gpu__time_duration.sum per launch, optionally
launch__grid_size): per (kernel, grid) totals, and the decode-step breakdown.
Usage: python tools/launch_summary.py gpurun_out/launches.csv"""
import collections
import csv
import re
import sys


def load(path):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", r["Kernel Name"]).replace("void ", "")
        rows.append((int(r["ID"]), name, r["Grid Size"], float(r["Metric Value"]) / 1e3))
    return rows


def main(path):
    rows = load(path)
    tot = sum(r[3] for r in rows)
    agg = collections.defaultdict(lambda: [0, 0.0])
    for _, n, g, us in rows:
        agg[(n, g)][0] += 1
        agg[(n, g)][1] += us
    print(f"{len(rows)} launches, {tot / 1e3:.2f} ms serialised")
    for (n, g), (c, us) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:30]:
        print(f"{100 * us / tot:6.2f}% {c:6d} x {us / c:9.2f} us  grid {g:14s} {n}")


if __name__ == "__main__":
    main(sys.argv[1])

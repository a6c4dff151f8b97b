#!/usr/bin/env python
"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch) into
per-kernel counts, mean durations and shares.  Usage:
    python tools/ncu_summary.py gpurun_out/launches.csv [> profiles/rNN/launches_summary.txt]"""
import collections
import csv
import re
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, vi, ui, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit"), hdr.index("Metric Name")
    out = []
    for r in rows[h + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[ui], 1.0)
        name = re.sub(r"\(.*", "", r[ki]).replace("void ", "")
        out.append((name, v * scale))
    return out


def main(path):
    rows = load(path)
    d = collections.defaultdict(list)
    for k, v in rows:
        d[k].append(v)
    tot = sum(v for _, v in rows)
    print(f"{'kernel':55s} {'launches':>8s} {'mean us':>9s} {'share':>7s}")
    for k, v in sorted(d.items(), key=lambda x: -sum(x[1])):
        print(f"{k[:55]:55s} {len(v):8d} {sum(v) / len(v):9.2f} {100 * sum(v) / tot:6.1f}%")
    print(f"total {len(rows)} launches, {tot:.1f} us (cold-cache, serialised: compare shares)")


if __name__ == "__main__":
    main(sys.argv[1])

# SPDX-License-Identifier: Apache-2.0
"""Summarises an ncu `--metrics gpu__time_duration.sum --csv` launch list by
kernel name: launches, total time, share.

  python profiles/launch_summary.py launches.csv [--skip N]
"""
import collections
import csv
import sys


def load(path, skip=0):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    out = []
    for r in rows[start + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "s": 1e6, "second": 1e6}[r[ui]]
        out.append((r[ki], v))  # (name, microseconds)
    return out[skip:]


def main():
    path = sys.argv[1]
    skip = int(sys.argv[sys.argv.index("--skip") + 1]) if "--skip" in sys.argv else 0
    launches = load(path, skip)
    agg = collections.defaultdict(lambda: [0, 0.0])
    for name, us in launches:
        short = name.split("(")[0].replace("asg::<unnamed>::", "").replace("void ", "")[:70]
        agg[short][0] += 1
        agg[short][1] += us
    tot = sum(a[1] for a in agg.values())
    print(f"{len(launches)} launches, {tot / 1e3:.3f} ms total (serialised, cold-cache ncu replay)")
    print(f"{'kernel':70s} {'n':>6s} {'ms':>10s} {'share':>6s}")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:70s} {c:6d} {t / 1e3:10.3f} {100 * t / tot:5.1f}%")


if __name__ == "__main__":
    main()

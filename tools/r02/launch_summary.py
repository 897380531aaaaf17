"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: launches, total ms and
share per kernel (serialised cold-cache replay: shares, not absolute step time)."""
import collections
import csv
import sys

lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
agg = collections.defaultdict(lambda: [0, 0.0])
for r in csv.DictReader(lines):
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    n = r["Kernel Name"].split("(")[0]
    n = n.replace("void ", "").replace("asg::<unnamed>::", "").replace("asg::", "")[:70]
    agg[n][0] += 1
    agg[n][1] += float(r["Metric Value"]) / 1e6
tot = sum(v[1] for v in agg.values())
print(f"{sum(v[0] for v in agg.values())} launches, {tot:.3f} ms total (serialised, cold-cache ncu replay)")
print(f"{'kernel':72s} {'n':>5s} {'ms':>9s} share")
for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 16]:
    print(f"{n:72s} {c:5d} {t:9.3f} {100 * t / tot:5.1f}%")

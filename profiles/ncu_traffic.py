# SPDX-License-Identifier: Apache-2.0
"""Per-launch summary of an `ncu --set full` report: duration, DRAM bytes
(read + write), tensor-pipe and DRAM utilisation, registers, for every
captured kernel.

  python profiles/ncu_traffic.py report.ncu-rep [--json WORKLOAD KERNEL_REGEX ALG_BYTES OUT.json]

With --json, the launch of KERNEL_REGEX with the largest duration is written
into OUT.json under WORKLOAD (the `traffic` field bench.py reports).
"""
import csv
import io
import json
import re
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "%": 1, "register/thread": 1, "": 1}


def rows(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True, check=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units = r[0], r[1]
    res = []
    for row in r[2:]:
        d = {"kernel": row[hdr.index("Kernel Name")]}
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                try:
                    d[m] = float(row[i].replace(",", "")) * SCALE.get(units[i], 1)
                except ValueError:
                    d[m] = None
        res.append(d)
    return res


def main():
    path = sys.argv[1]
    rs = rows(path)
    print(f"{'kernel':60s} {'us':>9s} {'DRAM MB':>9s} {'GB/s':>7s} {'tc%':>6s} {'dram%':>6s} {'sm%':>6s}")
    for d in rs:
        t = d.get("gpu__time_duration.sum") or 0
        b = (d.get("dram__bytes_read.sum") or 0) + (d.get("dram__bytes_write.sum") or 0)
        tc = d.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active")
        if tc is None:
            tc = d.get("sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active")
        print(f"{d['kernel'][:60]:60s} {t * 1e6:9.1f} {b / 1e6:9.1f} {b / t / 1e9 if t else 0:7.0f} "
              f"{tc or 0:6.1f} {d.get('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed') or 0:6.1f} "
              f"{d.get('sm__throughput.avg.pct_of_peak_sustained_elapsed') or 0:6.1f}")
    if "--json" in sys.argv:
        i = sys.argv.index("--json")
        wl, rx, alg, out = sys.argv[i + 1], sys.argv[i + 2], float(sys.argv[i + 3]), sys.argv[i + 4]
        cand = [d for d in rs if re.search(rx, d["kernel"])]
        top = max(cand, key=lambda d: d.get("gpu__time_duration.sum") or 0)
        try:
            doc = json.load(open(out))
        except FileNotFoundError:
            doc = {}
        doc[wl] = {"kernel": top["kernel"][:120],
                   "dram_bytes_per_launch": (top.get("dram__bytes_read.sum") or 0) + (top.get("dram__bytes_write.sum") or 0),
                   "alg_bytes_per_launch": alg, "duration_s": top.get("gpu__time_duration.sum"),
                   "source": f"ncu --set full --clock-control none ({path.split('/')[-1]}), longest launch of /{rx}/"}
        json.dump(doc, open(out, "w"), indent=1)
        print("wrote", out, doc[wl])


if __name__ == "__main__":
    main()

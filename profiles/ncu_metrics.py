# SPDX-License-Identifier: Apache-2.0
"""Prints the raw `ncu --set full` metrics whose names match the given
regular expressions, for every kernel captured in a report (profiling tool,
not a test).

  python profiles/ncu_metrics.py report.ncu-rep REGEX [REGEX ...]
"""
import csv
import io
import re
import subprocess
import sys


def main():
    path, pats = sys.argv[1], [re.compile(p) for p in sys.argv[2:]]
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units = r[0], r[1]
    cols = [i for i, h in enumerate(hdr) if any(p.search(h) for p in pats)]
    for row in r[2:]:
        print("==", row[hdr.index("Kernel Name")][:100])
        for i in cols:
            print(f"  {hdr[i]:90s} {row[i]:>16s} {units[i]}")


if __name__ == "__main__":
    main()

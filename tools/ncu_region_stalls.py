#!/usr/bin/env python
"""Stall reasons summed over SASS index ranges of one kernel (no GPU needed).

  python tools/ncu_region_stalls.py report.ncu-rep k_sweep_ws 200:1400 1400:3000
"""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
iE = h.index("Instructions Executed")
data = rows[2:]
for spec in sys.argv[3:]:
    a, b = (int(x) for x in spec.split(":"))
    acc = collections.Counter()
    ex = 0.0
    for r in data[a:b]:
        try:
            ex += float(r[iE] or 0)
            for c in reasons:
                acc[c] += float(r[h.index(c)] or 0)
        except ValueError:
            pass
    tot = sum(acc.values())
    print(f"[{a}:{b}] exec {ex:.3e} samples {tot:.0f}: " +
          ", ".join(f"{k[6:]}={100 * v / max(tot, 1):.0f}%" for k, v in acc.most_common(7)))

#!/usr/bin/env python
"""Executed-instruction mix of one kernel by SASS opcode (no GPU needed).

  python tools/ncu_opmix.py report.ncu-rep k_sweep_a
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
iS, iE = h.index("Source"), h.index("Instructions Executed")
mix = collections.Counter()
tot = 0
for r in rows[2:]:
    try:
        e = float(r[iE])
    except (ValueError, IndexError):
        continue
    src = r[iS].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    mix[op] += e
    tot += e
print(f"total {tot:.3e}")
for op, e in mix.most_common(30):
    print(f"{op:10s} {e:12.3e} {100 * e / tot:5.1f}%")
